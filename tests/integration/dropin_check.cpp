// Drop-in check: the reference's own code (rangelib, compiled unmodified from
// /root/reference/proj/src) driven with rl_gpu::GpuCddtMethod
// (include/rl_cddt_rangemethod.hpp) in place of its CPU CDDT. Built by
// `make -C oracle dropin` into oracle/_ref/dropin_check; run on the GPU box by
// tests/test_gpu_dropin.py. Prints one PASS/FAIL line per criterion.
#include <cstdio>
#include <memory>
#include <vector>

#include "rangelib/cddt.hpp"
#include "rangelib/mcl.hpp"
#include "rangelib/methods.hpp"
#include "rangelib/rng.hpp"
#include "rangelib/synthetic.hpp"
#include "rl_cddt_rangemethod.hpp"

using namespace rangelib;

static int g_fail = 0;
static void report(const char* what, bool ok, long detail) {
  std::printf("DROPIN %s %s (%ld)\n", ok ? "PASS" : "FAIL", what, detail);
  if (!ok) g_fail++;
}

int main() {
  // 1. casts and paired casts on the acceptance gate's random maps
  //    (proj/tests/test_acceptance.cpp:85-105), CDDT and PCDDT
  long bad = 0, total = 0;
  for (int m = 0; m < 4; m++) {
    OccupancyGrid g = make_random_map(64, 64, 0.08, 1000 + m);
    RangeMethodConfig cfg;  // theta_disc 216, max_range = diagonal
    for (bool prune : {false, true}) {
      auto ref = make_method(prune ? MethodKind::pcddt : MethodKind::cddt, g, cfg);
      rl_gpu::GpuCddtMethod gpu(g, cfg, prune);
      if (ref->memory_bytes() != gpu.memory_bytes()) bad++;
      SplitMix64 rng(77 + m);
      for (int i = 0; i < 1500; i++, total++) {
        RayQuery q(rng.uniform(-2.0, 66.0), rng.uniform(-2.0, 66.0), rng.uniform(-10.0, 10.0));
        if (ref->cast(q) != gpu.cast(q)) bad++;
        auto a = ref->cast_pair(q), b = gpu.cast_pair(q);
        if (a != b) bad++;
      }
    }
  }
  report("cast/cast_pair bit-identical to the reference CDDT/PCDDT", bad == 0, bad);

  // 2. the reference's sensor_update with the GPU method: weights identical
  {
    OccupancyGrid g = make_loop_map(128, 128);
    RangeMethodConfig cfg;
    auto ref = make_method(MethodKind::cddt, g, cfg);
    rl_gpu::GpuCddtMethod gpu(g, cfg, false);
    std::mt19937_64 rng(5);
    ScanSpec spec;
    BeamModelParams beam;
    beam.z_max = ref->max_range();
    std::vector<double> scan = simulate_scan(g, 40.5, 30.25, 0.3, spec, ref->max_range(), 2.0, rng);
    std::vector<Particle> pa(300), pb;
    std::normal_distribution<double> n(0.0, 4.0);
    for (auto& p : pa) p = Particle{40.5 + n(rng), 30.25 + n(rng), 0.3 + 0.05 * n(rng), 1.0 / 300};
    pb = pa;
    bool oka = sensor_update(pa, *ref, scan, spec, beam);
    bool okb = sensor_update(pb, gpu, scan, spec, beam);
    long diff = 0;
    for (size_t i = 0; i < pa.size(); i++) diff += pa[i].weight != pb[i].weight;
    report("sensor_update weights bit-identical (paired path)", oka == okb && diff == 0, diff);
  }

  // 3. the reference's Mcl closed loop: identical estimates step by step
  {
    OccupancyGrid g = make_loop_map(128, 128);
    RangeMethodConfig cfg;
    auto ref = make_method(MethodKind::cddt, g, cfg);
    rl_gpu::GpuCddtMethod gpu(g, cfg, false);
    MclConfig fc;
    fc.particle_count = 150;
    fc.seed = 9;
    Mcl a(*ref, fc), b(gpu, fc);
    a.init_gaussian(64.0, 22.0, 0.0, 3.0, 0.05);
    b.init_gaussian(64.0, 22.0, 0.0, 3.0, 0.05);
    std::mt19937_64 world(11);
    double x = 64.0, y = 22.0, th = 0.0;
    long diff = 0;
    for (int k = 0; k < 15; k++) {
      th += 0.03;
      x += 1.5 * std::cos(th);
      y += 1.5 * std::sin(th);
      std::vector<double> scan = simulate_scan(g, x, y, th, fc.scan, ref->max_range(), 2.0, world);
      MclStepResult ra = a.step(1.5, 0.0, 0.03, scan), rb = b.step(1.5, 0.0, 0.03, scan);
      diff += ra.estimate.x != rb.estimate.x || ra.estimate.y != rb.estimate.y ||
              ra.estimate.theta != rb.estimate.theta;
    }
    report("Mcl::step estimates bit-identical over a closed loop", diff == 0, diff);
  }

  // 4. errors surface as the reference's exception types
  {
    OccupancyGrid g = make_random_map(16, 16, 0.1, 3);
    bool ok = false;
    try {
      RangeMethodConfig bad_cfg;
      bad_cfg.theta_disc = 7;
      rl_gpu::GpuCddtMethod m(g, bad_cfg, false);
    } catch (const std::invalid_argument&) {
      ok = true;
    }
    rl_gpu::GpuCddtMethod p(g, RangeMethodConfig{}, true);
    bool ok2 = false;
    try {
      p.set_occupancy(1, 1, true);
    } catch (const std::logic_error&) {
      ok2 = true;
    }
    report("invalid_argument / logic_error mapping", ok && ok2, 0);
  }
  return g_fail ? 1 : 0;
}
