// Drop-in check: the reference's own code (rangelib, compiled unmodified from
// /root/reference/proj/src) driven with rl_gpu::GpuCddtMethod
// (include/rl_cddt_rangemethod.hpp) in place of its CPU CDDT, plus the
// reference's release gate (proj/tests/test_acceptance.cpp) criteria 2, 3, 4,
// 9 and 10 run through the GPU path. Built by `make -C oracle dropin` into
// oracle/_ref/dropin_check; run on the GPU box by tests/test_gpu_dropin.py.
// Prints one PASS/FAIL line per criterion.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>
#include <random>
#include <vector>

#include "rangelib/cddt.hpp"
#include "rangelib/mcl.hpp"
#include "rangelib/methods.hpp"
#include "rangelib/raycast.hpp"
#include "rangelib/rng.hpp"
#include "rangelib/synthetic.hpp"
#include "rl_cddt_mcl.hpp"
#include "rl_cddt_rangemethod.hpp"

using namespace rangelib;

static int g_fail = 0;
static void report(const char* what, bool ok, long detail) {
  std::printf("DROPIN %s %s (%ld)\n", ok ? "PASS" : "FAIL", what, detail);
  if (!ok) g_fail++;
}

// ---- the reference's acceptance gate (proj/tests/test_acceptance.cpp) through the GPU ----

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// device array of n doubles / ints, filled from host
template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t n_) : n(n_) {
    if (cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
  }
  Dev(const std::vector<T>& h) : Dev(h.size()) { put(h); }
  ~Dev() { cudaFree(p); }
  void put(const std::vector<T>& h) { cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice); }
  std::vector<T> get() const {
    std::vector<T> h(n);
    cudaMemcpy(h.data(), p, sizeof(T) * n, cudaMemcpyDeviceToHost);
    return h;
  }
};

// every (cell centre, lattice direction) state of a w x h map, as directional_batch input
struct States {
  std::vector<double> x, y;
  std::vector<int32_t> a;
  States(int w, int h, int K) {
    for (int d = 0; d < K; d++)
      for (int yy = 0; yy < h; yy++)
        for (int xx = 0; xx < w; xx++) {
          x.push_back(xx + 0.5);
          y.push_back(yy + 0.5);
          a.push_back(d);
        }
  }
};

static std::vector<double> gpu_states(rl_cddt* h, const States& st) {
  Dev<double> dx(st.x), dy(st.y), out(st.x.size());
  Dev<int32_t> da(st.a);
  rl_gpu::throw_on(rl_cddt_directional_batch(h, dx.p, dy.p, da.p, out.p, st.x.size(), nullptr));
  return out.get();
}

// 2. cddt and pcddt (the GPU structures) within 2 px of the exact oracle on
//    500 random queries per map over 20 random 64x64 maps (cddt: random
//    positions at lattice angles; pcddt: cell-centre lattice states), the
//    reference's sampling (test_acceptance.cpp:107-155).
static void acceptance_2() {
  double t0 = now_s();
  RangeMethodConfig cfg;
  const int K = cfg.theta_disc;
  long violations = 0, equal_ref = 0, total = 0;
  double worst = 0.0;
  for (int m = 0; m < 20; m++) {
    OccupancyGrid g = make_random_map(64, 64, 0.08, 1000 + m);
    const double mr = cfg.resolved_max_range(g);
    for (bool prune : {false, true}) {
      rl_gpu::GpuCddtMethod gpu(g, cfg, prune);
      auto ref = make_method(prune ? MethodKind::pcddt : MethodKind::cddt, g, cfg);
      std::mt19937 rng(7000 + m);
      std::uniform_real_distribution<double> ux(0.0, 64.0), uy(0.0, 64.0);
      std::uniform_int_distribution<int> ucell(0, 63), udir(0, K - 1);
      std::vector<double> xs, ys;
      std::vector<int32_t> as;
      for (int i = 0; i < 500; i++) {
        if (!prune) {
          xs.push_back(ux(rng));
          ys.push_back(uy(rng));
        } else {
          xs.push_back(ucell(rng) + 0.5);
          ys.push_back(ucell(rng) + 0.5);
        }
        as.push_back(udir(rng));
      }
      // batched through the C ABI (RayQuery(x, y, a * 2pi / K) maps back to direction a)
      Dev<double> dx(xs), dy(ys), out(xs.size());
      Dev<int32_t> da(as);
      rl_gpu::throw_on(rl_cddt_directional_batch(gpu.handle(), dx.p, dy.p, da.p, out.p, xs.size(), nullptr));
      std::vector<double> got = out.get();
      for (size_t i = 0; i < xs.size(); i++, total++) {
        RayQuery q(xs[i], ys[i], as[i] * kTwoPi / K);
        const double want = oracle_cast(g, q, mr);
        const double err = std::abs(got[i] - want);
        worst = std::max(worst, err);
        violations += err > 2.0;
        equal_ref += got[i] == ref->cast(q);
        // and the per-ray RangeMethod path agrees with the batched one
        if (i < 50 && gpu.cast(q) != got[i]) violations++;
      }
    }
  }
  char buf[200];
  std::snprintf(buf, sizeof buf, "acceptance 02: GPU cddt/pcddt within 2 px of the oracle on %ld queries, 20 maps (worst %.4f px, %.2f s)",
                total, worst, now_s() - t0);
  report(buf, violations == 0 && equal_ref == total, violations + (total - equal_ref));
}

// 3. The GPU-pruned structure equals the GPU-unpruned one, and both equal the
//    reference's unpruned Cddt, at every (cell centre, lattice direction)
//    state of 10 random 48x48 maps at K = 216 (test_acceptance.cpp:157-185).
static void acceptance_3() {
  double t0 = now_s();
  RangeMethodConfig cfg;
  long long states = 0, mism = 0;
  for (int m = 0; m < 10; m++) {
    OccupancyGrid g = make_random_map(48, 48, 0.08, 3000 + m);
    rl_gpu::GpuCddtMethod fresh(g, cfg, false), pruned(g, cfg, true);
    Cddt ref(g, cfg);
    States st(48, 48, cfg.theta_disc);
    std::vector<double> a = gpu_states(fresh.handle(), st), b = gpu_states(pruned.handle(), st);
    for (size_t i = 0; i < a.size(); i++, states++) {
      const double want = ref.directional_cast(st.x[i], st.y[i], st.a[i], nullptr);
      mism += (a[i] != want) + (b[i] != want);
    }
  }
  char buf[200];
  std::snprintf(buf, sizeof buf, "acceptance 03: GPU pcddt == GPU cddt == reference at %lld discrete states (%.2f s)",
                states, now_s() - t0);
  report(buf, mism == 0 && states == 10LL * 48 * 48 * 216, mism);
}

static void export_bins(rl_cddt* h, std::vector<uint64_t>* off, std::vector<float>* zp) {
  rl_cddt_info_t info;
  rl_gpu::throw_on(rl_cddt_info(h, &info));
  off->assign(info.rows + 1, 0);
  zp->assign(std::max<uint64_t>(info.zero_points, 1), 0.f);
  rl_gpu::throw_on(rl_cddt_export(h, nullptr, off->data(), zp->data(), nullptr, nullptr));
  zp->resize(info.zero_points);
}

// 4. After 200 random cell toggles (one set_occupancy each) the live GPU
//    structure answers every discrete state like a fresh GPU build and the
//    reference's fresh build, and inserting then removing 30 cells restores
//    every bin (test_acceptance.cpp:187-250), on 3 random 32x32 maps.
static void acceptance_4() {
  double t0 = now_s();
  RangeMethodConfig cfg;
  const int W = 32, H = 32;
  long long cast_mism = 0, bin_mism = 0;
  for (int m = 0; m < 3; m++) {
    OccupancyGrid g = make_random_map(W, H, 0.06, 4000 + m);
    rl_gpu::GpuCddtMethod live(g, cfg, false);
    std::mt19937 rng(4500 + m);
    std::uniform_int_distribution<int> ux(0, W - 1), uy(0, H - 1);
    for (int e = 0; e < 200; e++) {
      int x = ux(rng), y = uy(rng);
      bool occ = !g.at(x, y);
      g.set(x, y, occ);
      live.set_occupancy(x, y, occ);
    }
    rl_gpu::GpuCddtMethod fresh(g, cfg, false);
    Cddt ref(g, cfg);
    States st(W, H, cfg.theta_disc);
    std::vector<double> a = gpu_states(live.handle(), st), b = gpu_states(fresh.handle(), st);
    for (size_t i = 0; i < a.size(); i++) {
      const double want = ref.directional_cast(st.x[i], st.y[i], st.a[i], nullptr);
      cast_mism += (a[i] != want) + (b[i] != want);
    }
    std::vector<uint64_t> off0, off1;
    std::vector<float> zp0, zp1;
    export_bins(live.handle(), &off0, &zp0);
    std::vector<std::pair<int, int>> added;
    while (added.size() < 30) {
      int x = ux(rng), y = uy(rng);
      if (g.at(x, y)) continue;
      bool dup = false;
      for (auto& c : added) dup = dup || (c.first == x && c.second == y);
      if (!dup) added.push_back({x, y});
    }
    for (auto& c : added) live.set_occupancy(c.first, c.second, true);
    for (auto& c : added) live.set_occupancy(c.first, c.second, false);
    export_bins(live.handle(), &off1, &zp1);
    bin_mism += (off0 != off1) + (zp0 != zp1);
  }
  char buf[200];
  std::snprintf(buf, sizeof buf, "acceptance 04: 200-edit GPU structure == rebuild == reference at every state; insert+remove restores bins (%.2f s)",
                now_s() - t0);
  report(buf, cast_mism == 0 && bin_mism == 0, cast_mism + bin_mism);
}

// 9/10. Closed-loop localisation on the reference's 128x128 loop map
// (make_loop_map) with 1000 particles and a 61-beam 270 degree scan, the
// scenario of run_loop_demo (proj/include/rangelib/demo.hpp:12-31): a robot
// circles the map centre at radius 0.32 * min(w, h), 1.5 px per step, 200
// steps; odometry corrupted by N(0, 1.5 px) / N(0, 0.04 rad); scans from the
// reference's simulate_scan with sigma 6 px; re-seeded at the truth when the
// error exceeds 20 px. The filter under test is the GPU one (rl_gpu::GpuMcl,
// include/rl_cddt_mcl.hpp: rl_mcl_step's motion, fused sensor model,
// estimate and resampling); the ray-marching and LUT backends run the
// reference's own Mcl on the same sensor data.
struct LoopResult {
  double median_error = 0.0;
  int resets = 0;
};

static void pose_on_loop(const OccupancyGrid& g, int step, double* x, double* y, double* th) {
  const double cx = g.width() / 2.0, cy = g.height() / 2.0;
  const double r = 0.32 * std::min(g.width(), g.height());
  const double phi = 1.5 * step / r;  // arc length 1.5 px per step
  *x = cx + r * std::cos(phi);
  *y = cy + r * std::sin(phi);
  *th = normalize_angle_2pi(phi + kTwoPi / 4.0);  // tangent, counter-clockwise
}

static LoopResult run_loop(const OccupancyGrid& g, int K, const RangeMethod* ref_method,
                           bool gpu_prune, uint64_t seed) {
  const int steps = 200;
  const double step_px = 1.5, scan_sigma = 6.0, odo_t = 1.5, odo_r = 0.04;
  MclConfig fc;  // 1000 particles, 61 beams over 270 degrees
  fc.particle_count = 1000;
  fc.motion.trans_per_trans = (1.25 * odo_t + 0.05) / step_px;
  fc.motion.rot_per_trans = (1.25 * odo_r + 0.002) / step_px;
  fc.beam.sigma_hit = scan_sigma;
  fc.seed = seed;
  RangeMethodConfig cfg;
  cfg.theta_disc = K;
  // the filter under test: the reference's Mcl over a reference method, or
  // rl_gpu::GpuMcl (include/rl_cddt_mcl.hpp) over the GPU structure
  std::unique_ptr<rl_gpu::GpuCddtMethod> gpu;
  std::unique_ptr<Mcl> cpu;
  std::unique_ptr<rl_gpu::GpuMcl> gmcl;
  if (ref_method) {
    cpu = std::make_unique<Mcl>(*ref_method, fc);
  } else {
    gpu = std::make_unique<rl_gpu::GpuCddtMethod>(g, cfg, gpu_prune);
    gmcl = std::make_unique<rl_gpu::GpuMcl>(*gpu, fc);
  }
  const double mr = ref_method ? ref_method->max_range() : gpu->max_range();
  auto seed_at = [&](double x, double y, double th) {
    if (cpu)
      cpu->init_gaussian(x, y, th, 2.0, 0.1);
    else
      gmcl->init_gaussian(x, y, th, 2.0, 0.1);
  };
  std::mt19937_64 world(seed ^ 0x9e3779b97f4a7c15ull);
  std::normal_distribution<double> nt(0.0, odo_t), nr(0.0, odo_r);
  double tx, ty, tth;
  pose_on_loop(g, 0, &tx, &ty, &tth);
  seed_at(tx, ty, tth);
  std::vector<double> errs;
  LoopResult res;
  for (int step = 1; step <= steps; step++) {
    double nx, ny, nth;
    pose_on_loop(g, step, &nx, &ny, &nth);
    const double wx = nx - tx, wy = ny - ty, c = std::cos(tth), s = std::sin(tth);
    const double dx = wx * c + wy * s, dy = -wx * s + wy * c;
    const double dth = normalize_angle_pi(nth - tth);
    tx = nx;
    ty = ny;
    tth = nth;
    const double ox = dx + nt(world), oy = dy + nt(world), oth = dth + nr(world);
    std::vector<double> scan = simulate_scan(g, tx, ty, tth, fc.scan, mr, scan_sigma, world);
    const MclStepResult r = cpu ? cpu->step(ox, oy, oth, scan) : gmcl->step(ox, oy, oth, scan);
    const double err = std::hypot(r.estimate.x - tx, r.estimate.y - ty);
    if (step > 10) errs.push_back(err);
    if (err > 20.0) {
      seed_at(tx, ty, tth);
      if (step > 10) res.resets++;
    }
  }
  std::sort(errs.begin(), errs.end());
  res.median_error = errs[errs.size() / 2];
  return res;
}

static void acceptance_9_10() {
  double t0 = now_s();
  OccupancyGrid g = make_loop_map(128, 128);
  RangeMethodConfig cfg216;
  auto rm = make_method(MethodKind::ray_march, g, cfg216);
  auto lut = make_method(MethodKind::lut, g, cfg216);
  const LoopResult gc = run_loop(g, 216, nullptr, false, 1), gp = run_loop(g, 216, nullptr, true, 1);
  const LoopResult rr = run_loop(g, 216, rm.get(), false, 1), rlut = run_loop(g, 216, lut.get(), false, 1);
  const LoopResult g8 = run_loop(g, 8, nullptr, false, 1);
  double lo = gc.median_error, hi = gc.median_error;
  for (const LoopResult* r : {&gp, &rr, &rlut}) {
    lo = std::min(lo, r->median_error);
    hi = std::max(hi, r->median_error);
  }
  std::printf("  loop: GPU cddt %.3f px (%d resets), GPU pcddt %.3f (%d), ref rm %.3f (%d), ref lut %.3f (%d), GPU cddt@8 %.3f (%d)\n",
              gc.median_error, gc.resets, gp.median_error, gp.resets, rr.median_error, rr.resets,
              rlut.median_error, rlut.resets, g8.median_error, g8.resets);
  char buf[220];
  const bool c9 = gc.median_error < 3.0 && gc.resets <= 1 && gp.median_error < 3.0 &&
                  gp.resets <= 1 && hi <= 1.5 * lo;
  std::snprintf(buf, sizeof buf, "acceptance 09: GPU filter converges (median < 3 px, <= 1 reset), backend spread within 50%% (%.2f s)",
                now_s() - t0);
  report(buf, c9, long(1000 * gc.median_error));
  const bool c10 = double(g8.resets) >= 2.0 * double(gc.resets) &&
                   gc.median_error <= 1.5 * rr.median_error;
  std::snprintf(buf, sizeof buf, "acceptance 10: 8 directions reset >= 2x as often as 216; GPU cddt error within 1.5x of rm");
  report(buf, c10, g8.resets);
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
  // 5. run_batches' inner loop (proj/src/bench.cpp:86-106) over a std::vector<RayQuery>,
  //    as one cast_many call: ranges bit-identical to the reference's cast loop
  {
    OccupancyGrid g = make_random_map(96, 80, 0.07, 21);
    RangeMethodConfig cfg;
    long diff = 0;
    for (bool prune : {false, true}) {
      auto ref = make_method(prune ? MethodKind::pcddt : MethodKind::cddt, g, cfg);
      rl_gpu::GpuCddtMethod gpu(g, cfg, prune);
      SplitMix64 rng(123);
      std::vector<RayQuery> buf;
      for (int i = 0; i < 200000; i++)
        buf.emplace_back(rng.uniform(-1.0, 97.0), rng.uniform(-1.0, 81.0), rng.uniform(-7.0, 7.0));
      std::vector<double> out(buf.size());
      gpu.cast_many(buf.data(), buf.size(), out.data());
      for (size_t i = 0; i < buf.size(); i++) diff += ref->cast(buf[i]) != out[i];
    }
    report("cast_many(std::vector<RayQuery>) bit-identical to the reference's cast loop", diff == 0,
           diff);
  }
  acceptance_2();
  acceptance_3();
  acceptance_4();
  acceptance_9_10();
  return g_fail ? 1 : 0;
}
