// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library (rangelib,
// compiled from its own sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/librangelib_ref.so). It only calls the
// reference's public API: Cddt (proj/include/rangelib/cddt.hpp:149-196),
// make_method (methods.hpp:53-54), sensor_update / beam_likelihood
// (mcl.hpp:68-70, :59), serialize_cddt / deserialize_cddt (cddt.hpp:245-246).
//
// Used by tests/ to pin the C restatement (oracle/cddt_oracle.c) and the GPU
// path, and by bench.py --impl reference / cpu_baseline as the reference's
// own CPU implementation timed on the host cores.
#include <chrono>
#include <time.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "rangelib/bench.hpp"
#include "rangelib/cddt.hpp"
#include "rangelib/grid.hpp"
#include "rangelib/mcl.hpp"
#include "rangelib/methods.hpp"
#include "rangelib/raycast.hpp"

using namespace rangelib;

namespace {

enum { RS_OK = 0, RS_EINVAL = 1, RS_ELOGIC = 2, RS_ERANGE = 3, RS_EPARSE = 7, RS_EOTHER = 9 };

struct RefCddt {
  Cddt c;
  std::vector<size_t> row_base;  // global row index of (s, 0)
  explicit RefCddt(Cddt&& x) : c(std::move(x)) { index(); }
  void index() {
    row_base.assign(size_t(c.slice_count()) + 1, 0);
    for (int s = 0; s < c.slice_count(); s++) row_base[s + 1] = row_base[s] + size_t(c.slice(s).bin_count);
  }
};

// Captures the resolving candidate of one directional_cast (cddt.hpp:141-144).
struct LastMark final : MarkSink {
  int slice = -1, row = -1;
  size_t index = 0;
  void mark(int s, int r, size_t i, bool) override {
    slice = s;
    row = r;
    index = i;
  }
};

// RangeMethod view of a Cddt, as CddtMethod does (proj/src/methods.cpp:79-97);
// `paired` false mirrors UnpairedView (proj/tests/test_mcl.cpp:21-31).
class CddtView final : public RangeMethod {
 public:
  CddtView(const Cddt& c, bool paired) : c_(c), paired_(paired) { max_range_ = c.max_range(); }
  const char* name() const override { return "cddt-view"; }
  double cast(const RayQuery& q) const override { return c_.cast(q); }
  std::pair<double, double> cast_pair(const RayQuery& q) const override { return c_.cast_pair(q); }
  bool supports_paired_cast() const override { return paired_; }
  int direction_count() const override { return c_.theta_disc(); }
  size_t memory_bytes() const override { return c_.memory_bytes(); }

 private:
  const Cddt& c_;
  bool paired_;
};

OccupancyGrid make_grid(const uint8_t* g, int w, int h, double res) {
  OccupancyGrid grid(w, h, res);
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++)
      if (g[size_t(y) * w + x]) grid.set(x, y, true);
  return grid;
}

template <class F>
void parallel_for(size_t n, int nthreads, F&& f) {
  if (nthreads <= 1 || n < 1024) {
    f(size_t(0), n);
    return;
  }
  std::vector<std::thread> ts;
  size_t chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; t++) {
    size_t a = t * chunk, b = std::min(n, a + chunk);
    if (a >= b) break;
    ts.emplace_back([&f, a, b] { f(a, b); });
  }
  for (auto& t : ts) t.join();
}

}  // namespace

extern "C" {

int ref_cddt_create(const uint8_t* grid, int w, int h, double res, int K, double max_range,
                    int prune, void** out) {
  *out = nullptr;
  try {
    OccupancyGrid g = make_grid(grid, w, h, res);
    RangeMethodConfig cfg;
    cfg.max_range = max_range;
    cfg.theta_disc = K;
    Cddt c(g, cfg);
    if (prune) c.prune();
    *out = new RefCddt(std::move(c));
    return RS_OK;
  } catch (const std::invalid_argument&) {
    return RS_EINVAL;
  } catch (...) {
    return RS_EOTHER;
  }
}

void ref_cddt_destroy(void* h) { delete static_cast<RefCddt*>(h); }

int ref_cddt_prune(void* h) {
  static_cast<RefCddt*>(h)->c.prune();
  return RS_OK;
}

// w, h, K, S, rows, zero_points, pruned, memory_bytes
void ref_cddt_info(void* hp, int64_t* out) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  out[0] = r.c.grid().width();
  out[1] = r.c.grid().height();
  out[2] = r.c.theta_disc();
  out[3] = r.c.slice_count();
  out[4] = int64_t(r.row_base.back());
  out[5] = int64_t(r.c.zero_point_count());
  out[6] = r.c.pruned();
  out[7] = int64_t(r.c.memory_bytes());
}

double ref_cddt_max_range(void* hp) { return static_cast<RefCddt*>(hp)->c.max_range(); }

// Concatenation of bin(s, r).values() in (slice, row) order, plus membership
// and the slice projections.
void ref_cddt_export(void* hp, uint64_t* row_off, float* zp, uint8_t* member, double* yoff,
                     int32_t* nbins) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  uint64_t off = 0;
  size_t g = 0;
  for (int s = 0; s < r.c.slice_count(); s++) {
    if (yoff) yoff[s] = r.c.slice(s).y_offset;
    if (nbins) nbins[s] = r.c.slice(s).bin_count;
    for (int row = 0; row < r.c.slice(s).bin_count; row++, g++) {
      std::vector<float> v = r.c.bin(s, row).values();
      if (row_off) row_off[g] = off;
      if (zp && !v.empty()) std::memcpy(zp + off, v.data(), v.size() * sizeof(float));
      off += v.size();
    }
  }
  if (row_off) row_off[g] = off;
  if (member) {
    const int w = r.c.grid().width(), h = r.c.grid().height();
    for (int y = 0; y < h; y++)
      for (int x = 0; x < w; x++) member[size_t(y) * w + x] = r.c.membership(x, y) ? 1 : 0;
  }
}

void ref_cddt_grid(void* hp, uint8_t* out) {
  const OccupancyGrid& g = static_cast<RefCddt*>(hp)->c.grid();
  for (int y = 0; y < g.height(); y++)
    for (int x = 0; x < g.width(); x++) out[size_t(y) * g.width() + x] = g.at(x, y) ? 1 : 0;
}

// Cddt::cast over f32 queries widened to double (RayQuery normalises theta).
// res_row/res_idx (optional) come from directional_cast with a MarkSink.
void ref_cast_batch(void* hp, const float* qx, const float* qy, const float* qt, size_t n,
                    double* out, int64_t* res_row, int32_t* res_idx, int nthreads) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  parallel_for(n, nthreads, [&](size_t a, size_t b) {
    for (size_t i = a; i < b; i++) {
      RayQuery q(double(qx[i]), double(qy[i]), double(qt[i]));
      out[i] = r.c.cast(q);
      if (res_row || res_idx) {
        LastMark m;
        r.c.directional_cast(q.x, q.y, direction_index(q.theta, r.c.theta_disc()), &m);
        int64_t rr = m.slice < 0 ? -1 : int64_t(r.row_base[m.slice] + size_t(m.row));
        if (res_row) res_row[i] = rr;
        if (res_idx) res_idx[i] = m.slice < 0 ? -1 : int32_t(m.index);
      }
    }
  });
}

// Cddt::directional_cast at explicit (x, y, a) states (f64).
void ref_directional_batch(void* hp, const double* x, const double* y, const int32_t* a, size_t n,
                           double* out) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  for (size_t i = 0; i < n; i++) out[i] = r.c.directional_cast(x[i], y[i], a[i], nullptr);
}

void ref_cast_pair_batch(void* hp, const double* x, const double* y, const double* t, size_t n,
                         double* fwd, double* bwd) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  for (size_t i = 0; i < n; i++) {
    auto p = r.c.cast_pair(RayQuery(x[i], y[i], t[i]));
    fwd[i] = p.first;
    bwd[i] = p.second;
  }
}

int ref_set_occupancy(void* hp, int x, int y, int occ) {
  try {
    static_cast<RefCddt*>(hp)->c.set_occupancy(x, y, occ != 0);
    return RS_OK;
  } catch (const std::logic_error& e) {
    if (dynamic_cast<const std::out_of_range*>(&e)) return RS_ERANGE;
    return RS_ELOGIC;
  } catch (...) {
    return RS_EOTHER;
  }
}

// A batch of Cddt::set_occupancy calls (proj/src/cddt.cpp:332-377), the
// reference's per-cell API in order, timed on the calling thread (steady
// clock); stops at the first failing edit. Returns the seconds taken.
double ref_set_occupancy_timed(void* hp, const int32_t* xy, const uint8_t* occ, size_t n,
                               int* status) {
  Cddt& c = static_cast<RefCddt*>(hp)->c;
  *status = RS_OK;
  const auto t0 = std::chrono::steady_clock::now();
  try {
    for (size_t k = 0; k < n; k++) c.set_occupancy(xy[2 * k], xy[2 * k + 1], occ[k] != 0);
  } catch (const std::logic_error& e) {
    *status = dynamic_cast<const std::out_of_range*>(&e) ? RS_ERANGE : RS_ELOGIC;
  } catch (...) {
    *status = RS_EOTHER;
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// serialize_cddt (proj/src/cddt.cpp:458-500); returns the byte size, copies
// when cap is large enough.
size_t ref_serialize(void* hp, uint8_t* buf, size_t cap) {
  std::vector<uint8_t> b = serialize_cddt(static_cast<RefCddt*>(hp)->c);
  if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
  return b.size();
}

int ref_deserialize(const uint8_t* buf, size_t n, void** out) {
  *out = nullptr;
  try {
    std::vector<uint8_t> b(buf, buf + n);
    *out = new RefCddt(deserialize_cddt(b));
    return RS_OK;
  } catch (const ParseError&) {
    return RS_EPARSE;
  } catch (...) {
    return RS_EOTHER;
  }
}

// p = {w_hit, w_short, w_max, w_rand, sigma_hit, lambda_short, z_max}
static BeamModelParams beam_params(const double* p) {
  BeamModelParams b;
  b.w_hit = p[0];
  b.w_short = p[1];
  b.w_max = p[2];
  b.w_rand = p[3];
  b.sigma_hit = p[4];
  b.lambda_short = p[5];
  b.z_max = p[6];
  return b;
}

double ref_beam_likelihood(const double* p, double e, double m) {
  try {
    return beam_likelihood(beam_params(p), e, m);
  } catch (...) {
    return -1.0;
  }
}

// sensor_update (proj/src/mcl.cpp:58-120) on particles given as SoA doubles;
// returns 1 when weights were degenerate (the reference's false), 0 otherwise.
int ref_sensor_update(void* hp, const double* px, const double* py, const double* pt, long n,
                      const double* scan, int nb, double fov, const double* p, double* weight,
                      int paired) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  CddtView view(r.c, paired != 0);
  std::vector<Particle> ps(static_cast<size_t>(n));
  for (long i = 0; i < n; i++) ps[i] = Particle{px[i], py[i], pt[i], 1.0 / double(n)};
  ScanSpec spec;
  spec.beam_count = nb;
  spec.fov = fov;
  std::vector<double> sc(scan, scan + nb);
  bool ok = sensor_update(ps, view, sc, spec, beam_params(p));
  for (long i = 0; i < n; i++) weight[i] = ps[i].weight;
  return ok ? 0 : 1;
}

// oracle_cast (proj/src/raycast.cpp:9-16) and lut_build (:62-87) on the
// structure's grid and max_range.
void ref_oracle_batch(void* hp, const double* x, const double* y, const double* t, size_t n,
                      double* out) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  for (size_t i = 0; i < n; i++)
    out[i] = oracle_cast(r.c.grid(), RayQuery(x[i], y[i], t[i]), r.c.max_range());
}
int ref_lut_build(void* hp, int theta_disc, uint16_t* out) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  try {
    RangeMethodConfig cfg;
    cfg.max_range = r.c.max_range();
    cfg.theta_disc = theta_disc;
    LookupTable lut = lut_build(r.c.grid(), cfg, size_t(1) << 34);
    std::memcpy(out, lut.entries.data(), lut.entries.size() * sizeof(uint16_t));
    return RS_OK;
  } catch (...) {
    return RS_EOTHER;
  }
}

// run_random_benchmark / run_grid_benchmark (proj/src/bench.cpp:153-210) over
// the Cddt: out = {queries, checksum}; map_content_id into id (17 bytes).
void ref_bench(void* hp, int random_mode, size_t n, uint64_t seed, int stride, double* out,
               char* id) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  CddtView view(r.c, true);
  RangeMethodConfig cfg;
  cfg.max_range = r.c.max_range();
  cfg.theta_disc = r.c.theta_disc();
  BenchReport rep = random_mode ? run_random_benchmark(view, r.c.grid(), cfg, n, seed)
                                : run_grid_benchmark(view, r.c.grid(), cfg, stride);
  out[0] = double(rep.queries);
  out[1] = rep.checksum;
  out[2] = rep.total_seconds;  // summed per-batch thread cpu time (bench.cpp:52-121)
  std::strncpy(id, rep.map_id.c_str(), 17);
}

// Cddt::cast over f32 queries on the calling thread, timed like the
// reference's own benchmark (run_batches, proj/src/bench.cpp:52-121): thread
// cpu time, which does not advance while the core is taken away.
void ref_cast_batch_cpu1(void* hp, const float* qx, const float* qy, const float* qt, size_t n,
                         double* out, double* cpu_seconds) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  timespec a{}, b{};
  clock_gettime(CLOCK_THREAD_CPUTIME_ID, &a);
  for (size_t i = 0; i < n; i++) out[i] = r.c.cast(RayQuery(double(qx[i]), double(qy[i]), double(qt[i])));
  clock_gettime(CLOCK_THREAD_CPUTIME_ID, &b);
  *cpu_seconds = double(b.tv_sec - a.tv_sec) + 1e-9 * double(b.tv_nsec - a.tv_nsec);
}

// The reference's own particle filter (rangelib::Mcl, proj/src/mcl.cpp:156-201)
// over a CddtMethod-equivalent view (paired casts on): init_gaussian, then
// `iters` steps with odometry odo[3k..3k+2] and scan scans[k*nb..]; per step
// its MclStepResult.seconds and estimate. noise = MotionNoise fields, p =
// BeamModelParams fields. The reference's sensor model is the analytic
// beam_likelihood (it has no table path).
int ref_mcl_run(void* hp, int n, uint64_t seed, double x0, double y0, double t0, double sxy,
                double sth, const double* noise, const double* p, int nb, double fov, int iters,
                const double* odo, const double* scans, double* seconds, double* est) {
  const RefCddt& r = *static_cast<RefCddt*>(hp);
  try {
    CddtView view(r.c, true);
    MclConfig cfg;
    cfg.particle_count = n;
    cfg.seed = seed;
    cfg.scan.beam_count = nb;
    cfg.scan.fov = fov;
    cfg.motion.trans_per_trans = noise[0];
    cfg.motion.trans_per_rot = noise[1];
    cfg.motion.rot_per_rot = noise[2];
    cfg.motion.rot_per_trans = noise[3];
    cfg.beam = beam_params(p);
    Mcl mcl(view, cfg);
    mcl.init_gaussian(x0, y0, t0, sxy, sth);
    for (int k = 0; k < iters; k++) {
      std::vector<double> sc(scans + size_t(k) * nb, scans + size_t(k + 1) * nb);
      MclStepResult res = mcl.step(odo[3 * k], odo[3 * k + 1], odo[3 * k + 2], sc);
      seconds[k] = res.seconds;
      est[3 * k] = res.estimate.x;
      est[3 * k + 1] = res.estimate.y;
      est[3 * k + 2] = res.estimate.theta;
    }
    return RS_OK;
  } catch (...) {
    return RS_EOTHER;
  }
}

// Ray marching baseline (make_method(ray_march), proj/src/methods.cpp:55-72).
void* ref_rm_create(const uint8_t* grid, int w, int h, double max_range) {
  try {
    RangeMethodConfig cfg;
    cfg.max_range = max_range;
    return make_method(MethodKind::ray_march, make_grid(grid, w, h, 0.05), cfg).release();
  } catch (...) {
    return nullptr;
  }
}
void ref_rm_destroy(void* m) { delete static_cast<RangeMethod*>(m); }
void ref_rm_cast_batch(void* mp, const float* qx, const float* qy, const float* qt, size_t n,
                       double* out, int nthreads) {
  const RangeMethod& m = *static_cast<RangeMethod*>(mp);
  parallel_for(n, nthreads, [&](size_t a, size_t b) {
    for (size_t i = a; i < b; i++) out[i] = m.cast(RayQuery(double(qx[i]), double(qy[i]), double(qt[i])));
  });
}

}  // extern "C"
