// The reference's exact cast and lookup-table build on the GPU (SURVEY.md §8
// row f2): oracle_cast (proj/src/raycast.cpp:9-16) walks every cell along a
// continuous direction to the first occupied one, and lut_build (:62-87)
// fills the dense [theta][y][x] table of rounded oracle distances from every
// cell centre. Both reuse the CDDT handle's grid (query bits) and the exact
// walker of cddt_device.cuh.
//
// Directions: oracle_cast uses std::cos/std::sin of the query angle. For
// bit parity the caller passes glibc values (cos_t/sin_t); with NULL the
// device computes them with sincos() (within 1 ulp of glibc). lut_build's K
// lattice directions are always host glibc values.
#include <algorithm>
#include <cmath>
#include <vector>

#include "pf_device.cuh"
#include "rl_common.cuh"

namespace rl {

// oracle_cast: origin checks, then RayWalker::scan_to(max_range) from t = 0.
__device__ __forceinline__ double exact_cast(const CddtView& c, double x, double y, double cs,
                                             double sn) {
  const int cx = (int)floor(x), cy = (int)floor(y);
  if (!in_bounds(c, cx, cy)) return c.max_range;
  if (occupied(c, cx, cy)) return 0.0;
  Walker<false> wk;
  // reciprocals for div_rn: IEEE division, exact
  const double4 dir = make_double4(cs, sn, cs != 0.0 ? 1.0 / cs : 0.0, sn != 0.0 ? 1.0 / sn : 0.0);
  wk.init_at(x, y, dir, 0.0);
  const double r = wk.scan_to(c, c.max_range);
  return r >= 0.0 ? r : c.max_range;
}

__global__ void k_exact(CddtView c, const double* __restrict__ x, const double* __restrict__ y,
                        const double* __restrict__ theta, const double* __restrict__ cs,
                        const double* __restrict__ sn, double* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    double cv, sv;
    if (cs) {
      cv = cs[i];
      sv = sn[i];
    } else {
      sincos(normalize_angle_2pi(theta[i]), &sv, &cv);  // RayQuery normalises first
    }
    out[i] = exact_cast(c, x[i], y[i], cv, sv);
  }
}

// lut_build: entry (x, y, i) = clamp(llround(oracle_cast(x+0.5, y+0.5, theta_i)), 0, 65535)
__global__ void k_lut(CddtView c, const double2* __restrict__ dirs, int K,
                      uint16_t* __restrict__ entries) {
  const uint64_t total = uint64_t(K) * c.h * c.w;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int x = int(i % c.w);
    const uint64_t r = i / c.w;
    const int y = int(r % c.h), ti = int(r / c.h);
    const double2 d = dirs[ti];
    const double v = exact_cast(c, double(x) + 0.5, double(y) + 0.5, d.x, d.y);
    long long q = llround(v);
    q = q < 0 ? 0 : (q > 65535 ? 65535 : q);
    entries[i] = uint16_t(q);
  }
}

// simulate_scan (mcl.cpp:144-154), one thread per (pose, beam)
__global__ void k_scans(CddtView c, const double* __restrict__ px, const double* __restrict__ py,
                        const double* __restrict__ pt, uint64_t n, int nb, double fov,
                        double sigma, uint64_t seed, uint64_t stream_id,
                        const double* __restrict__ cs, const double* __restrict__ sn,
                        double* __restrict__ scan) {
  const uint64_t total = n * uint64_t(nb);
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = k / uint64_t(nb);
    const int b = int(k - i * uint64_t(nb));
    double cv, sv;
    if (cs) {
      cv = cs[k];
      sv = sn[k];
    } else {
      // RayQuery(x, y, theta + beam_offset(b)) normalises the angle (raycast.hpp:47)
      const double off = nb <= 1 ? 0.0 : -fov / 2.0 + fov * double(b) / double(nb - 1);
      sincos(normalize_angle_2pi(pt[i] + off), &sv, &cv);
    }
    const double d = exact_cast(c, px[i], py[i], cv, sv);
    // N(0, sigma): Box-Muller on one Philox draw keyed by (pose, beam)
    double u0, u1;
    philox_uniform2(seed, uint32_t(k), uint32_t(k >> 32), stream_id, u0, u1);
    const double z = sqrt(-2.0 * log(1.0 - u0)) * cos(kTwoPi * u1);
    const double v = d + sigma * z;
    scan[k] = v < 0.0 ? 0.0 : (c.max_range < v ? c.max_range : v);  // std::clamp
  }
}

static int blocks(uint64_t n) {
  const uint64_t b = (n + 255) / 256, cap = uint64_t(sm_count()) * 8;
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace rl

using namespace rl;

extern "C" {

int rl_exact_cast_batch(rl_cddt* c, const double* x, const double* y, const double* theta,
                        const double* cos_t, const double* sin_t, double* out, size_t n,
                        void* stream) {
  if (!c || (n && (!x || !y || !out || (!theta && !cos_t) || (!cos_t != !sin_t))))
    return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  k_exact<<<blocks(n), 256, 0, pick_stream(c, stream)>>>(c->view(), x, y, theta, cos_t, sin_t,
                                                         out, n);
  return finish(c, stream);
}

int rl_simulate_scans(rl_cddt* c, const double* x, const double* y, const double* theta,
                      size_t n, int32_t nbeams, double fov, double max_range,
                      double noise_sigma, uint64_t seed, uint64_t stream_id,
                      const double* cos_t, const double* sin_t, double* scan, void* stream) {
  if (!c || nbeams <= 0 || !(max_range >= 0.0) || (!cos_t != !sin_t) ||
      (n && (!x || !y || !scan || (!theta && !cos_t)))) {
    set_error("simulate_scan: invalid arguments");
    return RL_EINVAL;
  }
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  CddtView v = c->view();
  v.max_range = max_range;  // oracle_cast's own max_range argument
  const uint64_t total = uint64_t(n) * uint64_t(nbeams);
  k_scans<<<blocks(total), 256, 0, pick_stream(c, stream)>>>(
      v, x, y, theta, n, nbeams, fov, std::max(noise_sigma, 1e-12), seed, stream_id, cos_t,
      sin_t, scan);
  return finish(c, stream);
}

int rl_lut_build(rl_cddt* c, int32_t theta_disc, uint16_t* entries, void* stream) {
  if (!c || !entries || theta_disc < 4 || theta_disc % 2 != 0) {
    set_error("theta_disc must be even and >= 4");
    return RL_EINVAL;
  }
  DeviceGuard guard(c->dev);
  cudaStream_t st = pick_stream(c, stream);
  // theta_i = i * 2pi / K; RayQuery leaves it unchanged (< 2pi); glibc cos/sin
  std::vector<double2> dirs(theta_disc);
  for (int i = 0; i < theta_disc; i++) {
    const double t = double(i) * kTwoPi / double(theta_disc);
    dirs[i] = make_double2(std::cos(t), std::sin(t));
  }
  DevBuf<double2> d_dirs;
  RL_TRY(d_dirs.alloc(theta_disc));
  RL_CK(cudaMemcpyAsync(d_dirs.p, dirs.data(), sizeof(double2) * theta_disc,
                        cudaMemcpyHostToDevice, st));
  k_lut<<<blocks(uint64_t(theta_disc) * c->w * c->h), 256, 0, st>>>(c->view(), d_dirs.p,
                                                                    theta_disc, entries);
  RL_CK(cudaGetLastError());
  RL_CK(cudaStreamSynchronize(st));  // d_dirs is freed on return
  return RL_OK;
}

}  // extern "C"
