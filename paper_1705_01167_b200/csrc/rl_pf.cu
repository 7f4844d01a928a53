// Particle-filter step on the GPU: motion_update, weight normalisation,
// Mcl::estimate and resample_low_variance (proj/src/mcl.cpp:42-56, 108-142,
// 176-201), plus the single-GPU fused Mcl::step.
//
// Randomness is counter-based (Philox4x32-10): particle i's motion noise at
// iteration k is a pure function of (seed, i, k), so sharding particles over
// GPUs does not change any draw. The reference's std::mt19937_64 +
// std::normal_distribution stream is implementation-defined and cannot be
// reproduced bit-for-bit; the restatement in oracle/cddt_oracle.c uses the
// same Philox + Box-Muller and pins this path instead.
//
// Reductions are deterministic: per-block partials in a fixed-order second
// pass (no floating-point atomics), and the cumulative weights come from a
// CUB scan whose association depends only on n.
#include <cub/cub.cuh>

#include <cmath>

#include "rl_common.cuh"

namespace rl {

int sensor_logw_launch(rl_cddt* c, const double* px, const double* py, const double* pt,
                       size_t n, const double* scan, int nb, double fov,
                       const rl_beam_params_t* params, const float* table, int zdim,
                       double inv_res, double* logw, cudaStream_t st);

// Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0, k1).
struct U4 {
  uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// two uniforms in [0, 1) with 53 random bits each
__device__ __forceinline__ void philox_uniform2(uint64_t seed, uint32_t i, uint32_t draw,
                                                uint64_t iter, double& u0, double& u1) {
  const U4 r = philox4x32_10(U4{i, draw, uint32_t(iter), uint32_t(iter >> 32)}, uint32_t(seed),
                             uint32_t(seed >> 32));
  const uint64_t a = (uint64_t(r.y) << 32) | r.x, b = (uint64_t(r.w) << 32) | r.z;
  u0 = double(a >> 11) * 0x1.0p-53;
  u1 = double(b >> 11) * 0x1.0p-53;
}

constexpr uint32_t kResampleStream = 0xFFFFFFFFu;

__global__ void k_motion(double* __restrict__ x, double* __restrict__ y, double* __restrict__ t,
                         size_t n, uint64_t off, double dx, double dy, double dth, double st,
                         double sr, uint64_t seed, uint64_t iter) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const uint32_t gi = uint32_t(off + i);
    double a0, a1, b0, b1;
    philox_uniform2(seed, gi, 0, iter, a0, a1);
    philox_uniform2(seed, gi, 1, iter, b0, b1);
    // Box-Muller on (0, 1] x [0, 1)
    const double ra = sqrt(-2.0 * log(1.0 - a0)), rb = sqrt(-2.0 * log(1.0 - b0));
    double sa, ca, sb, cb;
    sincos(kTwoPi * a1, &sa, &ca);
    sincos(kTwoPi * b1, &sb, &cb);
    const double n0 = ra * ca, n1 = ra * sa, n2 = rb * cb;
    (void)sb;
    // motion_update (mcl.cpp:49-55)
    const double rdx = dx + st * n0, rdy = dy + st * n1, rdt = dth + sr * n2;
    double s, c;
    sincos(t[i], &s, &c);
    x[i] += rdx * c - rdy * s;
    y[i] += rdx * s + rdy * c;
    t[i] = normalize_angle_2pi(t[i] + rdt);
  }
}

// per-block partial moments, then a single-block fixed-order sum
constexpr int kMomentBlock = 256;
__global__ void __launch_bounds__(kMomentBlock) k_weights(
    const double* __restrict__ logw, const double* __restrict__ gmax,
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ t,
    size_t n, double* __restrict__ w, double* __restrict__ partial) {
  const double m = *gmax;
  double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double e = exp(logw[i] - m);
    w[i] = e;
    double s, c;
    sincos(t[i], &s, &c);
    acc[0] += e;
    acc[1] += e * x[i];
    acc[2] += e * y[i];
    acc[3] += e * c;
    acc[4] += e * s;
    acc[5] += 1.0;
    acc[6] += x[i];
    acc[7] += y[i];
    acc[8] += c;
    acc[9] += s;
  }
  typedef cub::BlockReduce<double, kMomentBlock> BR;
  __shared__ typename BR::TempStorage tmp;
#pragma unroll
  for (int k = 0; k < 10; k++) {
    const double v = BR(tmp).Sum(acc[k]);
    if (threadIdx.x == 0) partial[blockIdx.x * 10 + k] = v;
    __syncthreads();
  }
}

// one warp per moment: lane-strided partial sums, then a fixed shuffle tree
// (deterministic for a given block count)
__global__ void k_sum_partials(const double* __restrict__ partial, int nblk,
                               double* __restrict__ moments) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= 10) return;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += partial[b * 10 + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) moments[k] = s;
}

__global__ void k_normalize(double* __restrict__ w, size_t n, const double* __restrict__ moments,
                            uint64_t n_total, int32_t* __restrict__ degenerate) {
  const double s = moments[0];
  const bool bad = !(s > 0.0) || !isfinite(s);  // mcl.cpp:114-117
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    w[i] = bad ? 1.0 / double(n_total) : w[i] / s;
  if (degenerate && blockIdx.x == 0 && threadIdx.x == 0) *degenerate = bad ? 1 : 0;
}

// slot m takes the first particle i with cdf[i] >= r + m/n, capped at n-1
// (the sequential comb of mcl.cpp:130-140)
__global__ void k_comb(const double* __restrict__ cdf, const double* __restrict__ x,
                       const double* __restrict__ y, const double* __restrict__ t, size_t n,
                       size_t out_begin, size_t out_count, double* __restrict__ ox,
                       double* __restrict__ oy, double* __restrict__ ot, double* __restrict__ ow,
                       uint64_t seed, uint64_t iter) {
  double u, unused;
  philox_uniform2(seed, kResampleStream, kResampleStream, iter, u, unused);
  const double r = (1.0 / double(n)) * u;  // uniform_real_distribution(0, 1/n)
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < out_count;
       k += size_t(gridDim.x) * blockDim.x) {
    const size_t m = out_begin + k;
    const double target = r + double(m) / double(n);
    size_t lo = 0, len = n;
    while (len > 0) {
      const size_t half = len >> 1, mid = lo + half;
      if (cdf[mid] < target) {
        lo = mid + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    const size_t i = lo < n ? lo : n - 1;
    ox[k] = x[i];
    oy[k] = y[i];
    ot[k] = t[i];
    ow[k] = 1.0 / double(n);
  }
}

static int blocks(size_t n, int threads = 256, int per_sm = 8) {
  size_t b = (n + threads - 1) / threads;
  return int(std::max<size_t>(1, std::min(b, size_t(sm_count()) * per_sm)));
}

// grows c->ws to at least `need` bytes
static int workspace(rl_cddt* c, size_t need, uint8_t** p) {
  if (c->ws.n < need) RL_TRY(c->ws.alloc(need));
  *p = c->ws.p;
  return RL_OK;
}

int weights_launch(const double* logw, const double* gmax, const double* x, const double* y,
                   const double* t, size_t n, double* w, double* moments, double* partial,
                   cudaStream_t st) {
  const int nb = blocks(n, kMomentBlock, 2);
  k_weights<<<nb, kMomentBlock, 0, st>>>(logw, gmax, x, y, t, n, w, partial);
  k_sum_partials<<<1, 320, 0, st>>>(partial, nb, moments);
  RL_CK(cudaGetLastError());
  return RL_OK;
}

}  // namespace rl

using namespace rl;

extern "C" {

int rl_motion_update(double* x, double* y, double* theta, size_t n, uint64_t index_offset,
                     double dx, double dy, double dtheta, const rl_motion_noise_t* noise,
                     uint64_t seed, uint64_t iteration, void* stream) {
  if (!noise || (n && (!x || !y || !theta))) return RL_EINVAL;
  if (index_offset + n > (1ull << 32)) {
    set_error("motion_update: particle index exceeds the 32-bit RNG counter");
    return RL_EINVAL;
  }
  if (n == 0) return RL_OK;
  const double trans = std::hypot(dx, dy);  // mcl.cpp:44-48
  const double st = std::max(noise->trans_per_trans * trans + noise->trans_per_rot * std::fabs(dtheta),
                             1e-12);
  const double sr = std::max(noise->rot_per_rot * std::fabs(dtheta) + noise->rot_per_trans * trans,
                             1e-12);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_motion<<<blocks(n), 256, 0, s>>>(x, y, theta, n, index_offset, dx, dy, dtheta, st, sr, seed,
                                    iteration);
  RL_CK(cudaGetLastError());
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_pf_max(const double* logw, size_t n, double* out, void* stream) {
  if (!logw || !out || n == 0) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  size_t bytes = 0;
  cub::DeviceReduce::Max(nullptr, bytes, logw, out, int(n), s);
  DevBuf<uint8_t> tmp;
  RL_TRY(tmp.alloc(bytes));
  RL_CK(cub::DeviceReduce::Max(tmp.p, bytes, logw, out, int(n), s));
  RL_CK(cudaStreamSynchronize(s));  // tmp is freed on return
  return RL_OK;
}

int rl_pf_weights(const double* logw, const double* gmax, const double* x, const double* y,
                  const double* theta, size_t n, double* w, double* moments, void* stream) {
  if (!logw || !gmax || !x || !y || !theta || !w || !moments) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevBuf<double> partial;
  RL_TRY(partial.alloc(size_t(blocks(n, kMomentBlock, 2)) * 10));
  if (n == 0) {
    RL_CK(cudaMemsetAsync(moments, 0, 10 * sizeof(double), s));
  } else {
    RL_TRY(weights_launch(logw, gmax, x, y, theta, n, w, moments, partial.p, s));
  }
  RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_pf_normalize(double* w, size_t n, const double* moments, uint64_t n_total,
                    int32_t* degenerate, void* stream) {
  if (!moments || (n && !w) || n_total == 0) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_normalize<<<blocks(std::max<size_t>(n, 1)), 256, 0, s>>>(w, n, moments, n_total, degenerate);
  RL_CK(cudaGetLastError());
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_resample_low_variance(const double* x, const double* y, const double* theta,
                             const double* w, size_t n, size_t out_begin, size_t out_count,
                             double* ox, double* oy, double* otheta, double* ow, uint64_t seed,
                             uint64_t iteration, void* stream) {
  if (n == 0 || out_count == 0) return RL_OK;  // mcl.cpp:124
  if (!x || !y || !theta || !w || !ox || !oy || !otheta || !ow || out_begin + out_count > n)
    return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, w, (double*)nullptr, int(n), s);
  DevBuf<uint8_t> tmp;
  DevBuf<double> cdf;
  RL_TRY(tmp.alloc(bytes));
  RL_TRY(cdf.alloc(n));
  RL_CK(cub::DeviceScan::InclusiveSum(tmp.p, bytes, w, cdf.p, int(n), s));
  k_comb<<<blocks(out_count), 256, 0, s>>>(cdf.p, x, y, theta, n, out_begin, out_count, ox, oy,
                                          otheta, ow, seed, iteration);
  RL_CK(cudaGetLastError());
  RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_mcl_step(rl_cddt* c, double* x, double* y, double* theta, double* w, size_t n,
                double odo_dx, double odo_dy, double odo_dtheta, const double* scan,
                int32_t nbeams, double fov, const rl_motion_noise_t* noise,
                const rl_beam_params_t* params, const float* table, int32_t zdim, double inv_res,
                uint64_t seed, uint64_t iteration, double* estimate, void* stream) {
  if (!c || !noise || !scan || nbeams <= 0 || (n && (!x || !y || !theta || !w))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  cudaStream_t st = pick_stream(c, stream);
  // workspace: logw | w2 x y t (resample targets) | cdf | partials | moments | max | flag | cub
  size_t cub_bytes = 0, b2 = 0;
  cub::DeviceReduce::Max(nullptr, cub_bytes, (double*)nullptr, (double*)nullptr, int(n), st);
  cub::DeviceScan::InclusiveSum(nullptr, b2, (double*)nullptr, (double*)nullptr, int(n), st);
  cub_bytes = std::max(cub_bytes, b2);
  const int nbw = blocks(n, kMomentBlock, 2);
  const size_t need = 8 * n * 6 + 8 * size_t(nbw) * 10 + 8 * 16 + cub_bytes + 512;
  uint8_t* base = nullptr;
  RL_TRY(workspace(c, need, &base));
  double* logw = reinterpret_cast<double*>(base);
  double* nx = logw + n;
  double* ny = nx + n;
  double* nt = ny + n;
  double* nw = nt + n;
  double* cdf = nw + n;
  double* partial = cdf + n;
  double* moments = partial + size_t(nbw) * 10;
  double* gmax = moments + 10;
  int32_t* flag = reinterpret_cast<int32_t*>(gmax + 2);
  void* tmp = reinterpret_cast<uint8_t*>(gmax + 4);

  RL_TRY(rl_motion_update(x, y, theta, n, 0, odo_dx, odo_dy, odo_dtheta, noise, seed, iteration,
                          st));
  RL_TRY(sensor_logw_launch(c, x, y, theta, n, scan, nbeams, fov, params, table, zdim, inv_res,
                            logw, st));
  RL_CK(cub::DeviceReduce::Max(tmp, cub_bytes, logw, gmax, int(n), st));
  RL_TRY(weights_launch(logw, gmax, x, y, theta, n, w, moments, partial, st));
  k_normalize<<<blocks(n), 256, 0, st>>>(w, n, moments, n, flag);
  RL_CK(cub::DeviceScan::InclusiveSum(tmp, cub_bytes, w, cdf, int(n), st));
  k_comb<<<blocks(n), 256, 0, st>>>(cdf, x, y, theta, n, 0, n, nx, ny, nt, nw, seed, iteration);
  RL_CK(cudaGetLastError());
  RL_CK(cudaMemcpyAsync(x, nx, 8 * n, cudaMemcpyDeviceToDevice, st));
  RL_CK(cudaMemcpyAsync(y, ny, 8 * n, cudaMemcpyDeviceToDevice, st));
  RL_CK(cudaMemcpyAsync(theta, nt, 8 * n, cudaMemcpyDeviceToDevice, st));
  RL_CK(cudaMemcpyAsync(w, nw, 8 * n, cudaMemcpyDeviceToDevice, st));
  double mom[10];
  int32_t deg = 0;
  RL_CK(cudaMemcpyAsync(mom, moments, sizeof mom, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaMemcpyAsync(&deg, flag, sizeof deg, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
  if (estimate) {
    // Mcl::estimate (mcl.cpp:176-187) on the normalised weights: with
    // normalised w_i = e_i / S the sums are the e-moments divided by S; a
    // degenerate reset gives uniform weights 1/n.
    double sx, sy, sc, ss, sw;
    if (deg) {
      const double inv = 1.0 / double(n);
      sx = mom[6] * inv;
      sy = mom[7] * inv;
      sc = mom[8] * inv;
      ss = mom[9] * inv;
      sw = mom[5] * inv;
    } else {
      sx = mom[1] / mom[0];
      sy = mom[2] / mom[0];
      sc = mom[3] / mom[0];
      ss = mom[4] / mom[0];
      sw = 1.0;
    }
    if (!(sw > 0.0)) sw = 1.0;
    double th = std::fmod(std::atan2(ss, sc), kTwoPi);
    if (th < 0) th += kTwoPi;
    if (th >= kTwoPi) th = 0.0;
    estimate[0] = sx / sw;
    estimate[1] = sy / sw;
    estimate[2] = th;
  }
  return deg ? RL_EDEGENERATE : RL_OK;
}

}  // extern "C"
