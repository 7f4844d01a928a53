// Fused beam sensor model: sensor_update (proj/src/mcl.cpp:58-120) on the GPU.
//
// One CTA scores PB particles x nbeams beams: every (particle, beam) item is a
// CDDT cast (cddt_device.cuh) followed by the likelihood lookup, the per-beam
// log-likelihoods land in shared memory and one thread per particle sums them
// in beam order 0..nbeams-1 — the reference's summation order, so the FP64
// log-weight is reproducible. Normalisation (max-subtract, exp, sum, divide,
// degenerate reset, mcl.cpp:108-119) follows as a reduction.
#include <cooperative_groups.h>

#include <cmath>

#include "pf_device.cuh"
#include "rl_common.cuh"

namespace rl {

namespace cg = cooperative_groups;

// particles per CTA: 16 for large sets (config 4), 8 below kSmallSet so a
// few thousand particles still fill the GPU (config 2)
constexpr size_t kSmallSet = 16384;

struct BeamParams {
  double w_hit, w_short, w_max, w_rand, sigma_hit, lambda_short, z_max;
};

// beam_likelihood (mcl.cpp:11-40)
__device__ __forceinline__ double beam_likelihood(const BeamParams& p, double expected,
                                                  double measured) {
  const double zm = p.z_max;
  const double e = expected < 0.0 ? 0.0 : (zm < expected ? zm : expected);
  const double m = measured < 0.0 ? 0.0 : (zm < measured ? zm : measured);
  double hit = 0.0;
  if (p.w_hit > 0.0) {
    const double s = p.sigma_hit;
    const double inv_sqrt2 = 0.7071067811865476;
    double eta = 0.5 * (erf((zm - e) / s * inv_sqrt2) - erf((0.0 - e) / s * inv_sqrt2));
    if (eta > 1e-12) {
      double z = (m - e) / s;
      hit = exp(-0.5 * z * z) / (s * 2.5066282746310002) / eta;
    }
  }
  double shrt = 0.0;
  if (p.w_short > 0.0 && e > 0.0 && m <= e) {
    double denom = 1.0 - exp(-p.lambda_short * e);
    if (denom > 1e-12) shrt = p.lambda_short * exp(-p.lambda_short * m) / denom;
  }
  double mx = (m >= zm - 1.0) ? 1.0 : 0.0;
  double rnd = 1.0 / zm;
  return p.w_hit * hit + p.w_short * shrt + p.w_max * mx + p.w_rand * rnd;
}

__device__ __forceinline__ int table_index(double r, double inv_res, int zdim) {
  long i = iround(r * inv_res);
  if (i < 0) i = 0;
  if (i > zdim - 1) i = zdim - 1;
  return int(i);
}

// Per-item pieces of the sensor model.
__device__ __forceinline__ double beam_offset(int b, int nb, double fov) {
  return nb <= 1 ? 0.0 : -fov / 2.0 + fov * double(b) / double(nb - 1);  // mcl.hpp:42-51
}

__device__ __forceinline__ double item_loglike(double e, int b, const double* __restrict__ scan,
                                               const BeamParams& bp,
                                               const float* __restrict__ table, int mrow,
                                               int zdim, double inv_res) {
  double like;
  if (table)
    like = double(__ldg(table + size_t(unsigned(mrow)) + table_index(e, inv_res, zdim)));
  else
    like = beam_likelihood(bp, e, scan[b]);
  return log(like);
}

// MOTION: the CTA's particles first take their motion_update step (the fused
// Mcl::step, mcl.cpp:189-193) and write the moved poses back. gmax_key (may be
// null) receives the order-preserving atomic max of the log-weights.
// Resident CTAs per SM: 4 (64 registers, a few bytes of spill) for the large
// sets, where throughput decides (config 4); 3 (74 registers, no spill) for
// the small ones, where the slowest cast decides (config 2: -3.5 %).
#ifndef RL_SENSOR_MINB
#define RL_SENSOR_MINB 4
#endif
#ifndef RL_SENSOR_MINB_SMALL
#define RL_SENSOR_MINB_SMALL 3
#endif
template <bool MOTION, int kSensorParticlesPerCta>
__global__ void __launch_bounds__(256, kSensorParticlesPerCta < 16 ? RL_SENSOR_MINB_SMALL
                                                                   : RL_SENSOR_MINB)
    k_sensor_logw(
    CddtView c, double* __restrict__ px, double* __restrict__ py, double* __restrict__ pt,
    size_t n, const double* __restrict__ scan, int nb, double fov, BeamParams bp,
    const float* __restrict__ table, int zdim, double inv_res, double* __restrict__ logw,
    MotionArgs mot, unsigned long long* __restrict__ gmax_key) {
  extern __shared__ double ll[];  // [PB][nb] log-likelihoods | [nb] beam offsets | [nb] table rows
  double* boff = ll + kSensorParticlesPerCta * nb;
  int* mrow = reinterpret_cast<int*>(boff + nb);
  __shared__ double pose[3][kSensorParticlesPerCta];
  const size_t p0 = size_t(blockIdx.x) * kSensorParticlesPerCta;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    // ScanSpec::beam_offset (mcl.hpp:42-51)
    boff[b] = beam_offset(b, nb, fov);
    if (table) mrow[b] = table_index(scan[b], inv_res, zdim) * zdim;
  }
  if (threadIdx.x < kSensorParticlesPerCta) {
    const size_t i = p0 + threadIdx.x;
    if (i < n) {
      double x = px[i], y = py[i], t = pt[i];
      if (MOTION) {
        motion_one(mot, uint32_t(mot.index_offset + i), x, y, t);
        px[i] = x;
        py[i] = y;
        pt[i] = t;
      }
      pose[0][threadIdx.x] = x;
      pose[1][threadIdx.x] = y;
      pose[2][threadIdx.x] = t;
    }
  }
  __syncthreads();
  const int items = kSensorParticlesPerCta * nb;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int pl = it / nb, b = it % nb;
    if (p0 + pl >= n) continue;
    const double th = normalize_angle_2pi(pose[2][pl] + boff[b]);
    CastOut o;
    const double e = directional_cast(c, pose[0][pl], pose[1][pl], direction_index(th, c.K), o);
    ll[it] = item_loglike(e, b, scan, bp, table, mrow[b], zdim, inv_res);
  }
  __syncthreads();
  if (threadIdx.x < kSensorParticlesPerCta) {
    const size_t i = p0 + threadIdx.x;
    unsigned long long key = 0;
    if (i < n) {
      double lw = 0.0;
      const double* row = ll + threadIdx.x * nb;
      for (int b = 0; b < nb; b++) lw += row[b];  // mcl.cpp:102-103 order
      logw[i] = lw;
      key = order_key(lw);
    }
    if (gmax_key) {
#pragma unroll
      for (int o = kSensorParticlesPerCta / 2; o > 0; o >>= 1) {
        const unsigned long long k2 = __shfl_down_sync(
            unsigned((1ull << kSensorParticlesPerCta) - 1), key, o, kSensorParticlesPerCta);
        key = k2 > key ? k2 : key;
      }
      if (threadIdx.x == 0 && key) atomicMax(gmax_key, key);
    }
  }
}



// sensor_update's normalisation (mcl.cpp:104-119) after the log-weights: one
// cooperative launch. w = exp(logw - max) with the max from the atomic key,
// per-block sums in a fixed tree, every block sums the block sums in the same
// order, then w /= S (or 1/n and the degenerate flag when S is zero or not
// finite).
__global__ void __launch_bounds__(256) k_sensor_normalize(const double* __restrict__ logw,
                                                          const unsigned long long* __restrict__ key,
                                                          double* __restrict__ w, size_t n,
                                                          double* __restrict__ partial,
                                                          int* __restrict__ degenerate) {
  cg::grid_group grid = cg::this_grid();
  const double m = order_key_value(*key);
  double acc = 0.0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double e = exp(logw[i] - m);
    w[i] = e;
    acc += e;
  }
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int k = 0; k < 8; k++) b += red[k];
    partial[blockIdx.x] = b;
  }
  grid.sync();
  __shared__ double S_s;
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) v += __ldcg(partial + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) S_s = v;
  }
  __syncthreads();
  const double S = S_s;
  const bool bad = !(S > 0.0) || !isfinite(S);  // mcl.cpp:114
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    w[i] = bad ? 1.0 / double(n) : __ldcg(w + i) / S;
  if (blockIdx.x == 0 && threadIdx.x == 0) *degenerate = bad ? 1 : 0;
}


int sensor_logw_launch(rl_cddt* c, double* px, double* py, double* pt, size_t n,
                       const double* scan, int nb, double fov, const rl_beam_params_t* params,
                       const float* table, int zdim, double inv_res, double* logw,
                       const MotionArgs* mot, unsigned long long* gmax_key, cudaStream_t st) {
  BeamParams bp{};
  if (params)
    bp = BeamParams{params->w_hit,     params->w_short,      params->w_max, params->w_rand,
                    params->sigma_hit, params->lambda_short, params->z_max};
  const MotionArgs m = mot ? *mot : MotionArgs{};
  auto launch = [&](auto kernel, int pb) -> int {
    const int ctas = int((n + pb - 1) / pb);
    const size_t smem = sizeof(double) * (pb + 1) * nb + sizeof(int) * nb;
    if (smem > 48 * 1024)
      RL_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kernel<<<ctas, 256, smem, st>>>(c->view(), px, py, pt, n, scan, nb, fov, bp, table, zdim,
                                    inv_res, logw, m, gmax_key);
    return RL_OK;
  };
  if (n < kSmallSet) {
    RL_TRY(mot ? launch(k_sensor_logw<true, 8>, 8) : launch(k_sensor_logw<false, 8>, 8));
  } else {
    RL_TRY(mot ? launch(k_sensor_logw<true, 16>, 16) : launch(k_sensor_logw<false, 16>, 16));
  }
  RL_CK(cudaGetLastError());
  return RL_OK;
}

static int check_sensor_args(const rl_cddt* c, const double* px, const double* py,
                             const double* pt, size_t n, const double* scan, int32_t nbeams,
                             const rl_beam_params_t* params, const float* table, int32_t zdim,
                             double inv_res) {
  if (!c || nbeams <= 0 || (n && (!px || !py || !pt || !scan))) {
    set_error("scan length does not match beam count");  // mcl.cpp:61-62
    return RL_EINVAL;
  }
  if (!table && (!params || !(params->z_max > 0.0))) {
    set_error("beam model z_max must be positive");  // mcl.cpp:13
    return RL_EINVAL;
  }
  if (table && (zdim <= 0 || zdim > 32768 || !(inv_res > 0.0))) {
    set_error("likelihood table needs 0 < zdim <= 32768 and inv_res > 0");
    return RL_EINVAL;
  }
  return RL_OK;
}

}  // namespace rl

using namespace rl;

extern "C" {

int rl_sensor_logw(rl_cddt* c, const double* px, const double* py, const double* pt, size_t n,
                   const double* scan, int32_t nbeams, double fov, const rl_beam_params_t* params,
                   const float* table, int32_t zdim, double inv_res, double* logw, void* stream) {
  RL_TRY(check_sensor_args(c, px, py, pt, n, scan, nbeams, params, table, zdim, inv_res));
  if (!logw && n) return RL_EINVAL;
  if (n == 0) return RL_OK;
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  RL_TRY(sensor_logw_launch(c, const_cast<double*>(px), const_cast<double*>(py),
                            const_cast<double*>(pt), n, scan, nbeams, fov, params, table, zdim,
                            inv_res, logw, nullptr, nullptr, pick_stream(c, stream)));
  return finish(c, stream);
}

double rl_beam_likelihood(const rl_beam_params_t* p, double expected, double measured) {
  // host restatement of beam_likelihood (mcl.cpp:11-40) for table building
  const double zm = p->z_max;
  if (!(zm > 0.0)) return NAN;
  const double e = expected < 0.0 ? 0.0 : (zm < expected ? zm : expected);
  const double m = measured < 0.0 ? 0.0 : (zm < measured ? zm : measured);
  double hit = 0.0;
  if (p->w_hit > 0.0) {
    const double s = p->sigma_hit;
    const double inv_sqrt2 = 0.7071067811865476;
    double eta =
        0.5 * (std::erf((zm - e) / s * inv_sqrt2) - std::erf((0.0 - e) / s * inv_sqrt2));
    if (eta > 1e-12) {
      double z = (m - e) / s;
      hit = std::exp(-0.5 * z * z) / (s * 2.5066282746310002) / eta;
    }
  }
  double shrt = 0.0;
  if (p->w_short > 0.0 && e > 0.0 && m <= e) {
    double denom = 1.0 - std::exp(-p->lambda_short * e);
    if (denom > 1e-12) shrt = p->lambda_short * std::exp(-p->lambda_short * m) / denom;
  }
  double mx = (m >= zm - 1.0) ? 1.0 : 0.0;
  double rnd = 1.0 / zm;
  return p->w_hit * hit + p->w_short * shrt + p->w_max * mx + p->w_rand * rnd;
}

int rl_beam_table(const rl_beam_params_t* p, int32_t zdim, double inv_res, float* table) {
  if (!p || !table || zdim <= 0 || !(inv_res > 0.0)) return RL_EINVAL;
  if (!(p->z_max > 0.0)) {
    set_error("beam model z_max must be positive");  // mcl.cpp:13
    return RL_EINVAL;
  }
  for (int m = 0; m < zdim; m++)
    for (int e = 0; e < zdim; e++)
      table[size_t(m) * zdim + e] =
          float(rl_beam_likelihood(p, double(e) / inv_res, double(m) / inv_res));
  return RL_OK;
}

}  // extern "C"

// sensor_update: synchronous (degenerate_dev == nullptr: the flag is read back
// and returned as RL_EDEGENERATE) or asynchronous (the flag is written to
// degenerate_dev on the device and nothing waits).
static int sensor_update_impl(rl_cddt* c, const double* px, const double* py, const double* pt,
                              size_t n, const double* scan, int32_t nbeams, double fov,
                              const rl_beam_params_t* params, const float* table, int32_t zdim,
                              double inv_res, double* logw, double* weight,
                              int32_t* degenerate_dev, void* stream) {
  RL_TRY(check_sensor_args(c, px, py, pt, n, scan, nbeams, params, table, zdim, inv_res));
  if (n == 0) {
    if (degenerate_dev)
      RL_CK(cudaMemsetAsync(degenerate_dev, 0, sizeof(int32_t), pick_stream(c, stream)));
    return RL_OK;
  }
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  cudaStream_t st = pick_stream(c, stream);
  static const int coop = [] {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sensor_normalize, 256, 0);
    return per_sm;
  }();
  const int nblk = int(std::max<size_t>(
      1, std::min((n + 255) / 256, size_t(sm_count()) * size_t(std::min(coop, 2)))));
  // workspace: control {max key, flag} | logw (if not given) | w (if not given) | partials
  const size_t need = 64 + 16 * n + 8 * size_t(nblk);
  if (c->ws.n < need) RL_TRY(c->ws.alloc(need));
  uint8_t* base = c->ws.p;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(base);
  int* d_flag = degenerate_dev ? degenerate_dev : reinterpret_cast<int*>(base + 8);
  double* d_logw = logw ? logw : reinterpret_cast<double*>(base + 64);
  double* d_w = weight ? weight : reinterpret_cast<double*>(base + 64 + 8 * n);
  double* partial = reinterpret_cast<double*>(base + 64 + 16 * n);
  RL_CK(cudaMemsetAsync(key, 0, 8, st));
  RL_TRY(sensor_logw_launch(c, const_cast<double*>(px), const_cast<double*>(py),
                            const_cast<double*>(pt), n, scan, nbeams, fov, params, table, zdim,
                            inv_res, d_logw, nullptr, key, st));
  if (coop < 1) {
    set_error("sensor_update: normalisation kernel cannot be co-resident");
    return RL_ECUDA;
  }
  size_t nn = n;
  void* args[] = {&d_logw, &key, &d_w, &nn, &partial, &d_flag};
  RL_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_sensor_normalize), dim3(nblk),
                                    dim3(256), args, 0, st));
  if (degenerate_dev) return RL_OK;
  uint32_t* hs = nullptr;
  RL_TRY(host_small(c, &hs));
  RL_CK(cudaMemcpyAsync(hs, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
  return hs[0] ? RL_EDEGENERATE : RL_OK;
}

extern "C" {

int rl_sensor_update(rl_cddt* c, const double* px, const double* py, const double* pt, size_t n,
                     const double* scan, int32_t nbeams, double fov,
                     const rl_beam_params_t* params, const float* table, int32_t zdim,
                     double inv_res, double* logw, double* weight, void* stream) {
  return sensor_update_impl(c, px, py, pt, n, scan, nbeams, fov, params, table, zdim, inv_res,
                            logw, weight, nullptr, stream);
}

int rl_sensor_update_async(rl_cddt* c, const double* px, const double* py, const double* pt,
                           size_t n, const double* scan, int32_t nbeams, double fov,
                           const rl_beam_params_t* params, const float* table, int32_t zdim,
                           double inv_res, double* logw, double* weight, int32_t* degenerate,
                           void* stream) {
  if (!degenerate || !stream) {
    set_error("rl_sensor_update_async needs a device flag and a stream");
    return RL_EINVAL;
  }
  return sensor_update_impl(c, px, py, pt, n, scan, nbeams, fov, params, table, zdim, inv_res,
                            logw, weight, degenerate, stream);
}

}  // extern "C"
