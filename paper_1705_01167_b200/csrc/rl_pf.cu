// Particle-filter step on the GPU: motion_update, weight normalisation,
// Mcl::estimate and resample_low_variance (proj/src/mcl.cpp:42-56, 108-142,
// 176-201), plus the single-GPU fused Mcl::step.
//
// Randomness is counter-based (Philox4x32-10, pf_device.cuh): particle i's
// motion noise at iteration k is a pure function of (seed, i, k), so sharding
// particles over GPUs does not change any draw. The reference's
// std::mt19937_64 + std::normal_distribution stream is implementation-defined
// and cannot be reproduced bit-for-bit; the restatement in
// oracle/cddt_oracle.c uses the same Philox + Box-Muller and pins this path
// instead.
//
// Reductions are deterministic (run to run and for a given n): per-block
// partials summed in fixed order by the last block to finish (no
// floating-point atomics), and the cumulative weights are a tiled scan —
// fixed-shape block scans plus a sequential pass over tile totals — so the
// comb sees the same cumulative sums on every run and on every rank.
//
// The fused step (rl_mcl_step) is two kernels:
//   k_sensor_logw<true>  motion + casts + log-likelihood sums + atomic max
//   k_pf_finish          one cooperative launch, phases split by grid syncs:
//                        exp(logw - max) and moments | w / S tile scans |
//                        tile prefix | low-variance comb | copy back
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <math_constants.h>

#include <chrono>
#include <cmath>
#include <cstdio>

#include "pf_device.cuh"
#include "rl_common.cuh"

namespace rl {

namespace cg = cooperative_groups;

int sensor_logw_launch(rl_cddt* c, double* px, double* py, double* pt, size_t n,
                       const double* scan, int nb, double fov, const rl_beam_params_t* params,
                       const float* table, int zdim, double inv_res, double* logw,
                       const MotionArgs* mot, unsigned long long* gmax_key, cudaStream_t st,
                       double* tail_w = nullptr, int32_t* tail_flag = nullptr,
                       unsigned* tail_ticket = nullptr);

__global__ void k_motion(double* __restrict__ x, double* __restrict__ y, double* __restrict__ t,
                         size_t n, MotionArgs m) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    double xi = x[i], yi = y[i], ti = t[i];
    motion_one(m, uint32_t(m.index_offset + i), xi, yi, ti);
    x[i] = xi;
    y[i] = yi;
    t[i] = ti;
  }
}

// The sensor-model block of the step: moments[0..9] (see rl_pf_weights) and,
// for the fused step, the degenerate flag of mcl.cpp:114-117.
struct Moments {
  double m[10];
  int32_t degenerate;
  int32_t pad;
};

constexpr int kPfThreads = 256;
constexpr int kPfWarps = kPfThreads / 32;

// ---- shared pieces: every path (fused step, stage entry points) runs the
// same code with the same block count, so the sums are bit-identical ----

// exp(logw - m) for this thread's grid-stride particles, accumulated moments
__device__ __forceinline__ void weight_moments(const double* __restrict__ logw, double m,
                                               const double* __restrict__ x,
                                               const double* __restrict__ y,
                                               const double* __restrict__ t, size_t n,
                                               double* __restrict__ w, double acc[10]) {
#pragma unroll
  for (int k = 0; k < 10; k++) acc[k] = 0.0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double e = exp(logw[i] - m);
    w[i] = e;
    double s, c;
    sincos(t[i], &s, &c);
    const double xi = x[i], yi = y[i];
    acc[0] += e;
    acc[1] += e * xi;
    acc[2] += e * yi;
    acc[3] += e * c;
    acc[4] += e * s;
    acc[5] += 1.0;
    acc[6] += xi;
    acc[7] += yi;
    acc[8] += c;
    acc[9] += s;
  }
}

// block sum of the 10 accumulators (warp shuffle tree, then warps in order)
// into partial[blockIdx.x * 10 + k]
__device__ __forceinline__ void block_moments(double acc[10], double* __restrict__ partial) {
  __shared__ double red[kPfWarps][10];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 10; k++) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 10) {
    double v = 0.0;
#pragma unroll
    for (int wi = 0; wi < kPfWarps; wi++) v += red[wi][threadIdx.x];
    partial[blockIdx.x * 10 + threadIdx.x] = v;
  }
}

// sum over the nblk partials of moment k by one warp: lane-strided sums,
// then a fixed shuffle tree; lane 0 holds the result
__device__ __forceinline__ double sum_partials(const double* __restrict__ partial, int nblk, int k) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll 4
  for (int b = lane; b < nblk; b += 32) s += __ldcg(partial + b * 10 + k);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  return s;
}

__device__ __forceinline__ bool degenerate_sum(double s) {
  return !(s > 0.0) || !isfinite(s);  // mcl.cpp:114-117
}

// Tiled inclusive scan of the normalised weights. Tile j covers
// [j*T, (j+1)*T) with T = scan_tile_size(n) = 256 * ceil(n / 2^18), so there
// are at most kMaxTiles tiles; local[i] is the inclusive sum within the tile
// and tile_excl[j] the sum of the earlier tile totals, so the cumulative
// weight of particle i is tile_excl[i / T] + local[i]. With normalise the
// input is w/S (or 1/n when S is degenerate) exactly as k_normalize computes
// it. Every path (fused step, stage entry points, any rank count with the
// same n) runs these same fixed trees, so the cumulative weights agree bit
// for bit.
constexpr int kMaxTiles = 1024;

__host__ __device__ __forceinline__ size_t scan_items(size_t n) {
  return (n + size_t(kPfThreads) * kMaxTiles - 1) / (size_t(kPfThreads) * kMaxTiles);
}
__host__ __device__ __forceinline__ size_t scan_tile_size(size_t n) {
  return size_t(kPfThreads) * (scan_items(n) ? scan_items(n) : 1);
}

struct ScanSmem {
  typename cub::BlockScan<double, kPfThreads>::TempStorage scan;
};

// Particle sets as the scan and the comb read them: four plain arrays, or the
// rank-concatenated block an all-gather of per-rank {x, y, theta, w} shards
// leaves ([world][4][n_local], rank-major), read in place.
struct PlainSet {
  const double *x, *y, *t, *w;
  __device__ __forceinline__ double gx(size_t i) const { return x[i]; }
  __device__ __forceinline__ double gy(size_t i) const { return y[i]; }
  __device__ __forceinline__ double gt(size_t i) const { return t[i]; }
  __device__ __forceinline__ double gw(size_t i) const { return __ldcg(w + i); }
};
struct GatheredSet {
  const double* base;
  size_t n_local;
  __device__ __forceinline__ double at(int comp, size_t i) const {
    const size_t r = i / n_local, j = i - r * n_local;
    return base[(r * 4 + size_t(comp)) * n_local + j];
  }
  __device__ __forceinline__ double gx(size_t i) const { return at(0, i); }
  __device__ __forceinline__ double gy(size_t i) const { return at(1, i); }
  __device__ __forceinline__ double gt(size_t i) const { return at(2, i); }
  __device__ __forceinline__ double gw(size_t i) const { return at(3, i); }
};

// One tile: each thread sums its ipt consecutive items sequentially, a block
// exclusive scan of the thread totals, then each item's inclusive value is its
// thread's prefix plus the running sum.
template <class Set>
__device__ __forceinline__ void scan_tile(const Set& ps, size_t n, size_t tile,
                                          bool normalise, double s, bool bad,
                                          double* __restrict__ local,
                                          double* __restrict__ tile_total, ScanSmem& sm) {
  const size_t ipt = scan_tile_size(n) / kPfThreads;
  const size_t base = tile * scan_tile_size(n) + size_t(threadIdx.x) * ipt;
  auto item = [&](size_t i) {
    if (i >= n) return 0.0;
    const double wi = ps.gw(i);  // may come from another block of this grid
    return normalise ? (bad ? 1.0 / double(n) : wi / s) : wi;
  };
  double mine = 0.0;
  for (size_t k = 0; k < ipt; k++) mine += item(base + k);
  double pre, total;
  cub::BlockScan<double, kPfThreads>(sm.scan).ExclusiveSum(mine, pre, total);
  double run = pre;
  for (size_t k = 0; k < ipt && base + k < n; k++) {
    run += item(base + k);
    local[base + k] = run;
  }
  if (threadIdx.x == 0) tile_total[tile] = total;
}

// exclusive prefix of the tile totals by one warp: 32-wide Kogge-Stone scans
// with a running carry (fixed association); tile_excl may be shared memory
__device__ __forceinline__ void tile_prefix(const double* __restrict__ tile_total, size_t tiles,
                                            double* __restrict__ tile_excl) {
  const int lane = threadIdx.x & 31;
  double carry = 0.0;
  for (size_t j0 = 0; j0 < tiles; j0 += 32) {
    const size_t j = j0 + lane;
    const double v = j < tiles ? __ldcg(tile_total + j) : 0.0;
    double inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (j < tiles) tile_excl[j] = carry + (inc - v);
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// The comb's tile tables in shared memory: tile_excl (from global, or computed
// here when tile_excl_g is null) and the tiles' end values excl + total. All
// threads of the block call it.
struct CombSmem {
  double excl[kMaxTiles], end[kMaxTiles];
};
__device__ __forceinline__ void stage_tiles(const double* __restrict__ tile_total,
                                            const double* __restrict__ tile_excl_g, size_t tiles,
                                            CombSmem& cs) {
  if (tile_excl_g) {
    for (size_t t = threadIdx.x; t < tiles; t += blockDim.x) cs.excl[t] = __ldcg(tile_excl_g + t);
  } else if (threadIdx.x < 32) {
    tile_prefix(tile_total, tiles, cs.excl);
  }
  __syncthreads();
  for (size_t t = threadIdx.x; t < tiles; t += blockDim.x)
    cs.end[t] = cs.excl[t] + __ldcg(tile_total + t);
  __syncthreads();
}

// slot m takes the first particle i with cumulative weight >= r + m/n,
// capped at n-1 (the sequential comb of mcl.cpp:130-140): the tile by a
// binary search over the tiles' end values in shared memory, then the
// particle by a binary search within the tile.
template <class Set>
__device__ __forceinline__ void comb_slots(const double* __restrict__ local, const CombSmem& cs,
                                           size_t tiles, const Set& ps, size_t n,
                                           size_t out_begin, size_t out_count,
                                           double* __restrict__ ox, double* __restrict__ oy,
                                           double* __restrict__ ot, double* __restrict__ ow,
                                           uint64_t seed, uint64_t iter) {
  double u, unused;
  philox_uniform2(seed, kResampleStream, kResampleStream, iter, u, unused);
  const double r = (1.0 / double(n)) * u;  // uniform_real_distribution(0, 1/n)
  const size_t T = scan_tile_size(n);
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < out_count;
       k += size_t(gridDim.x) * blockDim.x) {
    const size_t m = out_begin + k;
    const double target = r + double(m) / double(n);
    size_t t = 0, len = tiles;
    while (len > 0) {
      const size_t half = len >> 1, mid = t + half;
      if (cs.end[mid] < target) {
        t = mid + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    if (t >= tiles) t = tiles - 1;
    const double e = cs.excl[t];
    const size_t base = t * T, cnt = (n - base < T) ? n - base : T;
    size_t lo = 0;
    len = cnt;
    while (len > 0) {
      const size_t half = len >> 1, mid = lo + half;
      if (e + __ldcg(local + base + mid) < target) {
        lo = mid + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    const size_t i = base + lo < n ? base + lo : n - 1;
    ox[k] = ps.gx(i);
    oy[k] = ps.gy(i);
    ot[k] = ps.gt(i);
    ow[k] = 1.0 / double(n);
  }
}

// ---- stage kernels (sharded step, standalone entry points) ----

// Per-block partial moments; the last block to finish (ticket counter) sums
// the partials.
__global__ void __launch_bounds__(kPfThreads) k_weights(
    const double* __restrict__ logw, const double* __restrict__ gmax,
    const double* __restrict__ x, const double* __restrict__ y, const double* __restrict__ t,
    size_t n, double* __restrict__ w, double* __restrict__ partial, unsigned* __restrict__ ticket,
    double* __restrict__ moments) {
  double acc[10];
  weight_moments(logw, *gmax, x, y, t, n, w, acc);
  block_moments(acc, partial);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = threadIdx.x >> 5; k < 10; k += kPfWarps) {
    const double s = sum_partials(partial, gridDim.x, k);
    if ((threadIdx.x & 31) == 0) moments[k] = s;
  }
  if (threadIdx.x == 0) *ticket = 0;
}

__global__ void k_normalize(double* __restrict__ w, size_t n, const double* __restrict__ moments,
                            uint64_t n_total, int32_t* __restrict__ degenerate) {
  const double s = moments[0];
  const bool bad = degenerate_sum(s);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    w[i] = bad ? 1.0 / double(n_total) : w[i] / s;
  if (degenerate && blockIdx.x == 0 && threadIdx.x == 0) *degenerate = bad ? 1 : 0;
}

// tile scan of already-normalised weights; the last tile to finish writes the
// tile prefix
template <class Set>
__global__ void __launch_bounds__(kPfThreads) k_tile_scan(
    Set ps, size_t n, double* __restrict__ local,
    double* __restrict__ tile_total, double* __restrict__ tile_excl,
    unsigned* __restrict__ ticket) {
  __shared__ ScanSmem sm;
  __shared__ bool last;
  scan_tile(ps, n, blockIdx.x, false, 1.0, false, local, tile_total, sm);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  tile_prefix(tile_total, gridDim.x, tile_excl);
  if (threadIdx.x == 0) *ticket = 0;
}

template <class Set>
__global__ void __launch_bounds__(kPfThreads) k_comb(
    const double* __restrict__ local, const double* __restrict__ tile_total,
    const double* __restrict__ tile_excl, Set ps, size_t n, size_t out_begin, size_t out_count,
    double* __restrict__ ox, double* __restrict__ oy, double* __restrict__ ot,
    double* __restrict__ ow, uint64_t seed, uint64_t iter) {
  __shared__ CombSmem cs;
  const size_t tiles = (n + scan_tile_size(n) - 1) / scan_tile_size(n);
  stage_tiles(tile_total, tile_excl, tiles, cs);
  comb_slots(local, cs, tiles, ps, n, out_begin, out_count, ox, oy, ot, ow, seed, iter);
}

// Mcl::estimate (mcl.cpp:176-187) from the weight moments of the step:
// normalised weights w_i = e_i / S make the sums the e-moments divided by S; a
// degenerate reset gives uniform weights 1/n. est = {x, y, theta, degenerate}.
__device__ __forceinline__ void estimate_from_moments(const double* m, bool deg, uint64_t n,
                                                      double* __restrict__ est) {
  double sx, sy, sc, ss, sw;
  if (deg) {
    const double inv = 1.0 / double(n);
    sx = m[6] * inv;
    sy = m[7] * inv;
    sc = m[8] * inv;
    ss = m[9] * inv;
    sw = m[5] * inv;
  } else {
    sx = m[1] / m[0];
    sy = m[2] / m[0];
    sc = m[3] / m[0];
    ss = m[4] / m[0];
    sw = 1.0;
  }
  if (!(sw > 0.0)) sw = 1.0;
  est[0] = sx / sw;
  est[1] = sy / sw;
  est[2] = normalize_angle_2pi(atan2(ss, sc));
  est[3] = deg ? 1.0 : 0.0;
}

__global__ void k_estimate(const double* __restrict__ moments,
                           const int32_t* __restrict__ degenerate, uint64_t n,
                           double* __restrict__ est) {
  estimate_from_moments(moments, degenerate && *degenerate != 0, n, est);
}

// ---- the fused step after the sensor model: one cooperative kernel ----
struct FinishArgs {
  const double* logw;
  unsigned long long* gmax_key;
  double *x, *y, *t, *w;
  size_t n;
  double *partial, *local, *tile_total, *tile_excl, *nxyzw;
  Moments* out;
  double* est;  // optional device {x, y, theta, degenerate} (the asynchronous step)
  uint64_t seed, iter;
};

__global__ void __launch_bounds__(kPfThreads, 2) k_pf_finish(FinishArgs a) {
  cg::grid_group grid = cg::this_grid();
  const size_t n = a.n;
  // 1. weights and per-block moments
  {
    double acc[10];
    weight_moments(a.logw, order_key_value(*a.gmax_key), a.x, a.y, a.t, n, a.w, acc);
    block_moments(acc, a.partial);
  }
  grid.sync();
  // 2. every block sums the partials the same way; block 0 publishes them
  __shared__ double mom[10];
  for (int k = threadIdx.x >> 5; k < 10; k += kPfWarps) {
    const double s = sum_partials(a.partial, gridDim.x, k);
    if ((threadIdx.x & 31) == 0) mom[k] = s;
  }
  __syncthreads();
  const double S = mom[0];
  const bool bad = degenerate_sum(S);
  if (blockIdx.x == 0 && threadIdx.x < 10) a.out->m[threadIdx.x] = mom[threadIdx.x];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out->degenerate = bad ? 1 : 0;
    if (a.est) estimate_from_moments(mom, bad, n, a.est);
  }
  // 3. normalised tile scans
  __shared__ ScanSmem sm;
  const size_t tiles = (n + scan_tile_size(n) - 1) / scan_tile_size(n);
  for (size_t j = blockIdx.x; j < tiles; j += gridDim.x) {
    scan_tile(PlainSet{a.x, a.y, a.t, a.w}, n, j, true, S, bad, a.local, a.tile_total, sm);
    __syncthreads();
  }
  grid.sync();
  // 4. every block computes the tile prefix itself (the same fixed tree as the
  // stage path's), so no further grid sync; comb into the scratch set, then
  // copy back over the caller's arrays
  __shared__ CombSmem cs;
  stage_tiles(a.tile_total, nullptr, tiles, cs);
  comb_slots(a.local, cs, tiles, PlainSet{a.x, a.y, a.t, a.w}, n, 0, n, a.nxyzw, a.nxyzw + n,
             a.nxyzw + 2 * n, a.nxyzw + 3 * n, a.seed, a.iter);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.gmax_key = 0;  // ready for the next step
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    a.x[i] = __ldcg(a.nxyzw + i);
    a.y[i] = __ldcg(a.nxyzw + n + i);
    a.t[i] = __ldcg(a.nxyzw + 2 * n + i);
    a.w[i] = __ldcg(a.nxyzw + 3 * n + i);
  }
}

__global__ void k_key_to_double(const unsigned long long* __restrict__ key,
                                double* __restrict__ out) {
  const unsigned long long k = *key;
  *out = k ? order_key_value(k) : -CUDART_INF;  // key 0: nothing was scored
}

__global__ void k_copy_back(const double* __restrict__ src, double* __restrict__ x,
                            double* __restrict__ y, double* __restrict__ t,
                            double* __restrict__ w, size_t n, unsigned long long* reset_key) {
  if (reset_key && blockIdx.x == 0 && threadIdx.x == 0) *reset_key = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    x[i] = src[i];
    y[i] = src[n + i];
    t[i] = src[2 * n + i];
    w[i] = src[3 * n + i];
  }
}

static int blocks(size_t n, int threads = 256, int per_sm = 8) {
  size_t b = (n + threads - 1) / threads;
  return int(std::max<size_t>(1, std::min(b, size_t(sm_count()) * per_sm)));
}

// block count of the moment reduction: a function of n and the SM count only,
// shared by every path so the sums agree bit for bit
static int moment_blocks(size_t n) { return blocks(n, kPfThreads, 2); }

static size_t scan_tiles(size_t n) { return (n + scan_tile_size(n) - 1) / scan_tile_size(n); }

static MotionArgs motion_args(double dx, double dy, double dth, const rl_motion_noise_t* noise,
                              uint64_t seed, uint64_t iter, uint64_t offset) {
  const double trans = std::hypot(dx, dy);  // mcl.cpp:44-48
  const double st = std::max(
      noise->trans_per_trans * trans + noise->trans_per_rot * std::fabs(dth), 1e-12);
  const double sr = std::max(
      noise->rot_per_rot * std::fabs(dth) + noise->rot_per_trans * trans, 1e-12);
  return MotionArgs{dx, dy, dth, st, sr, seed, iter, offset};
}

// grows c->ws to at least `need` bytes
static int workspace(rl_cddt* c, size_t need, uint8_t** p) {
  if (c->ws.n < need) RL_TRY(c->ws.alloc(need));
  *p = c->ws.p;
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
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_motion<<<blocks(n), 256, 0, s>>>(
      x, y, theta, n, motion_args(dx, dy, dtheta, noise, seed, iteration, index_offset));
  RL_CK(cudaGetLastError());
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_pf_max(const double* logw, size_t n, double* out, void* stream) {
  if (!logw || !out || n == 0) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  size_t bytes = 0;
  cub::DeviceReduce::Max(nullptr, bytes, logw, out, int(n), s);
  void* tmp = nullptr;  // stream-ordered scratch: no synchronisation needed
  RL_TRY(scratch_alloc(&tmp, bytes, s));
  RL_CK(cub::DeviceReduce::Max(tmp, bytes, logw, out, int(n), s));
  RL_TRY(scratch_free(tmp, s));
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_pf_weights(const double* logw, const double* gmax, const double* x, const double* y,
                  const double* theta, size_t n, double* w, double* moments, void* stream) {
  if (!logw || !gmax || !x || !y || !theta || !w || !moments) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    RL_CK(cudaMemsetAsync(moments, 0, 10 * sizeof(double), s));
    RL_CK(cudaStreamSynchronize(s));
    return RL_OK;
  }
  const int nb = moment_blocks(n);
  double* partial = nullptr;  // stream-ordered scratch: partials | ticket
  RL_TRY(scratch_alloc(reinterpret_cast<void**>(&partial), 8 * (size_t(nb) * 10 + 1), s));
  unsigned* ticket = reinterpret_cast<unsigned*>(partial + size_t(nb) * 10);
  RL_CK(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  k_weights<<<nb, kPfThreads, 0, s>>>(logw, gmax, x, y, theta, n, w, partial, ticket, moments);
  RL_CK(cudaGetLastError());
  RL_TRY(scratch_free(partial, s));
  if (!stream) RL_CK(cudaStreamSynchronize(s));
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
  const size_t T = scan_tiles(n);
  double* local = nullptr;  // stream-ordered scratch: local[n] | tile_total[T] | tile_excl[T] | ticket
  RL_TRY(scratch_alloc(reinterpret_cast<void**>(&local), 8 * (n + 2 * T + 1), s));
  double *tile_total = local + n, *tile_excl = tile_total + T;
  unsigned* ticket = reinterpret_cast<unsigned*>(tile_excl + T);
  RL_CK(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  const PlainSet ps{x, y, theta, w};
  k_tile_scan<<<int(T), kPfThreads, 0, s>>>(ps, n, local, tile_total, tile_excl, ticket);
  k_comb<<<blocks(out_count), 256, 0, s>>>(local, tile_total, tile_excl, ps, n, out_begin,
                                          out_count, ox, oy, otheta, ow, seed, iteration);
  RL_CK(cudaGetLastError());
  RL_TRY(scratch_free(local, s));
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

}  // extern "C"

// The fused Mcl::step. Synchronous form (est_dev == nullptr): the moments come
// back to the host and `estimate` is computed there. Asynchronous form: the
// estimate is computed on the device into est_dev and nothing waits.
static int mcl_step_impl(rl_cddt* c, double* x, double* y, double* theta, double* w, size_t n,
                         double odo_dx, double odo_dy, double odo_dtheta, const double* scan,
                         int32_t nbeams, double fov, const rl_motion_noise_t* noise,
                         const rl_beam_params_t* params, const float* table, int32_t zdim,
                         double inv_res, uint64_t seed, uint64_t iteration, double* estimate,
                         double* est_dev, void* stream) {
  if (!c || !noise || !scan || nbeams <= 0 || (n && (!x || !y || !theta || !w))) return RL_EINVAL;
  if (n > (1ull << 32)) {
    set_error("motion_update: particle index exceeds the 32-bit RNG counter");
    return RL_EINVAL;
  }
  if (n == 0) return RL_OK;
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  cudaStream_t st = pick_stream(c, stream);
  // control (pf_ctl): {gmax key, ticket} | Moments; workspace: logw[n] |
  // resampled x y t w [4n] | local[n] | tile_total[T] | tile_excl[T] | partial[nbw * 10]
  struct Control {
    unsigned long long gmax_key;
    unsigned ticket;
  };
  if (!c->pf_ctl.p) RL_TRY(c->pf_ctl.alloc(256));
  if (!c->pf_host) RL_CK(cudaMallocHost(&c->pf_host, sizeof(Moments)));
  const int nbw = moment_blocks(n);
  const size_t T = scan_tiles(n);
  const size_t need = 8 * (6 * n + 2 * T + 10 * size_t(nbw));
  uint8_t* base = nullptr;
  RL_TRY(workspace(c, need, &base));
  Control* ctl = reinterpret_cast<Control*>(c->pf_ctl.p);
  Moments* mom = reinterpret_cast<Moments*>(c->pf_ctl.p + 128);
  FinishArgs fa{};
  fa.logw = reinterpret_cast<double*>(base);
  fa.gmax_key = &ctl->gmax_key;
  fa.x = x;
  fa.y = y;
  fa.t = theta;
  fa.w = w;
  fa.n = n;
  fa.nxyzw = const_cast<double*>(fa.logw) + n;
  fa.local = fa.nxyzw + 4 * n;
  fa.tile_total = fa.local + n;
  fa.tile_excl = fa.tile_total + T;
  fa.partial = fa.tile_excl + T;
  fa.out = mom;
  fa.est = est_dev;
  fa.seed = seed;
  fa.iter = iteration;

#ifdef RL_PF_TRACE
  static cudaEvent_t ev[5];
  static bool evi = [] { for (auto& e : ev) cudaEventCreate(&e); return true; }();
  (void)evi;
  auto host_t0 = std::chrono::steady_clock::now();
  cudaEventRecord(ev[0], st);
#endif
  if (!c->pf_ctl_clean) RL_CK(cudaMemsetAsync(ctl, 0, sizeof(Control), st));
  c->pf_ctl_clean = false;
  const MotionArgs mot = motion_args(odo_dx, odo_dy, odo_dtheta, noise, seed, iteration, 0);
  RL_TRY(sensor_logw_launch(c, x, y, theta, n, scan, nbeams, fov, params, table, zdim, inv_res,
                            const_cast<double*>(fa.logw), &mot, &ctl->gmax_key, st));
#ifdef RL_PF_TRACE
  cudaEventRecord(ev[1], st);
#endif
  static const int coop_per_sm = [] {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pf_finish, kPfThreads, 0);
    return per_sm;
  }();
  if (coop_per_sm >= 2) {
    void* args[] = {&fa};
    RL_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_pf_finish), dim3(nbw),
                                      dim3(kPfThreads), args, 0, st));
  } else {
    // same arithmetic as k_pf_finish, stage by stage
    double* gmax = reinterpret_cast<double*>(c->pf_ctl.p + 64);
    k_key_to_double<<<1, 1, 0, st>>>(&ctl->gmax_key, gmax);
    k_weights<<<nbw, kPfThreads, 0, st>>>(fa.logw, gmax, x, y, theta, n, w, fa.partial,
                                          &ctl->ticket, mom->m);
    k_normalize<<<blocks(n), 256, 0, st>>>(w, n, mom->m, n, &mom->degenerate);
    const PlainSet ps{x, y, theta, w};
    k_tile_scan<<<int(T), kPfThreads, 0, st>>>(ps, n, fa.local, fa.tile_total, fa.tile_excl,
                                               &ctl->ticket);
    if (est_dev) k_estimate<<<1, 1, 0, st>>>(mom->m, &mom->degenerate, n, est_dev);
    k_comb<<<blocks(n), 256, 0, st>>>(fa.local, fa.tile_total, fa.tile_excl, ps, n, 0, n, fa.nxyzw,
                                      fa.nxyzw + n, fa.nxyzw + 2 * n, fa.nxyzw + 3 * n, seed,
                                      iteration);
    k_copy_back<<<blocks(n), 256, 0, st>>>(fa.nxyzw, x, y, theta, w, n, &ctl->gmax_key);
  }
  RL_CK(cudaGetLastError());
  if (est_dev) {
    // the key is reset by the step itself, in stream order
    c->pf_ctl_clean = true;
    return RL_OK;
  }
#ifdef RL_PF_TRACE
  cudaEventRecord(ev[2], st);
  auto host_t1 = std::chrono::steady_clock::now();
#endif
  Moments& h = *static_cast<Moments*>(c->pf_host);
  RL_CK(cudaMemcpyAsync(&h, mom, sizeof h, cudaMemcpyDeviceToHost, st));
#ifdef RL_PF_TRACE
  cudaEventRecord(ev[3], st);
#endif
  RL_CK(cudaStreamSynchronize(st));
  c->pf_ctl_clean = true;
#ifdef RL_PF_TRACE
  auto host_t2 = std::chrono::steady_clock::now();
  float a = 0, b = 0, c3 = 0;
  cudaEventElapsedTime(&a, ev[0], ev[1]);
  cudaEventElapsedTime(&b, ev[1], ev[2]);
  cudaEventElapsedTime(&c3, ev[2], ev[3]);
  fprintf(stderr, "trace memset+sensor %.1f finish %.1f d2h %.1f | host enqueue %.1f total %.1f us\n",
          a * 1e3, b * 1e3, c3 * 1e3,
          std::chrono::duration<double, std::micro>(host_t1 - host_t0).count(),
          std::chrono::duration<double, std::micro>(host_t2 - host_t0).count());
#endif
  const double* m = h.m;
  const bool deg = h.degenerate != 0;
  if (estimate) {
    // Mcl::estimate (mcl.cpp:176-187) on the normalised weights: with
    // normalised w_i = e_i / S the sums are the e-moments divided by S; a
    // degenerate reset gives uniform weights 1/n.
    double sx, sy, sc, ss, sw;
    if (deg) {
      const double inv = 1.0 / double(n);
      sx = m[6] * inv;
      sy = m[7] * inv;
      sc = m[8] * inv;
      ss = m[9] * inv;
      sw = m[5] * inv;
    } else {
      sx = m[1] / m[0];
      sy = m[2] / m[0];
      sc = m[3] / m[0];
      ss = m[4] / m[0];
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

extern "C" {

int rl_mcl_step(rl_cddt* c, double* x, double* y, double* theta, double* w, size_t n,
                double odo_dx, double odo_dy, double odo_dtheta, const double* scan,
                int32_t nbeams, double fov, const rl_motion_noise_t* noise,
                const rl_beam_params_t* params, const float* table, int32_t zdim, double inv_res,
                uint64_t seed, uint64_t iteration, double* estimate, void* stream) {
  return mcl_step_impl(c, x, y, theta, w, n, odo_dx, odo_dy, odo_dtheta, scan, nbeams, fov, noise,
                       params, table, zdim, inv_res, seed, iteration, estimate, nullptr, stream);
}

int rl_mcl_step_async(rl_cddt* c, double* x, double* y, double* theta, double* w, size_t n,
                      double odo_dx, double odo_dy, double odo_dtheta, const double* scan,
                      int32_t nbeams, double fov, const rl_motion_noise_t* noise,
                      const rl_beam_params_t* params, const float* table, int32_t zdim,
                      double inv_res, uint64_t seed, uint64_t iteration, double* estimate_dev,
                      void* stream) {
  if (!estimate_dev || !stream) {
    set_error("rl_mcl_step_async needs a device estimate buffer and a stream");
    return RL_EINVAL;
  }
  if (n == 0) return RL_OK;
  return mcl_step_impl(c, x, y, theta, w, n, odo_dx, odo_dy, odo_dtheta, scan, nbeams, fov, noise,
                       params, table, zdim, inv_res, seed, iteration, nullptr, estimate_dev,
                       stream);
}

int rl_pf_estimate(const double* moments, const int32_t* degenerate, uint64_t n_total,
                   double* estimate_dev, void* stream) {
  if (!moments || !estimate_dev || n_total == 0) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_estimate<<<1, 1, 0, s>>>(moments, degenerate, n_total, estimate_dev);
  RL_CK(cudaGetLastError());
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_resample_gathered(const double* gathered, size_t n_local, int32_t world, size_t out_begin,
                         size_t out_count, double* ox, double* oy, double* otheta, double* ow,
                         uint64_t seed, uint64_t iteration, void* stream) {
  if (world <= 0 || n_local == 0 || out_count == 0) return world > 0 ? RL_OK : RL_EINVAL;
  const size_t n = n_local * size_t(world);
  if (!gathered || !ox || !oy || !otheta || !ow || out_begin + out_count > n) return RL_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t T = scan_tiles(n);
  double* local = nullptr;  // stream-ordered scratch: local[n] | tile_total[T] | tile_excl[T] | ticket
  RL_TRY(scratch_alloc(reinterpret_cast<void**>(&local), 8 * (n + 2 * T + 1), s));
  double *tile_total = local + n, *tile_excl = tile_total + T;
  unsigned* ticket = reinterpret_cast<unsigned*>(tile_excl + T);
  RL_CK(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
  const GatheredSet ps{gathered, n_local};
  k_tile_scan<<<int(T), kPfThreads, 0, s>>>(ps, n, local, tile_total, tile_excl, ticket);
  k_comb<<<blocks(out_count), 256, 0, s>>>(local, tile_total, tile_excl, ps, n, out_begin,
                                          out_count, ox, oy, otheta, ow, seed, iteration);
  RL_CK(cudaGetLastError());
  RL_TRY(scratch_free(local, s));
  if (!stream) RL_CK(cudaStreamSynchronize(s));
  return RL_OK;
}

int rl_pf_shard_sensor(rl_cddt* c, double* x, double* y, double* theta, size_t n,
                       uint64_t index_offset, double odo_dx, double odo_dy, double odo_dtheta,
                       const rl_motion_noise_t* noise, uint64_t seed, uint64_t iteration,
                       const double* scan, int32_t nbeams, double fov,
                       const rl_beam_params_t* params, const float* table, int32_t zdim,
                       double inv_res, double* logw, double* local_max, void* stream) {
  if (!c || !local_max || !scan || nbeams <= 0 || (n && (!x || !y || !theta || !logw)))
    return RL_EINVAL;
  if (index_offset + n > (1ull << 32)) {
    set_error("motion_update: particle index exceeds the 32-bit RNG counter");
    return RL_EINVAL;
  }
  if (!table && (!params || !(params->z_max > 0.0))) {
    set_error("beam model z_max must be positive");  // mcl.cpp:13
    return RL_EINVAL;
  }
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  cudaStream_t st = pick_stream(c, stream);
  unsigned long long* key = nullptr;  // stream-ordered scratch: the max key
  RL_TRY(scratch_alloc(reinterpret_cast<void**>(&key), sizeof *key, st));
  RL_CK(cudaMemsetAsync(key, 0, sizeof *key, st));
  if (n) {
    MotionArgs mot{};
    if (noise) mot = motion_args(odo_dx, odo_dy, odo_dtheta, noise, seed, iteration, index_offset);
    RL_TRY(sensor_logw_launch(c, x, y, theta, n, scan, nbeams, fov, params, table, zdim, inv_res,
                              logw, noise ? &mot : nullptr, key, st));
  }
  // an empty shard reports -inf (key 0 decodes to NaN; the max all-reduce must ignore it)
  k_key_to_double<<<1, 1, 0, st>>>(key, local_max);
  RL_CK(cudaGetLastError());
  RL_TRY(scratch_free(key, st));
  return finish(c, stream);
}

}  // extern "C"
