// Fused beam sensor model: sensor_update (proj/src/mcl.cpp:58-120) on the GPU.
//
// One CTA scores PB particles x nbeams beams: every (particle, beam) item is a
// CDDT cast (cddt_device.cuh) followed by the likelihood lookup, the per-beam
// log-likelihoods land in shared memory and one thread per particle sums them
// in beam order 0..nbeams-1 — the reference's summation order, so the FP64
// log-weight is reproducible. Normalisation (max-subtract, exp, sum, divide,
// degenerate reset, mcl.cpp:108-119) follows as a reduction.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "pf_device.cuh"
#include "rl_common.cuh"

namespace rl {

namespace cg = cooperative_groups;

// particles per CTA: 16 for large sets (config 4), 8 below kSmallSet so a
// few thousand particles still fill the GPU (config 2)
constexpr size_t kSmallSet = 16384;
// sensor_update fuses its normalisation into the log-weight kernel up to this
// many particles (the last CTA normalises; beyond it a grid-wide pass is faster)
constexpr size_t kTailMax = 8192;

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

// Normalisation fused into the sensor kernel for small particle sets
// (mcl.cpp:104-119): the last CTA to finish (a ticket counter) takes the max
// log-weight from the atomic key, computes w = exp(logw - max), their sum in a
// fixed order (thread-strided partial sums, a fixed shuffle tree, warps in
// order), and w /= S or the degenerate reset; then it zeroes the key and the
// ticket for the next call. Saves the separate normalisation launch where the
// whole update is a few tens of microseconds (config 2).
struct NormTail {
  double* w;           // nullptr: no fused normalisation
  int32_t* degenerate;
  unsigned* ticket;
};

__device__ __forceinline__ void normalize_tail(const NormTail& nt,
                                               const double* __restrict__ logw, size_t n,
                                               unsigned long long* __restrict__ key) {
  __shared__ bool last;
  __shared__ double red[32];
  __syncthreads();  // this CTA's log-weights are written and fenced, its max is in the key
  if (threadIdx.x == 0) last = atomicAdd(nt.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double m = order_key_value(__ldcg(key));
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = exp(__ldcg(logw + i) - m);
    nt.w[i] = e;
    acc += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0;
    for (int k = 0; k < int(blockDim.x >> 5); k++) S += red[k];
    red[0] = S;
  }
  __syncthreads();
  const double S = red[0];
  const bool bad = !(S > 0.0) || !isfinite(S);  // mcl.cpp:114
  for (size_t i = threadIdx.x; i < n; i += blockDim.x)
    nt.w[i] = bad ? 1.0 / double(n) : nt.w[i] / S;
  if (threadIdx.x == 0) {
    *nt.degenerate = bad ? 1 : 0;
    *key = 0;
    *nt.ticket = 0;
  }
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
    MotionArgs mot, unsigned long long* __restrict__ gmax_key, NormTail nt) {
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
  __shared__ LongCast lq[kLongQueue];
  __shared__ unsigned lq_n;
  if (threadIdx.x == 0) lq_n = 0;
  __syncthreads();
  const int items = kSensorParticlesPerCta * nb;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int pl = it / nb, b = it % nb;
    if (p0 + pl >= n) continue;
    const double th = normalize_angle_2pi(pose[2][pl] + boff[b]);
    const int a = direction_index(th, c.K);
    double e;
    int next, cap = RL_COOP_WCAP;
    bool queued = false;
#pragma unroll 1
    while (!directional_cast_capped(c, pose[0][pl], pose[1][pl], a, cap, &e, &next)) {
      const unsigned slot = atomicAdd(&lq_n, 1u);
      if (slot < kLongQueue) {  // a warp finishes it in phase B
        lq[slot] = LongCast{pose[0][pl], pose[1][pl], a, next, unsigned(it), 0u};
        queued = true;
        break;
      }
      cap = -1;  // queue full: this thread finishes the cast itself
    }
    if (!queued) ll[it] = item_loglike(e, b, scan, bp, table, mrow[b], zdim, inv_res);
  }
  __syncthreads();
  {  // phase B: queued long casts, one warp each
    const unsigned nq = min(lq_n, unsigned(kLongQueue));
    for (unsigned k = threadIdx.x >> 5; k < nq; k += blockDim.x >> 5) {
      const LongCast lc = lq[k];
      const double e = resume_coop(c, lc.x, lc.y, lc.a, lc.idx);
      if ((threadIdx.x & 31) == 0) {
        const int b = int(lc.slot) % nb;
        ll[lc.slot] = item_loglike(e, b, scan, bp, table, mrow[b], zdim, inv_res);
      }
    }
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
      if (nt.w) __threadfence();  // visible to the CTA that normalises
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
  if (nt.w) normalize_tail(nt, logw, n, gmax_key);
}



// ---- paired beams: one row search for the casts at a and a + K/2 ----
//
// sensor_update pairs beams whose directions are opposite (mcl.cpp:66-96): a
// direction a < S and a + S share the slice s = a, hence the row and the
// projected x' (cddt.cpp:213-221). Forward visits the zero points above x'
// (std::upper_bound), backward those below (std::lower_bound, cddt.hpp:106-131);
// the two partition points differ only across zero points equal to x', so
// one search gives both starts ("a single additional memory read", PAPER.md).
// Each direction then runs the reference's near-field walk and candidate loop
// on its own, so the pair returns exactly what two directional_casts return
// (cast_pair, cddt.cpp:275-279).
struct PairSearch {
  uint32_t pb, pf;  // backward / forward partition points (pb <= pf)
  uint32_t kb, kf;  // indices whose zero points the search loaded (~0u: none)
  float vb, vf;
};

__device__ __forceinline__ PairSearch partition_point_pair(const float* __restrict__ v,
                                                           uint32_t n, double xq, float4 h,
                                                           float4 h2) {
  PairSearch r{0, 0, ~0u, ~0u, 0.f, 0.f};
  // backward threshold: double(e) < xq  <=>  e < RU_f32(xq)
  const float rd = __double2float_rd(xq), thr = __double2float_ru(xq);
  uint32_t first = 0, len = n, path = 0;
#pragma unroll
  for (int l = 0; l < kHintLevels; l++) {
    if (len == 0) break;
    const uint32_t half = len >> 1, mid = first + half;
    float e;
    if (l == 0) {
      e = h.z;
    } else if (l == 1) {
      e = path ? h2.x : h.w;
    } else {
      e = path == 0 ? h2.y : path == 1 ? h2.z : path == 2 ? h2.w : __ldg(v + mid);
    }
    const bool pass = e < thr;
    if (pass) {  // rightmost passing probe: backward's first candidate when it is first - 1
      r.kb = mid;
      r.vb = e;
      first = mid + 1;
      len -= half + 1;
    } else {  // leftmost failing probe: forward's first candidate when it is first
      r.kf = mid;
      r.vf = e;
      len = half;
    }
    path = (path << 1) | (pass ? 1u : 0u);
  }
  while (len > kLinearTail) {
    const uint32_t half = len >> 1, mid = first + half;
    const float e = __ldg(v + mid);
    if (e < thr) {
      r.kb = mid;
      r.vb = e;
      first = mid + 1;
      len -= half + 1;
    } else {
      r.kf = mid;
      r.vf = e;
      len = half;
    }
  }
  if (len > 0) {
    float e[kLinearTail > 0 ? kLinearTail : 1];
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kLinearTail; k++) {
      e[k] = uint32_t(k) < len ? __ldg(v + first + k) : __int_as_float(0x7f800000);
      cnt += e[k] < thr ? 1u : 0u;
    }
    float cb = e[0], cf = e[0];
#pragma unroll
    for (int k = 1; k < kLinearTail; k++) {
      cb = int(cnt) - 1 == k ? e[k] : cb;
      cf = int(cnt) == k ? e[k] : cf;
    }
    if (cnt > 0) {
      r.kb = first + cnt - 1;
      r.vb = cb;
    }
    if (cnt < len) {
      r.kf = first + cnt;
      r.vf = cf;
    }
    first += cnt;
  }
  r.pb = r.pf = first;
  if (rd == thr) {
    // x' is a float X: zero points equal to X lie below it for the forward
    // direction (double(e) <= x') and not for the backward one (double(e) < x')
    const float thf = nextafterf(rd, __int_as_float(0x7f800000));
    while (r.pf < n && (r.pf == r.kf ? r.vf : __ldg(v + r.pf)) < thf) r.pf++;
  }
  return r;
}

// One direction of a pair: the near-field walk when the origin is not clear
// (cddt.cpp:225-232), then the candidate loop from idx (cddt.cpp:236-262).
__device__ __forceinline__ double pair_side(const CddtView& c, double x, double y, int a,
                                            bool fwd, double xq, const float* __restrict__ v,
                                            int n, int idx, uint32_t kidx, float kval,
                                            bool clear) {
  const double4 dir = c.dirs[a];
  Walker<false> wk;
  bool have_walker = false;
  if (!clear) {
    wk.init_at(x, y, dir, 0.0);
    have_walker = true;
    const double r = wk.scan_to(c, kNearField);
    if (r >= 0.0) return (c.max_range < r) ? c.max_range : r;
    if (r == kWalkExit) return c.max_range;
  }
  const int step = fwd ? 1 : -1;
  for (; idx >= 0 && idx < n; idx += step) {
    const double vv = (double)(uint32_t(idx) == kidx ? kval : __ldg(v + idx));
    const double d = fwd ? vv - xq : xq - vv;
    if (d >= c.max_range) break;
    int32_t cell;
    if (landing_hit(c, x + d * dir.x, y + d * dir.y, &cell)) return d;
#if RL_PROBE_SENSOR
    if (window_probe_hit(c, x, y, dir.x, dir.y, d)) return d;
#endif
    if (!have_walker) {
      wk.init_at(x, y, dir, d - kVerifyHalf);
      have_walker = true;
    } else {
      wk.seek(d - kVerifyHalf);
    }
    const double r = wk.scan_to(c, d + kVerifyHalf);
    if (r == kWalkExit) break;
    if (r < 0.0) continue;
    return d;
  }
  return c.max_range;
}

// directional_cast at the directions of one slice s: s itself when want_f,
// s + S when want_b (one or both), from one origin test, row and search.
__device__ __forceinline__ void slice_casts(const CddtView& c, double x, double y, int s,
                                            bool want_f, bool want_b, double* rf, double* rb) {
  const int cxi = (int)floor(x), cyi = (int)floor(y);
  if (!in_bounds(c, cxi, cyi)) {  // cddt.cpp:209
    *rf = *rb = c.max_range;
    return;
  }
  const QueryRow q = query_row(c, x, y, s);
  RL_DCHECK(c, unsigned(cxi) < unsigned(c.w) && unsigned(cyi) < unsigned(c.h), 5);
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {  // cddt.cpp:210
    *rf = *rb = 0.0;
    return;
  }
  const bool clear = (w0.y >> (cxi & 31)) & 1u;
  const float* __restrict__ v = c.zp + q.lo;
  const int n = (int)(q.hi - q.lo);
  const PairSearch ps = partition_point_pair(v, uint32_t(n), q.xq, q.hint, q.hint2);
#pragma unroll 1
  for (int side = want_f ? 0 : 1; side < (want_b ? 2 : 1); side++) {
    const bool fwd = side == 0;
    const double r = pair_side(c, x, y, fwd ? s : s + c.S, fwd, q.xq, v, n,
                               fwd ? int(ps.pf) : int(ps.pb) - 1, fwd ? ps.kf : ps.kb,
                               fwd ? ps.vf : ps.vb, clear);
    if (fwd)
      *rf = r;
    else
      *rb = r;
  }
}

// The beam jobs of one scan: pairs (b1, b2) whose offsets differ by about pi
// (cast as a pair when the particle's two directions are exactly opposite,
// otherwise as two casts), then the unpaired beams (b2 = -1).
constexpr int kMaxJobs = 256;
struct BeamJobs {
  int n;
  int16_t b1[kMaxJobs], b2[kMaxJobs];
};

#ifndef RL_SENSOR_PAIRED_MINB
#define RL_SENSOR_PAIRED_MINB 3  // 80 registers: -1.5 % against 64 with spills (config 4)
#endif
template <bool MOTION, int kSensorParticlesPerCta>
__global__ void __launch_bounds__(256, kSensorParticlesPerCta < 16 ? RL_SENSOR_MINB_SMALL
                                                                   : RL_SENSOR_PAIRED_MINB)
    k_sensor_logw_paired(
    CddtView c, double* __restrict__ px, double* __restrict__ py, double* __restrict__ pt,
    size_t n, const double* __restrict__ scan, int nb, double fov, BeamParams bp,
    const float* __restrict__ table, int zdim, double inv_res, double* __restrict__ logw,
    MotionArgs mot, unsigned long long* __restrict__ gmax_key, NormTail nt,
    const __grid_constant__ BeamJobs jobs) {
  extern __shared__ double ll[];  // [PB][nb] log-likelihoods | [nb] beam offsets | [nb] table rows
  double* boff = ll + kSensorParticlesPerCta * nb;
  int* mrow = reinterpret_cast<int*>(boff + nb);
  __shared__ double pose[3][kSensorParticlesPerCta];
  __shared__ unsigned next_item;
  const size_t p0 = size_t(blockIdx.x) * kSensorParticlesPerCta;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    boff[b] = beam_offset(b, nb, fov);  // ScanSpec::beam_offset (mcl.hpp:42-51)
    if (table) mrow[b] = table_index(scan[b], inv_res, zdim) * zdim;
  }
  if (threadIdx.x == 0) next_item = 0;
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
  // jobs are handed out to warps 32 at a time, so a warp that drew short
  // casts takes more instead of idling at the barrier
  const unsigned items = unsigned(kSensorParticlesPerCta * jobs.n);
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&next_item, 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= items) break;
    const unsigned it = base + unsigned(lane);
    if (it >= items) continue;
#ifndef RL_SENSOR_PARTICLE_MAJOR
    // job-major: consecutive items are one job for consecutive particles, so a
    // warp's lanes run the same kind of job (pairs with pairs, singles with singles)
    const int j = int(it / unsigned(kSensorParticlesPerCta)),
              pl = int(it % unsigned(kSensorParticlesPerCta));
#else
    const int pl = int(it / unsigned(jobs.n)), j = int(it % unsigned(jobs.n));
#endif
    if (p0 + pl >= n) continue;
    const double x = pose[0][pl], y = pose[1][pl], t = pose[2][pl];
    const int b1 = jobs.b1[j], b2 = jobs.b2[j];
    RL_DCHECK(c, j < jobs.n && b1 >= 0 && b1 < nb && b2 < nb && pl < kSensorParticlesPerCta, 20);
    const int a1 = direction_index(normalize_angle_2pi(t + boff[b1]), c.K);
    const int a2 = b2 < 0 ? -1 : direction_index(normalize_angle_2pi(t + boff[b2]), c.K);
    // one slice visit for an exactly opposite pair, else one per beam
    const bool paired = a2 >= 0 && a2 == (a1 < c.S ? a1 + c.S : a1 - c.S);
    double e1 = 0.0, e2 = 0.0;
#pragma unroll 1
    for (int k = 0; k < (paired || b2 < 0 ? 1 : 2); k++) {
      const int a = k == 0 ? a1 : a2;
      const int sl = a < c.S ? a : a - c.S;
      const bool f1 = a1 < c.S;  // beam 1 is this slice's forward direction
      double rf, rb;
      slice_casts(c, x, y, sl, paired ? true : a < c.S, paired ? true : a >= c.S, &rf, &rb);
      if (paired) {
        e1 = f1 ? rf : rb;
        e2 = f1 ? rb : rf;
      } else if (k == 0) {
        e1 = a < c.S ? rf : rb;
      } else {
        e2 = a < c.S ? rf : rb;
      }
    }
    if (b2 >= 0) ll[pl * nb + b2] = item_loglike(e2, b2, scan, bp, table, mrow[b2], zdim, inv_res);
    ll[pl * nb + b1] = item_loglike(e1, b1, scan, bp, table, mrow[b1], zdim, inv_res);
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
      if (nt.w) __threadfence();  // visible to the CTA that normalises
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
  if (nt.w) normalize_tail(nt, logw, n, gmax_key);
}

// Host: the job list of a scan (nb beams over fov) for theta_disc K. Beam b
// pairs with the beam whose offset is nearest off(b) + pi when they differ by
// pi within half a direction step (then the particle's two directions are
// opposite for most headings; the kernel checks each particle exactly).
static bool beam_jobs(int nb, double fov, int K, BeamJobs* jobs) {
  if (nb > kMaxJobs) return false;
  std::vector<double> off(nb);
  for (int b = 0; b < nb; b++) off[b] = nb <= 1 ? 0.0 : -fov / 2.0 + fov * double(b) / double(nb - 1);
  std::vector<int> partner(nb, -1);
  const double tol = 3.14159265358979323846 / double(K);
  for (int b = 0; b < nb; b++) {
    if (partner[b] >= 0) continue;
    int best = -1;
    double bd = tol;
    for (int b2 = b + 1; b2 < nb; b2++) {
      const double d = std::fabs(off[b2] - off[b] - 3.14159265358979323846);
      if (partner[b2] < 0 && d < bd) {
        bd = d;
        best = b2;
      }
    }
    if (best >= 0) {
      partner[b] = best;
      partner[best] = b;
    }
  }
  static const bool singles = [] {  // A/B hook: every beam its own job
    const char* e = std::getenv("RL_SENSOR_JOBS_SINGLE");
    return e && std::atoi(e) != 0;
  }();
  if (singles) std::fill(partner.begin(), partner.end(), -1);
  jobs->n = 0;
  for (int b = 0; b < nb; b++)
    if (partner[b] > b) {
      jobs->b1[jobs->n] = int16_t(b);
      jobs->b2[jobs->n] = int16_t(partner[b]);
      jobs->n++;
    }
  for (int b = 0; b < nb; b++)
    if (partner[b] < 0) {
      jobs->b1[jobs->n] = int16_t(b);
      jobs->b2[jobs->n] = -1;
      jobs->n++;
    }
  return true;
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


// Kernel choice: the paired-beam kernel for large sets, where throughput
// decides (config 4: -12 % per filter step); one cast per beam for small ones,
// where the slowest cast decides (config 2: the paired form is +4 %).
// RL_SENSOR_PAIRED / RL_SENSOR_PAIRED_SMALL override (A/B and the bitwise
// paired-vs-unpaired test).
int sensor_logw_launch(rl_cddt* c, double* px, double* py, double* pt, size_t n,
                       const double* scan, int nb, double fov, const rl_beam_params_t* params,
                       const float* table, int zdim, double inv_res, double* logw,
                       const MotionArgs* mot, unsigned long long* gmax_key, cudaStream_t st,
                       double* tail_w, int32_t* tail_flag, unsigned* tail_ticket) {
  BeamParams bp{};
  if (params)
    bp = BeamParams{params->w_hit,     params->w_short,      params->w_max, params->w_rand,
                    params->sigma_hit, params->lambda_short, params->z_max};
  const MotionArgs m = mot ? *mot : MotionArgs{};
  const NormTail nt{tail_w, tail_flag, tail_ticket};
  // CTA size: enough threads for one work item each (up to 256)
  auto threads_for = [](int items) { return std::min(256, std::max(32, (items + 31) / 32 * 32)); };
  auto launch = [&](auto kernel, int pb) -> int {
    const int ctas = int((n + pb - 1) / pb);
    const size_t smem = sizeof(double) * (pb + 1) * nb + sizeof(int) * nb;
    if (smem > 48 * 1024)
      RL_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kernel<<<ctas, threads_for(pb * nb), smem, st>>>(c->view(), px, py, pt, n, scan, nb, fov, bp,
                                                     table, zdim, inv_res, logw, m, gmax_key, nt);
    return RL_OK;
  };
  static const int pb_small = [] {
    const char* e = std::getenv("RL_SENSOR_PB_SMALL");
    return e ? std::atoi(e) : 8;
  }();
  auto env_flag = [](const char* name, bool dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) != 0 : dflt;
  };
  static const bool paired_large = env_flag("RL_SENSOR_PAIRED", true);
  static const bool paired_small = env_flag("RL_SENSOR_PAIRED_SMALL", env_flag("RL_SENSOR_PAIRED", false));
  const bool small = n < kSmallSet;
  BeamJobs jobs;
  if ((small ? paired_small : paired_large) && beam_jobs(nb, fov, c->K, &jobs)) {
    auto launch_p = [&](auto kernel, int pb) -> int {
      const int ctas = int((n + pb - 1) / pb);
      const size_t smem = sizeof(double) * (pb + 1) * nb + sizeof(int) * nb;
      if (smem > 48 * 1024)
        RL_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
      kernel<<<ctas, threads_for(pb * jobs.n), smem, st>>>(c->view(), px, py, pt, n, scan, nb,
                                                           fov, bp, table, zdim, inv_res, logw, m,
                                                           gmax_key, nt, jobs);
      return RL_OK;
    };
    if (small && pb_small == 4) {
      RL_TRY(mot ? launch_p(k_sensor_logw_paired<true, 4>, 4)
                 : launch_p(k_sensor_logw_paired<false, 4>, 4));
    } else if (small) {
      RL_TRY(mot ? launch_p(k_sensor_logw_paired<true, 8>, 8)
                 : launch_p(k_sensor_logw_paired<false, 8>, 8));
    } else {
      RL_TRY(mot ? launch_p(k_sensor_logw_paired<true, 16>, 16)
                 : launch_p(k_sensor_logw_paired<false, 16>, 16));
    }
  } else if (small && pb_small == 4) {
    RL_TRY(mot ? launch(k_sensor_logw<true, 4>, 4) : launch(k_sensor_logw<false, 4>, 4));
  } else if (small) {
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
                            inv_res, logw, nullptr, nullptr, pick_stream(c, stream), nullptr,
                            nullptr, nullptr));
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
  static const size_t tail_max = [] {
    const char* e = std::getenv("RL_SENSOR_TAIL_MAX");
    return e ? size_t(std::strtoull(e, nullptr, 10)) : size_t(kTailMax);
  }();
  if (n <= tail_max) {
    // one kernel: log-weights, then the last CTA normalises (normalize_tail).
    // Its control words {max key, ticket, flag} live in sensor_ctl and are
    // left zeroed by every completed launch.
    if (!c->sensor_ctl.p) {
      RL_TRY(c->sensor_ctl.alloc(64));
      RL_CK(cudaMemsetAsync(c->sensor_ctl.p, 0, 64, st));
    } else if (!c->sensor_ctl_clean) {
      RL_CK(cudaMemsetAsync(c->sensor_ctl.p, 0, 16, st));
    }
    c->sensor_ctl_clean = false;
    unsigned long long* key = reinterpret_cast<unsigned long long*>(c->sensor_ctl.p);
    unsigned* ticket = reinterpret_cast<unsigned*>(c->sensor_ctl.p + 8);
    int* d_flag = degenerate_dev ? degenerate_dev : reinterpret_cast<int*>(c->sensor_ctl.p + 16);
    double* d_logw = logw ? logw : reinterpret_cast<double*>(base + 64);
    double* d_w = weight ? weight : reinterpret_cast<double*>(base + 64 + 8 * n);
    RL_TRY(sensor_logw_launch(c, const_cast<double*>(px), const_cast<double*>(py),
                              const_cast<double*>(pt), n, scan, nbeams, fov, params, table, zdim,
                              inv_res, d_logw, nullptr, key, st, d_w, d_flag, ticket));
    c->sensor_ctl_clean = true;
    if (degenerate_dev) return RL_OK;
    uint32_t* hs = nullptr;
    RL_TRY(host_small(c, &hs));
    RL_CK(cudaMemcpyAsync(hs, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    RL_CK(cudaStreamSynchronize(st));
    return hs[0] ? RL_EDEGENERATE : RL_OK;
  }
  unsigned long long* key = reinterpret_cast<unsigned long long*>(base);
  int* d_flag = degenerate_dev ? degenerate_dev : reinterpret_cast<int*>(base + 8);
  double* d_logw = logw ? logw : reinterpret_cast<double*>(base + 64);
  double* d_w = weight ? weight : reinterpret_cast<double*>(base + 64 + 8 * n);
  double* partial = reinterpret_cast<double*>(base + 64 + 16 * n);
  RL_CK(cudaMemsetAsync(key, 0, 8, st));
  RL_TRY(sensor_logw_launch(c, const_cast<double*>(px), const_cast<double*>(py),
                            const_cast<double*>(pt), n, scan, nbeams, fov, params, table, zdim,
                            inv_res, d_logw, nullptr, key, st, nullptr, nullptr, nullptr));
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
