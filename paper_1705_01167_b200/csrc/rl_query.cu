// Batched and single CDDT queries on sm_100a (K3): the split pipeline for large
// f32 batches (phase 1, near field, window passes), the single-kernel form for
// everything else, and the query entry points of the C ABI (include/rl_cddt.h).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <type_traits>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include <vector>

#include "rl_common.cuh"

namespace rl {

// ---------------------------------------------------------------------------
// K3: batched casts.
//
// Monolithic form (f64 / hit-cell / resolving-index outputs, and batches
// below kDeferMinQueries, 786k): one thread per query, grid-stride, a single full wave
// sized by the occupancy calculator (4 x 256-thread CTAs per SM at 64 regs).
template <class T, class I, bool HIT, bool RES>
__global__ void __launch_bounds__(256, 4) k_cast(CddtView c, const T* __restrict__ qx,
                                                 const T* __restrict__ qy,
                                                 const T* __restrict__ qt, T* __restrict__ out,
                                                 int32_t* __restrict__ hit,
                                                 int64_t* __restrict__ res_row,
                                                 int32_t* __restrict__ res_idx, I n) {
  for (I i = I(blockIdx.x) * I(blockDim.x) + I(threadIdx.x); i < n;
       i += I(gridDim.x) * I(blockDim.x)) {
    // query streams are touched once: evict-first so the structure stays in L2
    const double x = double(__ldcs(qx + i)), y = double(__ldcs(qy + i));
    const double th = normalize_angle_2pi(double(__ldcs(qt + i)));  // RayQuery ctor, raycast.hpp:47
    CastOut o;
    const double r = directional_cast(c, x, y, direction_index(th, c.K), o, HIT);
    if (out) __stcs(out + i, T(r));
    if (HIT && hit) hit[i] = o.hit;
    if (RES) {
      if (res_row) res_row[i] = o.res_idx >= 0 ? int64_t(o.res_g) : -1;
      if (res_idx) res_idx[i] = o.res_idx;
    }
  }
}

// Deferred-walk form (f32 ranges only, >= kDeferMinQueries; the bench path).
// About a third of the queries need a RayWalker (a near-field walk or a
// verification window). Run inline, those walks execute with ~5 of 32 lanes
// active and cost half the kernel time (profiles/r01/ncu_k_cast_v3.txt).
// Phase 1 settles every query that needs no walker with uniform control flow
// and queues the rest — with the CSR row and the pending candidate — through
// a per-CTA shared-memory compaction (one global atomic per CTA iteration).
// The window passes (k_walk_pass) resume exactly there, every lane walking;
// near-field queries are redone in full by k_cast_near. Records are streamed
// evict-first past L2.
struct __align__(32) WalkRecord {
  float x, y, t;
  uint32_t i, lo, n;
  int32_t idx, pad;
};

// A 32-byte record moved by one 256-bit evict-first access (LDG/STG.E.EF.256):
// one L1 wavefront per lane instead of two.
__device__ __forceinline__ void ld256_cs(const void* p, float4& a, float4& b) {
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void st256_cs(void* p, const float4& a, const float4& b) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.x),
               "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
               : "memory");
}

#ifndef RL_P1_CTAS
#define RL_P1_CTAS 8  // resident 256-thread equivalents per SM the register budget of phase 1 targets (32 registers)
#endif
#ifndef RL_WIN_CAPS
#define RL_WIN_CAPS 1, 2, 4  // windows per query in each capped window pass; a last pass finishes
#endif
#ifndef RL_CONT_A_DIV
#define RL_CONT_A_DIV 4  // continuation queue capacities: n / DIV records
#endif
#ifndef RL_CONT_B_DIV
#define RL_CONT_B_DIV 16
#endif
#ifndef RL_P1_THREADS
#define RL_P1_THREADS 64  // small CTAs: the per-iteration compaction barrier waits for fewer warps
#endif
constexpr int kP1Threads = RL_P1_THREADS, kP1Warps = kP1Threads / 32;
template <class T>
__global__ void __launch_bounds__(kP1Threads, RL_P1_CTAS * 256 / kP1Threads) k_cast_defer_p1(
    CddtView c, const T* __restrict__ qx, const T* __restrict__ qy, const T* __restrict__ qt,
    T* __restrict__ out, uint32_t n, WalkRecord* __restrict__ q, unsigned* __restrict__ qn) {
  // queue layout: window records grow up from q[0], near-field records down
  // from q[n-1]; qn[0], qn[1] count them
  __shared__ unsigned cnt_s[2][kP1Warps], base_s[2];
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < n; b0 += gridDim.x * blockDim.x) {
    const uint32_t i = b0 + threadIdx.x;
    {  // next iteration's query stream into L2 while this one waits on the structure
      const uint32_t nx = i + gridDim.x * blockDim.x;
      if (nx < n && (threadIdx.x & 31) < 3) {
        const T* base = (threadIdx.x & 31) == 0 ? qx : ((threadIdx.x & 31) == 1 ? qy : qt);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (nx & ~31u)));
      }
    }
    bool defer = false;
    WalkRecord rec{};  // defined on every path: no stale fields to keep (or spill) across iterations
    if (i < n) {
      rec.x = __ldcs(qx + i);
      rec.y = __ldcs(qy + i);
      rec.t = __ldcs(qt + i);
      rec.i = i;
      const double th = normalize_angle_2pi(double(rec.t));
      double r;
      WalkDefer def;
      if (directional_cast_p1(c, rec.x, rec.y, direction_index(th, c.K), &r, &def)) {
        __stcs(out + i, T(r));
      } else {
        defer = true;
        rec.lo = def.lo;
        rec.n = def.n;
        rec.idx = def.idx;
        rec.pad = __float_as_int(def.cval);  // windows: the candidate's zero point
      }
    }
    const bool near = defer && rec.idx < 0, win = defer && !near;
    const unsigned bw = __ballot_sync(0xffffffffu, win), bn = __ballot_sync(0xffffffffu, near);
    if (lane == 0) {
      cnt_s[0][wid] = __popc(bw);
      cnt_s[1][wid] = __popc(bn);
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      unsigned tot = 0;
      for (int w = 0; w < kP1Warps; w++) {
        const unsigned k = cnt_s[threadIdx.x][w];
        cnt_s[threadIdx.x][w] = tot;
        tot += k;
      }
      base_s[threadIdx.x] = tot ? atomicAdd(qn + threadIdx.x, tot) : 0u;
    }
    __syncthreads();
    if (defer) {
      const unsigned below = (1u << lane) - 1;
      const size_t slot = win ? base_s[0] + cnt_s[0][wid] + __popc(bw & below)
                              : n - 1 - (base_s[1] + cnt_s[1][wid] + __popc(bn & below));
      // window records grow up, near-field records down: together at most n
      RL_DCHECK(c, slot < n && base_s[0] + base_s[1] <= n, 10);
      const float4* src = reinterpret_cast<const float4*>(&rec);
      st256_cs(q + slot, src[0], src[1]);
    }
    __syncthreads();
  }
}

// Window passes. A query needing many verification windows (a ray grazing a
// wall meets one failing candidate per wall cell) holds its whole warp in a
// single resume-to-completion pass; instead, pass k scans at most cap_k
// windows per query and queues the unfinished ones, with the candidate loop's
// state, for pass k+1 (the last pass has no cap). Each pass is a full-width
// walk over a shrinking queue.
struct __align__(16) ContRecord {
  float x, y, t;
  uint32_t i, lo, n;
  int32_t idx, cx, cy, a;  // a: the query's direction index (not recomputed per pass)
  double wt;
};

#ifndef RL_WALK_THREADS
#define RL_WALK_THREADS 64  // small CTAs: cheap compaction barriers
#endif
constexpr int kWalkThreads = RL_WALK_THREADS;
// resident CTAs per SM the walk kernels' register budget targets: 18 x 64
// threads at 56 registers without spills (16 at 60-62 registers: +0.4 % per
// step; 20 at 48 registers spills: +3 %)
#ifdef RL_P2_MINCTAS
constexpr int kWalkMinCtas = RL_P2_MINCTAS;
#else
constexpr int kWalkMinCtas = 18;
#endif

// out-of-line: the rare overflow path must not add to the pass's registers
__device__ __noinline__ double finish_windows(const CddtView& c, double x, double y, int a,
                                              WinState s) {
  double res;
  resume_windows<false>(c, x, y, a, s, 0x7fffffff, &res);
  return res;
}

template <class T, bool CONT, bool LAST>
__global__ void __launch_bounds__(kWalkThreads, kWalkMinCtas) k_walk_pass(
    CddtView c, const void* __restrict__ in, const unsigned* __restrict__ in_count,
    uint32_t in_cap, int cap, ContRecord* __restrict__ oq, unsigned* __restrict__ out_count,
    uint32_t out_cap, T* __restrict__ out) {
  __shared__ unsigned cnt_s[kWalkThreads / 32], base_s;
  // the producer counts every continuation, stored or (queue full) finished
  const unsigned m = min(*in_count, in_cap);
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (unsigned b0 = blockIdx.x * blockDim.x; b0 < m; b0 += gridDim.x * blockDim.x) {
    const unsigned k = b0 + threadIdx.x;
    {  // next iteration's record into L2
      const unsigned nk = k + gridDim.x * blockDim.x;
      if (nk < m) {
        const char* rp = CONT ? reinterpret_cast<const char*>(static_cast<const ContRecord*>(in) + nk)
                              : reinterpret_cast<const char*>(static_cast<const WalkRecord*>(in) + nk);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
      }
    }
    bool defer = false;
    float fx = 0.f, fy = 0.f, ft = 0.f;
    uint32_t qi = 0;
    WinState s{};
    int a = 0;
    if (k < m) {
      if (CONT) {
        const float4* src = reinterpret_cast<const float4*>(static_cast<const ContRecord*>(in) + k);
        const float4 w0 = __ldcs(src), w1 = __ldcs(src + 1), w2 = __ldcs(src + 2);
        fx = w0.x;
        fy = w0.y;
        ft = w0.z;
        qi = __float_as_uint(w0.w);
        s = WinState{__float_as_uint(w1.x), __float_as_uint(w1.y), __float_as_int(w1.z),
                     __float_as_int(w1.w), __float_as_int(w2.x),
                     __hiloint2double(__float_as_int(w2.w), __float_as_int(w2.z)), 0.f};
        a = __float_as_int(w2.y);
      } else {
        float4 w0, w1;
        ld256_cs(static_cast<const WalkRecord*>(in) + k, w0, w1);
        fx = w0.x;
        fy = w0.y;
        ft = w0.z;
        qi = __float_as_uint(w0.w);
        s = WinState{__float_as_uint(w1.x), __float_as_uint(w1.y), __float_as_int(w1.z), 0, 0, 0.0,
                     w1.w};
      }
      if (!CONT) a = direction_index(normalize_angle_2pi(double(ft)), c.K);
      double res;
      if (resume_windows<!CONT>(c, double(fx), double(fy), a, s, LAST ? 0x7fffffff : cap, &res))
        __stcs(out + qi, T(res));
      else
        defer = true;
    }
    if (LAST) continue;
    const unsigned bal = __ballot_sync(0xffffffffu, defer);
    if (lane == 0) cnt_s[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w = 0; w < kWalkThreads / 32; w++) {
        const unsigned q = cnt_s[w];
        cnt_s[w] = tot;
        tot += q;
      }
      base_s = tot ? atomicAdd(out_count, tot) : 0u;
    }
    __syncthreads();
    if (defer) {
      const unsigned slot = base_s + cnt_s[wid] + __popc(bal & ((1u << lane) - 1));
      RL_DCHECK(c, qi < 0x80000000u && k < in_cap, 11);
      if (slot < out_cap) {  // ContRecord layout, as three 16-byte stores
        float4* dst = reinterpret_cast<float4*>(oq + slot);
        __stcs(dst, make_float4(fx, fy, ft, __uint_as_float(qi)));
        __stcs(dst + 1, make_float4(__uint_as_float(s.lo), __uint_as_float(s.n),
                                    __int_as_float(s.idx), __int_as_float(s.cx)));
        __stcs(dst + 2, make_float4(__int_as_float(s.cy), __int_as_float(a),
                                    __int_as_float(__double2loint(s.t)),
                                    __int_as_float(__double2hiint(s.t))));
      } else {  // queue full: finish here
        __stcs(out + qi, T(finish_windows(c, double(fx), double(fy), a, s)));
      }
    }
    __syncthreads();
  }
}

// The finishing pass, warp-cooperative. What reaches it are the rays grazing
// walls: few records, but chains of tens to hundreds of verification windows,
// so a lane-per-record pass lasts as long as its longest chain (45 us whether
// the batch has 1M or 50M queries). Each lane first scans up to `cap` more
// windows of its own record; a record still unfinished is then taken by the
// whole warp, 32 candidates at a time (resume_coop: every candidate's verdict
// is a pure function of the candidate, the first non-clean one in candidate
// order decides, exactly as the sequential loop does).
#ifndef RL_LAST_COOP
#define RL_LAST_COOP 1
#endif
#ifndef RL_LAST_COOP_CAP
#define RL_LAST_COOP_CAP 8  // 0 / 2 / 4: slower (whole warps spent on short chains); 12-40: equal to slower
#endif
template <class T>
__global__ void __launch_bounds__(kWalkThreads, kWalkMinCtas) k_walk_last_coop(
    CddtView c, const ContRecord* __restrict__ in, const unsigned* __restrict__ in_count,
    uint32_t in_cap, int cap, T* __restrict__ out) {
  const unsigned m = min(*in_count, in_cap);
  const unsigned lane = threadIdx.x & 31;
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned warps = (gridDim.x * blockDim.x) >> 5;
  for (unsigned b0 = warp * 32u; b0 < m; b0 += warps * 32u) {
    const unsigned k = b0 + lane;
    bool open = false;
    float fx = 0.f, fy = 0.f;
    uint32_t qi = 0;
    WinState s{};
    int a = 0;
    if (k < m) {
      const float4* src = reinterpret_cast<const float4*>(in + k);
      const float4 w0 = __ldcs(src), w1 = __ldcs(src + 1), w2 = __ldcs(src + 2);
      fx = w0.x;
      fy = w0.y;
      qi = __float_as_uint(w0.w);
      s = WinState{__float_as_uint(w1.x), __float_as_uint(w1.y), __float_as_int(w1.z),
                   __float_as_int(w1.w), __float_as_int(w2.x),
                   __hiloint2double(__float_as_int(w2.w), __float_as_int(w2.z)), 0.f};
      a = __float_as_int(w2.y);
      double res;
      if (resume_windows<false>(c, double(fx), double(fy), a, s, cap, &res))
        __stcs(out + qi, T(res));
      else
        open = true;
    }
    unsigned todo = __ballot_sync(0xffffffffu, open);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const float x = __shfl_sync(0xffffffffu, fx, j), y = __shfl_sync(0xffffffffu, fy, j);
      const int aj = __shfl_sync(0xffffffffu, a, j), ij = __shfl_sync(0xffffffffu, s.idx, j);
      const uint32_t oj = __shfl_sync(0xffffffffu, qi, j);
      const double r = resume_coop(c, double(x), double(y), aj, ij);
      if (lane == 0) __stcs(out + oj, T(r));
    }
  }
}

// Near-field records (origin not clear): near-field walk, search and landing
// probes here; queries that need a verification window join the window
// passes as continuations (queue A, after pass 0's own).
template <class T>
__global__ void __launch_bounds__(kWalkThreads, kWalkMinCtas) k_cast_near(
    CddtView c, const WalkRecord* __restrict__ q, const unsigned* __restrict__ qn, uint32_t n,
    ContRecord* __restrict__ oq, unsigned* __restrict__ out_count, uint32_t out_cap,
    T* __restrict__ out) {
  __shared__ unsigned cnt_s[kWalkThreads / 32], base_s;
  const unsigned m = qn[1];
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (unsigned b0 = blockIdx.x * blockDim.x; b0 < m; b0 += gridDim.x * blockDim.x) {
    const unsigned k = b0 + threadIdx.x;
    bool defer = false;
    float4 w0 = make_float4(0.f, 0.f, 0.f, 0.f);
    WinState s{};
    int a = 0;
    if (k < m) {
      RL_DCHECK(c, k < n, 12);
      w0 = __ldcs(reinterpret_cast<const float4*>(q + (n - 1 - k)));  // x, y, theta, index
      a = direction_index(normalize_angle_2pi(double(w0.z)), c.K);
      double res;
      if (near_cast_p1(c, double(w0.x), double(w0.y), a, &res, &s))
        __stcs(out + __float_as_uint(w0.w), T(res));
      else
        defer = true;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, defer);
    if (lane == 0) cnt_s[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int w = 0; w < kWalkThreads / 32; w++) {
        const unsigned x = cnt_s[w];
        cnt_s[w] = tot;
        tot += x;
      }
      base_s = tot ? atomicAdd(out_count, tot) : 0u;
    }
    __syncthreads();
    if (defer) {
      const unsigned slot = base_s + cnt_s[wid] + __popc(bal & ((1u << lane) - 1));
      if (slot < out_cap) {
        float4* dst = reinterpret_cast<float4*>(oq + slot);
        __stcs(dst, w0);
        __stcs(dst + 1, make_float4(__uint_as_float(s.lo), __uint_as_float(s.n),
                                    __int_as_float(s.idx), __int_as_float(s.cx)));
        __stcs(dst + 2, make_float4(__int_as_float(s.cy), __int_as_float(a),
                                    __int_as_float(__double2loint(s.t)),
                                    __int_as_float(__double2hiint(s.t))));
      } else {  // queue full: finish here
        __stcs(out + __float_as_uint(w0.w),
               T(finish_windows(c, double(w0.x), double(w0.y), a, s)));
      }
    }
    __syncthreads();
  }
}

// CTAs per SM for a kernel at 256 threads (one full wave, no partial tail).
template <class K>
static int resident_ctas(K kernel) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
  return std::max(per_sm, 1);
}

template <class T, class I, bool HIT, bool RES>
static void launch_k_cast(const CddtView& v, const T* x, const T* y, const T* t, T* out,
                          int32_t* hit, int64_t* rr, int32_t* ri, size_t n, cudaStream_t st) {
  static const int per_sm = resident_ctas(k_cast<T, I, HIT, RES>);
  const size_t b = std::max<size_t>(1, std::min((n + 255) / 256, size_t(sm_count()) * per_sm));
  k_cast<T, I, HIT, RES><<<int(b), 256, 0, st>>>(v, x, y, t, out, hit, rr, ri, I(n));
}

// Batch-size plan of the range-only f32 cast (measured on B200, configs 2 and 3):
//   n <  kDeferMinQueries   single kernel (the split pipeline's six dependent launches cost more)
//   n >= kDeferMinQueries   split pipeline; with window caps {2} (one capped pass, then the
//                           finishing pass) while a pipeline holds fewer than kShortPlanMax
//                           queries, {1, 2, 4} above
//   n >= kTwoPipeMin        two pipelines over the halves of the batch
// RL_DEFER_MIN / RL_TWO_PIPE_MIN / RL_SHORT_PLAN_MAX (environment) override them for A/B runs.
static size_t env_size(const char* name, size_t dflt) {
  const char* e = std::getenv(name);
  return e ? size_t(std::strtoull(e, nullptr, 10)) : dflt;
}
static const size_t kDeferMinQueries = env_size("RL_DEFER_MIN", size_t(3) << 18);   // 786k
static const size_t kTwoPipeMin = env_size("RL_TWO_PIPE_MIN", size_t(1) << 22);     // 4.2M
static const size_t kShortPlanMax = env_size("RL_SHORT_PLAN_MAX", size_t(1) << 23);  // per pipeline

// Dispatch of the batched cast kernels for the device-pointer entry points.
template <class T>
static int launch_cast(const rl_cddt* c, const T* x, const T* y, const T* t, T* out,
                       int32_t* hit, int64_t* rr, int32_t* ri, size_t n, cudaStream_t st,
                       bool split = true) {
  const CddtView v = c->view();
  const bool small = n < (size_t(1) << 31);
#ifndef RL_DEFER_MAX_LOG2
#define RL_DEFER_MAX_LOG2 28
#endif
  constexpr size_t kDeferMaxQueries = size_t(1) << RL_DEFER_MAX_LOG2;  // bounds the workspace (~12 GB)
  if (!rr && !ri && !hit && n > kDeferMaxQueries) {
    for (size_t off = 0; off < n; off += kDeferMaxQueries) {
      const size_t m = std::min(kDeferMaxQueries, n - off);
      RL_TRY(launch_cast<T>(c, x + off, y + off, t + off, out + off, nullptr, nullptr, nullptr,
                            m, st));
    }
    return RL_OK;
  }
  static const int parts = [] {
    const char* e = std::getenv("RL_SPLIT_PARTS");
    return e ? std::max(1, std::atoi(e)) : 2;
  }();
  // the split pipeline's records hold the query as floats: f32 batches only
  // (f64 queries need not be float-representable; they take k_cast)
  constexpr bool kF32 = std::is_same<T, float>::value;
  if (kF32 && split && parts > 1 && !rr && !ri && !hit && small && n >= kTwoPipeMin &&
      n >= kDeferMinQueries * parts) {
    // two independent pipelines over the halves of the batch, on the caller's
    // stream and a forked one: the late, thinly occupied window passes of one
    // overlap the other's phase 1
    struct Part {
      cudaStream_t s = nullptr;
      cudaEvent_t fork = nullptr, join = nullptr;
    };
    static thread_local Part part[64];
    int dev = 0;
    RL_CK(cudaGetDevice(&dev));
    Part& pp = part[dev & 63];
    if (!pp.s) {
      RL_CK(cudaStreamCreateWithFlags(&pp.s, cudaStreamNonBlocking));
      RL_CK(cudaEventCreateWithFlags(&pp.fork, cudaEventDisableTiming));
      RL_CK(cudaEventCreateWithFlags(&pp.join, cudaEventDisableTiming));
    }
    RL_CK(cudaEventRecord(pp.fork, st));
    RL_CK(cudaStreamWaitEvent(pp.s, pp.fork, 0));
    for (int k = 0; k < parts; k++) {  // chunks alternate between the two streams
      const size_t a = n * size_t(k) / size_t(parts), b = n * size_t(k + 1) / size_t(parts);
      RL_TRY(launch_cast<T>(c, x + a, y + a, t + a, out + a, nullptr, nullptr, nullptr, b - a,
                            (k & 1) ? pp.s : st, false));
    }
    RL_CK(cudaEventRecord(pp.join, pp.s));
    RL_CK(cudaStreamWaitEvent(st, pp.join, 0));
    return RL_OK;
  }
  if constexpr (kF32) if (!rr && !ri && !hit && small && n >= kDeferMinQueries) {
    // stream-ordered scratch: concurrent batches on other streams (e.g. the
    // pipelined host path) each get their own queue; the pool keeps the
    // memory reserved, so steady-state allocation is free
      // workspace: counters | n walk records (windows up from 0, near field down
    // from n-1) | continuation queues A and B (the window passes alternate)
    // (RL_CDDT_CONT_CAP overrides the queue capacity: a test hook for the
    // queue-full path)
    static const size_t cap_env = [] {
      const char* e = std::getenv("RL_CDDT_CONT_CAP");
      return e ? size_t(std::strtoull(e, nullptr, 10)) : size_t(0);
    }();
    // capped window passes of this pipeline; one more pass finishes
    // (RL_WIN_CAPS_ENV / RL_SHORT_CAPS_ENV: decimal digits, e.g. 124 -> {1, 2, 4}, for A/B runs)
    struct Caps {
      int n = 0, v[4] = {0, 0, 0, 0};
      Caps(const char* name, std::initializer_list<int> dflt) {
        const char* e = std::getenv(name);
        if (e && *e) {
          for (const char* q = e; *q && n < 4; q++) v[n++] = *q - '0';
        } else {
          for (int d : dflt) v[n++] = d;
        }
      }
    };
    static const Caps caps_full("RL_WIN_CAPS_ENV", {RL_WIN_CAPS}), caps_short("RL_SHORT_CAPS_ENV", {2});
    const bool short_plan = n < kShortPlanMax;
    const int* kCaps = short_plan ? caps_short.v : caps_full.v;
    const int kPasses = short_plan ? caps_short.n : caps_full.n;
    constexpr int kMaxPasses = 4;
    const size_t cap_a = cap_env ? cap_env : std::max<size_t>(n / RL_CONT_A_DIV, size_t(1) << 16);
    const size_t cap_b = cap_env ? cap_env : std::max<size_t>(n / RL_CONT_B_DIV, size_t(1) << 16);
    uint8_t* ws = nullptr;
    RL_TRY(scratch_alloc(reinterpret_cast<void**>(&ws),
                          256 + sizeof(WalkRecord) * n + sizeof(ContRecord) * (cap_a + cap_b),
                          st));
    unsigned* qn = reinterpret_cast<unsigned*>(ws);  // windows, near, one per capped pass
    WalkRecord* q = reinterpret_cast<WalkRecord*>(ws + 256);
    ContRecord* qa = reinterpret_cast<ContRecord*>(q + n);
    ContRecord* qb = qa + cap_a;
    static const int p1 = [] {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cast_defer_p1<T>, kP1Threads, 0);
      return std::max(per_sm, 1);
    }();
    auto walk_ctas = [](auto kernel) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kWalkThreads, 0);
      return std::max(per_sm, 1);
    };
    static const int pw0 = walk_ctas(k_walk_pass<T, false, false>);
    static const int pwc = walk_ctas(k_walk_pass<T, true, false>);
    static const int pwl = walk_ctas(k_walk_pass<T, true, true>);
    static const int pn = walk_ctas(k_cast_near<T>);
    RL_CK(cudaMemsetAsync(qn, 0, (2 + kMaxPasses) * sizeof(unsigned), st));
    const size_t b1 = std::max<size_t>(
        1, std::min((n + kP1Threads - 1) / kP1Threads, size_t(sm_count()) * p1));
    k_cast_defer_p1<T><<<int(b1), kP1Threads, 0, st>>>(v, x, y, t, out, uint32_t(n), q, qn);
    // the near-field kernel and window pass 0 read disjoint ends of the record
    // queue and both append to queue A: they run side by side (fork / join)
    struct Side {
      cudaStream_t s = nullptr;
      cudaEvent_t fork = nullptr, join = nullptr;
    };
    static thread_local Side side[64];
    int dev = 0;
    RL_CK(cudaGetDevice(&dev));
    Side& sd = side[dev & 63];
    if (!sd.s) {
      RL_CK(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
      RL_CK(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming));
      RL_CK(cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming));
    }
    RL_CK(cudaEventRecord(sd.fork, st));
    RL_CK(cudaStreamWaitEvent(sd.s, sd.fork, 0));
    k_cast_near<T><<<sm_count() * pn, kWalkThreads, 0, sd.s>>>(v, q, qn, uint32_t(n), qa, qn + 2,
                                                               uint32_t(cap_a), out);
    RL_CK(cudaEventRecord(sd.join, sd.s));
    k_walk_pass<T, false, false><<<sm_count() * pw0, kWalkThreads, 0, st>>>(
        v, q, qn, uint32_t(n), kCaps[0], qa, qn + 2, uint32_t(cap_a), out);
    RL_CK(cudaStreamWaitEvent(st, sd.join, 0));
    for (int p = 1; p < kPasses; p++) {  // queue p-1 -> queue p (A, B, A, ...)
      const bool from_a = (p & 1) != 0;
      k_walk_pass<T, true, false><<<sm_count() * pwc, kWalkThreads, 0, st>>>(
          v, from_a ? qa : qb, qn + 1 + p, uint32_t(from_a ? cap_a : cap_b), kCaps[p],
          from_a ? qb : qa, qn + 2 + p, uint32_t(from_a ? cap_b : cap_a), out);
    }
    const bool last_a = (kPasses & 1) != 0;
#if RL_LAST_COOP
    static const int pwk = walk_ctas(k_walk_last_coop<T>);
    k_walk_last_coop<T><<<sm_count() * pwk, kWalkThreads, 0, st>>>(
        v, last_a ? qa : qb, qn + 1 + kPasses, uint32_t(last_a ? cap_a : cap_b),
        RL_LAST_COOP_CAP, out);
#else
    k_walk_pass<T, true, true><<<sm_count() * pwl, kWalkThreads, 0, st>>>(
        v, last_a ? qa : qb, qn + 1 + kPasses, uint32_t(last_a ? cap_a : cap_b), 0, nullptr,
        nullptr, 0, out);
#endif
#ifdef RL_DEBUG_COUNTS
    {
      unsigned h[2 + kMaxPasses];
      cudaMemcpyAsync(h, qn, (2 + kPasses) * sizeof(unsigned), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "counts n=%zu windows=%u near=%u", n, h[0], h[1]);
      for (int p = 0; p < kPasses; p++) fprintf(stderr, " after pass %d: %u", p, h[2 + p]);
      fprintf(stderr, "\n");
    }
#endif
    RL_TRY(scratch_free(ws, st));
    return RL_OK;
  }
  if (rr || ri) {
    launch_k_cast<T, size_t, true, true>(v, x, y, t, out, hit, rr, ri, n, st);
  } else if (hit) {
    if (small)
      launch_k_cast<T, uint32_t, true, false>(v, x, y, t, out, hit, rr, ri, n, st);
    else
      launch_k_cast<T, size_t, true, false>(v, x, y, t, out, hit, rr, ri, n, st);
  } else {
    if (small)
      launch_k_cast<T, uint32_t, false, false>(v, x, y, t, out, hit, rr, ri, n, st);
    else
      launch_k_cast<T, size_t, false, false>(v, x, y, t, out, hit, rr, ri, n, st);
  }
  return RL_OK;
}

__global__ void k_directional(CddtView c, const double* __restrict__ x,
                              const double* __restrict__ y, const int32_t* __restrict__ a,
                              double* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    CastOut o;
    out[i] = directional_cast(c, x[i], y[i], a[i], o, false);
  }
}

__global__ void k_single(CddtView c, double x, double y, double theta, int pair,
                         double* __restrict__ out) {
  const double th = normalize_angle_2pi(theta);
  const int a = direction_index(th, c.K);
  CastOut o;
  out[0] = directional_cast(c, x, y, a, o, false);
  if (pair) out[1] = directional_cast(c, x, y, (a + c.K / 2) % c.K, o);  // cddt.cpp:275-279
}

// The per-query loop of run_batches (proj/src/bench.cpp:86-106) over an array
// of RayQuery {double x, y, theta} (raycast.hpp:42-49), read in place.
__global__ void __launch_bounds__(256, 4) k_cast_queries(CddtView c, const double* __restrict__ q,
                                                         double* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const double x = __ldcs(q + 3 * i), y = __ldcs(q + 3 * i + 1);
    const double th = normalize_angle_2pi(__ldcs(q + 3 * i + 2));  // RayQuery ctor (idempotent)
    CastOut o;
    __stcs(out + i, directional_cast(c, x, y, direction_index(th, c.K), o, false));
  }
}

static int dir_blocks(size_t n) {
  size_t b = (n + 255) / 256;
  return int(std::max<size_t>(1, std::min(b, size_t(sm_count()) * 8)));
}

}  // namespace rl

using namespace rl;

// ---------------------------------------------------------------------------
// Pageable host buffers (what a reference caller holds: std::vector<RayQuery>
// fields, numpy arrays). cudaMemcpyAsync from pageable memory is staged by the
// driver through one bounce buffer, synchronously: 134 ms per 100M queries
// against 24 ms from pinned memory. Here the chunks are staged through a ring
// of pinned buffers by a few host threads (plain memcpy) while the DMA engines
// and the kernels work on the other lanes' chunks.
constexpr size_t kStageMinQueries = size_t(1) << 20;  // below: one driver-staged copy is as fast

// true when the DMA engines can read/write the range directly (page-locked,
// registered, managed or device memory)
static bool dma_direct(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type != cudaMemoryTypeUnregistered;
}

struct CopySeg {
  void* dst;
  const void* src;
  size_t bytes;
};

// memcpy with non-temporal stores: the destination is not read for ownership
// and does not displace the source from the caches (a staging copy is written
// once and read by the DMA engine, or by the caller much later)
static void stream_copy(char* dst, const char* src, size_t bytes) {
#if defined(__x86_64__) && defined(__SSE2__)
  static const bool nt = [] {
    const char* e = std::getenv("RL_HOST_NT");
    return e ? std::atoi(e) != 0 : true;
  }();
  if (nt && bytes >= 4096) {
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    bytes -= head;
    size_t k = 0;
    for (; k + 64 <= bytes; k += 64) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 16));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 32));
      const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 48), d);
    }
    _mm_sfence();
    std::memcpy(dst + k, src + k, bytes - k);
    return;
  }
#endif
  std::memcpy(dst, src, bytes);
}

// the segments copied by `threads` host threads, each taking an equal slice of
// every segment (the caller's thread is one of them)
static void parallel_copy(const std::vector<CopySeg>& segs, int threads) {
  auto work = [&segs, threads](int t) {
    for (const CopySeg& g : segs) {
      const size_t per = ((g.bytes + size_t(threads) - 1) / size_t(threads) + 63) & ~size_t(63);
      const size_t a = std::min(g.bytes, per * size_t(t)), b = std::min(g.bytes, a + per);
      if (b > a) stream_copy(static_cast<char*>(g.dst) + a, static_cast<const char*>(g.src) + a, b - a);
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(size_t(threads > 1 ? threads - 1 : 0));
  for (int t = 1; t < threads; t++) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
}

static int cast_batch_staged(rl_cddt* c, const float* x, const float* y, const float* theta,
                             float* out, size_t n) {
  constexpr int NSTREAM = 3;
  static const int threads = [] {
    const char* e = std::getenv("RL_HOST_COPY_THREADS");
    const int hw = int(std::thread::hardware_concurrency());
    return std::max(1, e ? std::atoi(e) : std::min(8, hw > 1 ? hw / 2 : 1));
  }();
  static const size_t chunk_max = [] {
    const char* e = std::getenv("RL_HOST_STAGE_CHUNK_LOG2");
    return size_t(1) << (e ? std::atoi(e) : 22);  // 4M queries (two pipelines of 2M each)
  }();
  const size_t chunk = std::min(n, chunk_max);
  struct Lane {
    cudaStream_t s = nullptr;
    DevBuf<float> dev;      // x | y | theta | out
    float* pin = nullptr;   // the same layout in page-locked host memory
    size_t pend_off = 0, pend_m = 0;  // results waiting in pin's out block
    ~Lane() {
      if (pin) cudaFreeHost(pin);
      if (s) cudaStreamDestroy(s);
    }
  };
  static thread_local std::vector<Lane> lanes;  // reused across calls on this thread
  static thread_local size_t lane_chunk = 0;
  static thread_local int lane_dev = -1;
  if (lanes.empty() || lane_chunk < chunk || lane_dev != c->dev) {
    lanes.clear();
    lanes = std::vector<Lane>(NSTREAM);
    lane_chunk = 0;
    for (auto& l : lanes) {
      RL_CK(cudaStreamCreateWithFlags(&l.s, cudaStreamNonBlocking));
      RL_TRY(l.dev.alloc(4 * chunk));
      RL_CK(cudaHostAlloc(reinterpret_cast<void**>(&l.pin), 4 * chunk * sizeof(float),
                          cudaHostAllocDefault));
    }
    lane_chunk = chunk;
    lane_dev = c->dev;
  }
  for (auto& l : lanes) l.pend_m = 0;
  cudaEvent_t ready;
  RL_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  struct EventGuard {  // released on every return path
    cudaEvent_t e;
    ~EventGuard() { cudaEventDestroy(e); }
  } ready_guard{ready};
  RL_CK(cudaEventRecord(ready, c->stream));  // order after pending structure work
  const size_t stride = lane_chunk;
  std::vector<CopySeg> segs;
  size_t k = 0;
  for (size_t off = 0; off < n; k++) {
    // the first chunks are small so the link starts early; the rest are full
    const size_t m = std::min(n - off, k < 2 ? std::max<size_t>(chunk >> (2 - k), 1) : chunk);
    Lane& l = lanes[k % NSTREAM];
    segs.clear();
    if (l.pend_m) {  // the lane's previous results leave its pinned block first
      RL_CK(cudaStreamSynchronize(l.s));
      segs.push_back({out + l.pend_off, l.pin + 3 * stride, l.pend_m * sizeof(float)});
    }
    segs.push_back({l.pin, x + off, m * sizeof(float)});
    segs.push_back({l.pin + stride, y + off, m * sizeof(float)});
    segs.push_back({l.pin + 2 * stride, theta + off, m * sizeof(float)});
    parallel_copy(segs, threads);
    float* dx = l.dev.p;
    RL_CK(cudaStreamWaitEvent(l.s, ready, 0));
    if (m == stride) {  // x | y | theta are contiguous: one copy
      RL_CK(cudaMemcpyAsync(dx, l.pin, 3 * m * sizeof(float), cudaMemcpyHostToDevice, l.s));
    } else {
      for (int a = 0; a < 3; a++)
        RL_CK(cudaMemcpyAsync(dx + a * stride, l.pin + a * stride, m * sizeof(float),
                              cudaMemcpyHostToDevice, l.s));
    }
    RL_TRY(launch_cast<float>(c, dx, dx + stride, dx + 2 * stride, dx + 3 * stride, nullptr,
                              nullptr, nullptr, m, l.s, true));
    RL_CK(cudaGetLastError());
    RL_CK(cudaMemcpyAsync(l.pin + 3 * stride, dx + 3 * stride, m * sizeof(float),
                          cudaMemcpyDeviceToHost, l.s));
    l.pend_off = off;
    l.pend_m = m;
    off += m;
  }
  // drain in submission order
  for (size_t j = (k >= NSTREAM ? k - NSTREAM : 0); j < k; j++) {
    Lane& l = lanes[j % NSTREAM];
    if (!l.pend_m) continue;
    RL_CK(cudaStreamSynchronize(l.s));
    parallel_copy({{out + l.pend_off, l.pin + 3 * stride, l.pend_m * sizeof(float)}}, threads);
    l.pend_m = 0;
  }
  return RL_OK;
}

// rl_cddt_cast_queries_host: chunks of the RayQuery array go host -> device,
// through k_cast_queries, and their ranges back, over three streams; pageable
// arrays (a std::vector<RayQuery>) are staged through pinned buffers by the
// host threads like cast_batch_staged's.
static int cast_queries_pipeline(rl_cddt* c, const double* q, double* out, size_t n) {
  constexpr int NSTREAM = 3;
  static const int threads = [] {
    const char* e = std::getenv("RL_HOST_COPY_THREADS");
    const int hw = int(std::thread::hardware_concurrency());
    return std::max(1, e ? std::atoi(e) : std::min(8, hw > 1 ? hw / 2 : 1));
  }();
  const size_t chunk = std::min(n, size_t(1) << 21);  // 2M queries: 48 MB in, 16 MB out
  const bool in_direct = dma_direct(q), out_direct = dma_direct(out);
  struct Lane {
    cudaStream_t s = nullptr;
    DevBuf<double> dev;      // 3 x chunk queries | chunk ranges
    double* pin = nullptr;   // the same layout in page-locked host memory
    size_t pend_off = 0, pend_m = 0;
    ~Lane() {
      if (pin) cudaFreeHost(pin);
      if (s) cudaStreamDestroy(s);
    }
  };
  static thread_local std::vector<Lane> lanes;
  static thread_local size_t lane_chunk = 0;
  static thread_local int lane_dev = -1;
  if (lanes.empty() || lane_chunk < chunk || lane_dev != c->dev) {
    lanes.clear();
    lanes = std::vector<Lane>(NSTREAM);
    lane_chunk = 0;
    for (auto& l : lanes) {
      RL_CK(cudaStreamCreateWithFlags(&l.s, cudaStreamNonBlocking));
      RL_TRY(l.dev.alloc(4 * chunk));
      RL_CK(cudaHostAlloc(reinterpret_cast<void**>(&l.pin), 4 * chunk * sizeof(double),
                          cudaHostAllocDefault));
    }
    lane_chunk = chunk;
    lane_dev = c->dev;
  }
  for (auto& l : lanes) l.pend_m = 0;
  cudaEvent_t ready;
  RL_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  struct EventGuard {
    cudaEvent_t e;
    ~EventGuard() { cudaEventDestroy(e); }
  } ready_guard{ready};
  RL_CK(cudaEventRecord(ready, c->stream));  // order after pending structure work
  const size_t stride = lane_chunk;
  const CddtView v = c->view();
  std::vector<CopySeg> segs;
  size_t k = 0;
  for (size_t off = 0; off < n; k++) {
    const size_t m = std::min(n - off, k < 2 ? std::max<size_t>(chunk >> (2 - k), 1) : chunk);
    Lane& l = lanes[k % NSTREAM];
    segs.clear();
    // the lane's pinned block is reused: its previous upload must have left it,
    // and its previous ranges go to the caller first
    if (k >= NSTREAM && (!in_direct || l.pend_m)) RL_CK(cudaStreamSynchronize(l.s));
    if (l.pend_m) {
      segs.push_back({out + l.pend_off, l.pin + 3 * stride, l.pend_m * sizeof(double)});
      l.pend_m = 0;
    }
    if (!in_direct) segs.push_back({l.pin, q + 3 * off, 3 * m * sizeof(double)});
    if (!segs.empty()) parallel_copy(segs, threads);
    RL_CK(cudaStreamWaitEvent(l.s, ready, 0));
    RL_CK(cudaMemcpyAsync(l.dev.p, in_direct ? q + 3 * off : l.pin, 3 * m * sizeof(double),
                          cudaMemcpyHostToDevice, l.s));
    k_cast_queries<<<dir_blocks(m), 256, 0, l.s>>>(v, l.dev.p, l.dev.p + 3 * stride, m);
    RL_CK(cudaGetLastError());
    RL_CK(cudaMemcpyAsync(out_direct ? out + off : l.pin + 3 * stride, l.dev.p + 3 * stride,
                          m * sizeof(double), cudaMemcpyDeviceToHost, l.s));
    if (!out_direct) {
      l.pend_off = off;
      l.pend_m = m;
    }
    off += m;
  }
  for (size_t j = (k >= NSTREAM ? k - NSTREAM : 0); j < k; j++) {  // drain in submission order
    Lane& l = lanes[j % NSTREAM];
    RL_CK(cudaStreamSynchronize(l.s));
    if (!l.pend_m) continue;
    parallel_copy({{out + l.pend_off, l.pin + 3 * stride, l.pend_m * sizeof(double)}}, threads);
    l.pend_m = 0;
  }
  return RL_OK;
}

extern "C" {

int rl_cddt_cast_queries_host(rl_cddt* c, const double* queries, double* out, size_t n) {
  if (!c || (n && (!queries || !out))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  return cast_queries_pipeline(c, queries, out, n);
}

// One query (Cddt::cast / cast_pair): a one-thread kernel that writes its
// answer straight into the handle's pinned host words (device-visible under
// unified addressing), then one stream synchronisation — no copy operation.
// The round trip is launch-latency bound (INTEGRATION.md "Per-ray calls");
// batches go through the _batch entry points.
static int single(rl_cddt* c, double x, double y, double theta, int pair, double* o0,
                  double* o1) {
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  uint32_t* hs = nullptr;
  RL_TRY(host_small(c, &hs));
  double* r = reinterpret_cast<double*>(hs);
  k_single<<<1, 1, 0, c->stream>>>(c->view(), x, y, theta, pair, r);
  RL_CK(cudaGetLastError());
  RL_CK(cudaStreamSynchronize(c->stream));
  *o0 = r[0];
  if (pair) *o1 = r[1];
  return RL_OK;
}

int rl_cddt_cast(rl_cddt* c, double x, double y, double theta, double* out) {
  if (!c || !out) return RL_EINVAL;
  return single(c, x, y, theta, 0, out, nullptr);
}

int rl_cddt_cast_pair(rl_cddt* c, double x, double y, double theta, double* f, double* b) {
  if (!c || !f || !b) return RL_EINVAL;
  return single(c, x, y, theta, 1, f, b);
}

int rl_cddt_cast_batch(rl_cddt* c, const float* x, const float* y, const float* theta, float* out,
                       int32_t* hit, size_t n, void* stream) {
  if (!c || (n && (!x || !y || !theta || !out))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  RL_TRY(launch_cast<float>(c, x, y, theta, out, hit, nullptr, nullptr, n, pick_stream(c, stream)));
  return finish(c, stream);
}

int rl_cddt_cast_batch_f64(rl_cddt* c, const double* x, const double* y, const double* theta,
                           double* out, int32_t* hit, int64_t* res_row, int32_t* res_idx,
                           size_t n, void* stream) {
  if (!c || (n && (!x || !y || !theta))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  RL_TRY(launch_cast<double>(c, x, y, theta, out, hit, res_row, res_idx, n,
                             pick_stream(c, stream)));
  return finish(c, stream);
}

int rl_cddt_directional_batch(rl_cddt* c, const double* x, const double* y, const int32_t* a,
                              double* out, size_t n, void* stream) {
  if (!c || (n && (!x || !y || !a || !out))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  k_directional<<<dir_blocks(n), 256, 0, pick_stream(c, stream)>>>(c->view(), x, y, a, out, n);
  return finish(c, stream);
}

// Host-buffer batches: chunked H2D -> kernel -> D2H over NSTREAM streams so
// both copy directions overlap the kernel. Page-locked buffers are copied from
// and to directly; pageable ones go through cast_batch_staged above.
int rl_cddt_cast_batch_host(rl_cddt* c, const float* x, const float* y, const float* theta,
                            float* out, size_t n) {
  if (!c || (n && (!x || !y || !theta || !out))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
  static const bool stage_pageable = [] {
    const char* e = std::getenv("RL_HOST_STAGE");
    return e ? std::atoi(e) != 0 : true;
  }();
  if (stage_pageable && n >= kStageMinQueries &&
      !(dma_direct(x) && dma_direct(y) && dma_direct(theta) && dma_direct(out)))
    return cast_batch_staged(c, x, y, theta, out, n);
  constexpr int NSTREAM = 3;
  const size_t chunk = std::min<size_t>(n, size_t(1) << 23);  // 8M queries = 128 MB per chunk
  struct Lane {
    cudaStream_t s = nullptr;
    DevBuf<float> buf;  // x | y | theta | out
  };
  static thread_local std::vector<Lane> lanes;  // reused across calls on this thread
  static thread_local size_t lane_chunk = 0;
  static thread_local int lane_dev = -1;
  if (lanes.empty() || lane_chunk < chunk || lane_dev != c->dev) {
    for (auto& l : lanes)
      if (l.s) cudaStreamDestroy(l.s);
    lanes.clear();
    lanes.resize(NSTREAM);
    for (auto& l : lanes) {
      RL_CK(cudaStreamCreateWithFlags(&l.s, cudaStreamNonBlocking));
      RL_TRY(l.buf.alloc(4 * chunk));
    }
    lane_chunk = chunk;
    lane_dev = c->dev;
  }
  cudaEvent_t ready;
  RL_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  struct EventGuard {  // released on every return path
    cudaEvent_t e;
    ~EventGuard() { cudaEventDestroy(e); }
  } ready_guard{ready};
  RL_CK(cudaEventRecord(ready, c->stream));  // order after pending structure work
  const size_t stride = lane_chunk;
  // Chunk plan. The link is the bottleneck; once the last upload is done it
  // idles for the last chunk's cast and download, so the final `chunk`
  // queries go as a ramp of halving chunks (1/2, 1/4, 1/8, 1/8).
  static const bool ramp = [] {
    const char* e = std::getenv("RL_HOST_RAMP");
    return e ? std::atoi(e) != 0 : true;
  }();
  std::vector<size_t> plan;
  const size_t tail = ramp ? std::min(n, chunk) : 0;
  for (size_t b = n - tail; b > 0;) {
    plan.push_back(std::min(chunk, b));
    b -= plan.back();
  }
  for (size_t rem = tail, part = 0; rem > 0; part++) {
    const size_t m = part < 3 ? std::max<size_t>(1, tail >> (part + 1)) : rem;
    plan.push_back(std::min(m, rem));
    rem -= plan.back();
  }
  size_t k = 0, off = 0;
  for (const size_t m : plan) {
    Lane& l = lanes[k++ % NSTREAM];
    float* dx = l.buf.p;
    float* dy = dx + stride;
    float* dt = dy + stride;
    float* dout = dt + stride;
    RL_CK(cudaStreamWaitEvent(l.s, ready, 0));
    RL_CK(cudaMemcpyAsync(dx, x + off, m * 4, cudaMemcpyHostToDevice, l.s));
    RL_CK(cudaMemcpyAsync(dy, y + off, m * 4, cudaMemcpyHostToDevice, l.s));
    RL_CK(cudaMemcpyAsync(dt, theta + off, m * 4, cudaMemcpyHostToDevice, l.s));
    RL_TRY(launch_cast<float>(c, dx, dy, dt, dout, nullptr, nullptr, nullptr, m, l.s));
    RL_CK(cudaGetLastError());
    RL_CK(cudaMemcpyAsync(out + off, dout, m * 4, cudaMemcpyDeviceToHost, l.s));
    off += m;
  }
  for (auto& l : lanes) RL_CK(cudaStreamSynchronize(l.s));
  return RL_OK;
}

}  // extern "C"
