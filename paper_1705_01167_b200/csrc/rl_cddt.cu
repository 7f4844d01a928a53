// CDDT / PCDDT construction, pruning and batched queries on sm_100a, behind
// the C ABI in include/rl_cddt.h.
//
// Device layout:
//   flags[w*h]      u8  bit0 occupied, bit1 clear-3x3, bit2 membership
//   row_off[rows+1] u32 CSR offsets, rows = sum over slices of bin_count,
//                       slice s owns global rows [row_base[s], row_base[s]+bin_count)
//   zp[zero_points] f32 zero points, ascending within each row
//   slices[S]       SliceParam (cos, sin, y_offset, bin_count, row_base)
//   dirs[K]         double4 direction lattice (cos, sin, 1/cos, 1/sin), host glibc, axis snapped
//
// Construction (Cddt::Cddt, proj/src/cddt.cpp:136-171) is a count -> scan ->
// scatter -> segmented sort pipeline; pruning (cddt.cpp:281-330) is a marking
// pass of K casts per free cell followed by a stream compaction.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "rl_common.cuh"

namespace rl {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int finish(const rl_cddt* c, void* s) {
  RL_CK(cudaGetLastError());
  if (!s) RL_CK(cudaStreamSynchronize(c->stream));
  return RL_OK;
}

// direction_components (cddt.cpp:30-42), host glibc.
static void direction_components(int i, int K, double* c, double* s) {
  long long q4 = 4LL * i;
  if (q4 % K == 0) {
    int q = int(q4 / K) & 3;
    *c = (q == 0) ? 1.0 : (q == 2) ? -1.0 : 0.0;
    *s = (q == 1) ? 1.0 : (q == 3) ? -1.0 : 0.0;
  } else {
    double t = double(i) * kTwoPi / double(K);
    *c = std::cos(t);
    *s = std::sin(t);
  }
}

static inline double smin(double a, double b) { return (b < a) ? b : a; }  // std::min
static inline double smax(double a, double b) { return (a < b) ? b : a; }  // std::max

// Direction tables and slice projections (SliceProjection::make, cddt.cpp:44-60).
int init_geometry(rl_cddt* c) {
  c->S = c->K / 2;
  c->dcos.resize(c->K);
  c->dsin.resize(c->K);
  for (int a = 0; a < c->K; a++) direction_components(a, c->K, &c->dcos[a], &c->dsin[a]);
  c->slices.resize(c->S);
  uint64_t base = 0;
  for (int s = 0; s < c->S; s++) {
    double sn = c->dsin[s], cs = c->dcos[s];
    double A = 0.0, B = -double(c->w) * sn, C = double(c->h) * cs, D = B + C;
    double lo = smin(smin(A, B), smin(C, D)), hi = smax(smax(A, B), smax(C, D));
    SliceParam& p = c->slices[s];
    p.cos_t = cs;
    p.sin_t = sn;
    p.y_offset = -lo;
    p.bin_count = int(std::ceil(hi - lo)) + 1;
    p.row_base = uint32_t(base);
    base += uint64_t(p.bin_count);
  }
  if (base >= (1ull << 31)) {
    set_error("cddt: %llu bin rows exceed the 32-bit row index", (unsigned long long)base);
    return RL_EINVAL;
  }
  c->rows = base;
  RL_TRY(c->d_slices.alloc(c->S));
  RL_TRY(c->d_dirs.alloc(c->K));
  // reciprocals for the walker's boundary divisions (cddt_device.cuh div_rn)
  std::vector<double4> dirs(c->K);
  for (int a = 0; a < c->K; a++)
    dirs[a] = make_double4(c->dcos[a], c->dsin[a], c->dcos[a] != 0.0 ? 1.0 / c->dcos[a] : 0.0,
                           c->dsin[a] != 0.0 ? 1.0 / c->dsin[a] : 0.0);
  RL_CK(cudaMemcpyAsync(c->d_slices.p, c->slices.data(), sizeof(SliceParam) * c->S,
                        cudaMemcpyHostToDevice, c->stream));
  RL_CK(cudaMemcpyAsync(c->d_dirs.p, dirs.data(), sizeof(double4) * c->K, cudaMemcpyHostToDevice,
                        c->stream));
  RL_CK(cudaStreamSynchronize(c->stream));
  return RL_OK;
}

// ---------------------------------------------------------------------------
// K1: per-cell flags. occupied; clear = cell and all in-bounds 8-neighbours
// free (clear_around, cddt.cpp:173-180); member = occupied with a free or
// out-of-bounds 8-neighbour (is_edge_cell, grid.cpp:110-119).
__global__ void k_flags(const uint8_t* __restrict__ grid, uint8_t* __restrict__ flags, int w,
                        int h) {
  const size_t n = size_t(w) * h;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int x = int(i % w), y = int(i / w);
    const bool occ = grid[i] != 0;
    bool any_occ_nb = false, any_free_or_oob_nb = false;
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        if (dx == 0 && dy == 0) continue;
        int nx = x + dx, ny = y + dy;
        if (nx < 0 || ny < 0 || nx >= w || ny >= h) {
          any_free_or_oob_nb = true;
        } else if (grid[size_t(ny) * w + nx]) {
          any_occ_nb = true;
        } else {
          any_free_or_oob_nb = true;
        }
      }
    uint8_t f = 0;
    if (occ) f |= kOcc;
    if (!occ && !any_occ_nb) f |= kClear;
    if (occ && any_free_or_oob_nb) f |= kMember;
    flags[i] = f;
  }
}

// Query occupancy bits: per 32-cell run of a grid row, {occupied, clear}.
__global__ void k_rowbits(const uint8_t* __restrict__ flags, int w, int h, int wpr,
                          uint2* __restrict__ bits) {
  const int n = wpr * h;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int y = t / wpr, x0 = (t % wpr) * 32;
    unsigned occ = 0, clr = 0;
    for (int b = 0; b < 32 && x0 + b < w; b++) {
      const uint8_t f = flags[size_t(y) * w + x0 + b];
      if (f & kOcc) occ |= 1u << b;
      if (f & kClear) clr |= 1u << b;
    }
    bits[t] = make_uint2(occ, clr);
  }
}

int refresh_query_bits(rl_cddt* c) {
  c->wpr = (c->w + 31) / 32;
  const size_t nw = size_t(c->wpr) * c->h;
  if (c->rowbits.n != nw) RL_TRY(c->rowbits.alloc(nw));
  k_rowbits<<<int(std::min<size_t>((nw + 255) / 256, size_t(sm_count()) * 16)), 256, 0,
              c->stream>>>(c->flags.p, c->w, c->h, c->wpr, c->rowbits.p);
  RL_CK(cudaGetLastError());
  return RL_OK;
}

__global__ void k_row_hints(const uint32_t* __restrict__ row_off, const float* __restrict__ zp,
                            uint64_t rows, float* __restrict__ hints) {
  for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < rows;
       g += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t lo = row_off[g], n = row_off[g + 1] - lo;
    float h[kHintFloats];
    int slot = 0;
    h[slot++] = __uint_as_float(lo);
    h[slot++] = __uint_as_float(n);
    for (int level = 0; level < kHintLevels; level++)
      for (uint32_t path = 0; path < (1u << level) && slot < kHintFloats; path++, slot++) {
        uint32_t idx;
        h[slot] = hint_index(n, level, path, &idx) ? zp[lo + idx] : 0.f;
      }
    for (; slot < kHintFloats; slot++) h[slot] = 0.f;
    for (int k = 0; k < kHintFloats; k += 4)
      reinterpret_cast<float4*>(hints + g * kHintFloats)[k / 4] =
          make_float4(h[k], h[k + 1], h[k + 2], h[k + 3]);
  }
}

int refresh_row_hints(rl_cddt* c) {
  if (c->hints.n != c->rows * kHintFloats) RL_TRY(c->hints.alloc(c->rows * kHintFloats));
  if (c->rows)
    k_row_hints<<<int(std::min<uint64_t>((c->rows + 255) / 256, uint64_t(sm_count()) * 16)), 256,
                  0, c->stream>>>(c->row_off.p, c->zp.p, c->rows, c->hints.p);
  RL_CK(cudaGetLastError());
  return RL_OK;
}

// Compact member cells into an (unordered) edge list; warp-aggregated atomics.
__global__ void k_edge_list(const uint8_t* __restrict__ flags, size_t n, int32_t* __restrict__ edges,
                            unsigned int* __restrict__ count) {
  for (size_t base = blockIdx.x * size_t(blockDim.x); base < n;
       base += size_t(gridDim.x) * blockDim.x) {
    size_t i = base + threadIdx.x;
    bool m = i < n && (flags[i] & kMember);
    unsigned ballot = __ballot_sync(0xffffffffu, m);
    unsigned lane = threadIdx.x & 31;
    unsigned pos0 = 0;
    if (lane == 0 && ballot) pos0 = atomicAdd(count, __popc(ballot));
    pos0 = __shfl_sync(0xffffffffu, pos0, 0);
    if (m) edges[pos0 + __popc(ballot & ((1u << lane) - 1))] = int32_t(i);
  }
}

// for_each_bin_of_pixel (cddt.cpp:118-134): rows [r0, r1] of slice sp whose
// unit strip overlaps pixel (px, py) with positive area, and the pixel
// centre's projected x' rounded to f32.
__device__ __forceinline__ void pixel_rows(const SliceParam& sp, int px, int py, int& r0, int& r1,
                                           float& v) {
  auto py_of = [&](double x, double y) { return -x * sp.sin_t + y * sp.cos_t + sp.y_offset; };
  double c0 = py_of(double(px), double(py));
  double c1 = py_of(double(px + 1), double(py));
  double c2 = py_of(double(px), double(py + 1));
  double c3 = py_of(double(px + 1), double(py + 1));
  double lo = fmin_std(fmin_std(c0, c1), fmin_std(c2, c3));
  double hi = fmax_std(fmax_std(c0, c1), fmax_std(c2, c3));
  r0 = int(floor(lo));
  r1 = int(ceil(hi)) - 1;
  if (r0 < 0) r0 = 0;
  if (r1 >= sp.bin_count) r1 = sp.bin_count - 1;
  const double cx = double(px) + 0.5, cy = double(py) + 0.5;
  v = __double2float_rn(cx * sp.cos_t + cy * sp.sin_t);
}

// K2a/K2b: per (edge pixel, slice): count rows, then scatter values.
template <bool SCATTER>
__global__ void k_points(const int32_t* __restrict__ edges, unsigned n_edges,
                         const SliceParam* __restrict__ slices, int S, int w,
                         uint32_t* __restrict__ cnt, const uint32_t* __restrict__ row_off,
                         float* __restrict__ zp) {
  const uint64_t total = uint64_t(n_edges) * S;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned e = unsigned(i / S);
    const int s = int(i % S);
    const int32_t cell = edges[e];
    const int px = cell % w, py = cell / w;
    const SliceParam sp = slices[s];
    int r0, r1;
    float v;
    pixel_rows(sp, px, py, r0, r1, v);
    for (int r = r0; r <= r1; r++) {
      const uint32_t g = sp.row_base + uint32_t(r);
      if (SCATTER) {
        uint32_t pos = row_off[g] + atomicAdd(&cnt[g], 1u);
        zp[pos] = v;
      } else {
        atomicAdd(&cnt[g], 1u);
      }
    }
  }
}

struct ToU64 {
  __host__ __device__ unsigned long long operator()(uint32_t v) const { return v; }
};

static int grid_blocks(size_t work, int threads) {
  size_t b = (work + threads - 1) / threads;
  size_t cap = size_t(sm_count()) * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return int(b);
}

// Full construction from c->grid_h: flags, membership mirror, CSR.
int build_structure(rl_cddt* c) {
  const size_t wh = size_t(c->w) * c->h;
  cudaStream_t st = c->stream;
  DevBuf<uint8_t> d_grid;
  RL_TRY(d_grid.alloc(wh));
  RL_TRY(c->flags.alloc(wh));
  RL_CK(cudaMemcpyAsync(d_grid.p, c->grid_h.data(), wh, cudaMemcpyHostToDevice, st));
  k_flags<<<grid_blocks(wh, 256), 256, 0, st>>>(d_grid.p, c->flags.p, c->w, c->h);
  RL_CK(cudaGetLastError());

  DevBuf<int32_t> edges;
  DevBuf<unsigned> d_count;
  RL_TRY(edges.alloc(wh));
  RL_TRY(d_count.alloc(1));
  RL_CK(cudaMemsetAsync(d_count.p, 0, sizeof(unsigned), st));
  k_edge_list<<<grid_blocks(wh, 256), 256, 0, st>>>(c->flags.p, wh, edges.p, d_count.p);
  unsigned n_edges = 0;
  RL_CK(cudaMemcpyAsync(&n_edges, d_count.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));

  const uint64_t rows = c->rows;
  DevBuf<uint32_t> cnt;
  RL_TRY(cnt.alloc(rows + 1));
  RL_TRY(c->row_off.alloc(rows + 1));
  RL_CK(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * (rows + 1), st));
  const uint64_t pairs = uint64_t(n_edges) * c->S;
  if (pairs)
    k_points<false><<<grid_blocks(pairs, 256), 256, 0, st>>>(edges.p, n_edges, c->d_slices.p,
                                                             c->S, c->w, cnt.p, nullptr, nullptr);
  RL_CK(cudaGetLastError());
  {
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, c->row_off.p, int(rows + 1), st);
    DevBuf<uint8_t> tmp;
    RL_TRY(tmp.alloc(tmp_bytes));
    RL_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, c->row_off.p, int(rows + 1), st));
  }
  uint64_t total = 0;
  {
    // 64-bit total so a wrapped 32-bit CSR offset is detected, not silently used
    DevBuf<unsigned long long> d_total;
    RL_TRY(d_total.alloc(1));
    auto wide = cub::TransformInputIterator<unsigned long long, ToU64, const uint32_t*>(cnt.p, ToU64());
    size_t tmp_bytes = 0;
    cub::DeviceReduce::Sum(nullptr, tmp_bytes, wide, d_total.p, int(rows), st);
    DevBuf<uint8_t> tmp;
    RL_TRY(tmp.alloc(tmp_bytes));
    RL_CK(cub::DeviceReduce::Sum(tmp.p, tmp_bytes, wide, d_total.p, int(rows), st));
    RL_CK(cudaMemcpyAsync(&total, d_total.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    RL_CK(cudaStreamSynchronize(st));
  }
  if (total >= (1ull << 31)) {
    set_error("cddt: %llu zero points exceed the 31-bit CSR offset", (unsigned long long)total);
    return RL_EINVAL;
  }
  c->zero_points = total;

  DevBuf<float> unsorted;
  RL_TRY(unsorted.alloc(total));
  RL_TRY(c->zp.alloc(total));
  RL_CK(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * (rows + 1), st));
  if (pairs)
    k_points<true><<<grid_blocks(pairs, 256), 256, 0, st>>>(edges.p, n_edges, c->d_slices.p, c->S,
                                                            c->w, cnt.p, c->row_off.p, unsorted.p);
  RL_CK(cudaGetLastError());
  if (total) {
    size_t tmp_bytes = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, unsorted.p, c->zp.p, int(total),
                                       int(rows), c->row_off.p, c->row_off.p + 1, st);
    DevBuf<uint8_t> tmp;
    RL_TRY(tmp.alloc(tmp_bytes));
    RL_CK(cub::DeviceSegmentedSort::SortKeys(tmp.p, tmp_bytes, unsorted.p, c->zp.p, int(total),
                                             int(rows), c->row_off.p, c->row_off.p + 1, st));
  }
  RL_TRY(refresh_query_bits(c));
  RL_TRY(refresh_row_hints(c));
  // host membership mirror
  c->member_h.assign(wh, 0);
  {
    std::vector<uint8_t> fl(wh);
    RL_CK(cudaMemcpyAsync(fl.data(), c->flags.p, wh, cudaMemcpyDeviceToHost, st));
    RL_CK(cudaStreamSynchronize(st));
    for (size_t i = 0; i < wh; i++) c->member_h[i] = (fl[i] & kMember) ? 1 : 0;
  }
  return RL_OK;
}

// ---------------------------------------------------------------------------
// K3: batched casts.
//
// Monolithic form (f64 / hit-cell / resolving-index outputs, and batches
// below 4M queries): one thread per query, grid-stride, a single full wave
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
    const double r = directional_cast(c, x, y, direction_index(th, c.K), o);
    if (out) __stcs(out + i, T(r));
    if (HIT && hit) hit[i] = o.hit;
    if (RES) {
      if (res_row) res_row[i] = o.res_idx >= 0 ? int64_t(o.res_g) : -1;
      if (res_idx) res_idx[i] = o.res_idx;
    }
  }
}

// Deferred-walk form (f32 ranges only, >= 4M queries; the bench path).
// About a third of the queries need a RayWalker (a near-field walk or a
// verification window). Run inline, those walks execute with ~5 of 32 lanes
// active and cost half the kernel time (profiles/r01/ncu_k_cast_v3.txt).
// Phase 1 settles every query that needs no walker with uniform control flow
// and queues the rest — with the CSR row and the pending candidate — through
// a per-CTA shared-memory compaction (one global atomic per CTA iteration).
// The window passes (k_walk_pass) resume exactly there, every lane walking;
// near-field queries are redone in full by k_cast_near. Records are streamed
// evict-first past L2.
struct __align__(16) WalkRecord {
  float x, y, t;
  uint32_t i, lo, n;
  int32_t idx, pad;
};

#ifndef RL_P1_CTAS
#define RL_P1_CTAS 6  // resident CTAs per SM the register budget of phase 1 targets
#endif
#ifndef RL_P2_CTAS
#define RL_P2_CTAS 4
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
    WalkRecord rec;
    if (i < n) {
      rec.x = __ldcs(qx + i);
      rec.y = __ldcs(qy + i);
      rec.t = __ldcs(qt + i);
      rec.i = i;
      const double th = normalize_angle_2pi(double(rec.t));
      double r;
      WalkDefer def;
      if (directional_cast_p1(c, double(rec.x), double(rec.y), direction_index(th, c.K), &r,
                              &def)) {
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
      const float4* src = reinterpret_cast<const float4*>(&rec);
      float4* dst = reinterpret_cast<float4*>(q + slot);
      __stcs(dst, src[0]);
      __stcs(dst + 1, src[1]);
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
  int32_t idx, cx, cy, pad;
  double wt;
};

#ifndef RL_WALK_THREADS
#define RL_WALK_THREADS 64  // small CTAs: cheap compaction barriers
#endif
constexpr int kWalkThreads = RL_WALK_THREADS;

// out-of-line: the rare overflow path must not add to the pass's registers
__device__ __noinline__ double finish_windows(const CddtView& c, double x, double y, int a,
                                              WinState s) {
  double res;
  resume_windows<false>(c, x, y, a, s, 0x7fffffff, &res);
  return res;
}

template <class T, bool CONT, bool LAST>
__global__ void __launch_bounds__(kWalkThreads, RL_P2_CTAS * 256 / kWalkThreads) k_walk_pass(
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
      } else {
        const float4* src = reinterpret_cast<const float4*>(static_cast<const WalkRecord*>(in) + k);
        const float4 w0 = __ldcs(src), w1 = __ldcs(src + 1);
        fx = w0.x;
        fy = w0.y;
        ft = w0.z;
        qi = __float_as_uint(w0.w);
        s = WinState{__float_as_uint(w1.x), __float_as_uint(w1.y), __float_as_int(w1.z), 0, 0, 0.0,
                     w1.w};
      }
      a = direction_index(normalize_angle_2pi(double(ft)), c.K);
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
      if (slot < out_cap) {  // ContRecord layout, as three 16-byte stores
        float4* dst = reinterpret_cast<float4*>(oq + slot);
        __stcs(dst, make_float4(fx, fy, ft, __uint_as_float(qi)));
        __stcs(dst + 1, make_float4(__uint_as_float(s.lo), __uint_as_float(s.n),
                                    __int_as_float(s.idx), __int_as_float(s.cx)));
        __stcs(dst + 2, make_float4(__int_as_float(s.cy), 0.f,
                                    __int_as_float(__double2loint(s.t)),
                                    __int_as_float(__double2hiint(s.t))));
      } else {  // queue full: finish here
        __stcs(out + qi, T(finish_windows(c, double(fx), double(fy), a, s)));
      }
    }
    __syncthreads();
  }
}

// Near-field records (origin not clear): near-field walk, search and landing
// probes here; queries that need a verification window join the window
// passes as continuations (queue A, after pass 0's own).
template <class T>
__global__ void __launch_bounds__(kWalkThreads, RL_P2_CTAS * 256 / kWalkThreads) k_cast_near(
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
        __stcs(dst + 2, make_float4(__int_as_float(s.cy), 0.f,
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

#ifndef RL_DEFER_MIN_LOG2
#define RL_DEFER_MIN_LOG2 22
#endif
constexpr size_t kDeferMinQueries = size_t(1) << RL_DEFER_MIN_LOG2;

// Dispatch of the batched cast kernels for the device-pointer entry points.
template <class T>
static int launch_cast(const rl_cddt* c, const T* x, const T* y, const T* t, T* out,
                       int32_t* hit, int64_t* rr, int32_t* ri, size_t n, cudaStream_t st) {
  const CddtView v = c->view();
  const bool small = n < (size_t(1) << 31);
  if (!rr && !ri && !hit && small && n >= kDeferMinQueries) {
    // stream-ordered scratch: concurrent batches on other streams (e.g. the
    // pipelined host path) each get their own queue; the pool keeps the
    // memory reserved, so steady-state allocation is free
    static const bool pool_ready = [] {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      return true;
    }();
    (void)pool_ready;
    // workspace: counters | n walk records (windows up from 0, near field down
    // from n-1) | continuation queues A and B (the window passes alternate)
    // (RL_CDDT_CONT_CAP overrides the queue capacity: a test hook for the
    // queue-full path)
    static const size_t cap_env = [] {
      const char* e = std::getenv("RL_CDDT_CONT_CAP");
      return e ? size_t(std::strtoull(e, nullptr, 10)) : size_t(0);
    }();
#ifdef RL_WIN_CAPS_CODE  // A/B builds: decimal digits, e.g. 1124 -> {1, 1, 2, 4}
    constexpr int kPasses = RL_WIN_CAPS_CODE >= 1000 ? 4 : RL_WIN_CAPS_CODE >= 100 ? 3
                                                     : RL_WIN_CAPS_CODE >= 10 ? 2 : 1;
    int kCaps[kPasses];
    for (int p = kPasses - 1, v = RL_WIN_CAPS_CODE; p >= 0; p--, v /= 10) kCaps[p] = v % 10;
#else
    constexpr int kCaps[] = {RL_WIN_CAPS};
    constexpr int kPasses = sizeof(kCaps) / sizeof(kCaps[0]);  // capped passes; one more runs out
#endif
    const size_t cap_a = cap_env ? cap_env : std::max<size_t>(n / RL_CONT_A_DIV, size_t(1) << 16);
    const size_t cap_b = cap_env ? cap_env : std::max<size_t>(n / RL_CONT_B_DIV, size_t(1) << 16);
    uint8_t* ws = nullptr;
    RL_CK(cudaMallocAsync(reinterpret_cast<void**>(&ws),
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
    RL_CK(cudaMemsetAsync(qn, 0, (2 + kPasses) * sizeof(unsigned), st));
    const size_t b1 = std::max<size_t>(
        1, std::min((n + kP1Threads - 1) / kP1Threads, size_t(sm_count()) * p1));
    k_cast_defer_p1<T><<<int(b1), kP1Threads, 0, st>>>(v, x, y, t, out, uint32_t(n), q, qn);
    k_cast_near<T><<<sm_count() * pn, kWalkThreads, 0, st>>>(v, q, qn, uint32_t(n), qa, qn + 2,
                                                             uint32_t(cap_a), out);
    k_walk_pass<T, false, false><<<sm_count() * pw0, kWalkThreads, 0, st>>>(
        v, q, qn, uint32_t(n), kCaps[0], qa, qn + 2, uint32_t(cap_a), out);
    for (int p = 1; p < kPasses; p++) {  // queue p-1 -> queue p (A, B, A, ...)
      const bool from_a = (p & 1) != 0;
      k_walk_pass<T, true, false><<<sm_count() * pwc, kWalkThreads, 0, st>>>(
          v, from_a ? qa : qb, qn + 1 + p, uint32_t(from_a ? cap_a : cap_b), kCaps[p],
          from_a ? qb : qa, qn + 2 + p, uint32_t(from_a ? cap_b : cap_a), out);
    }
    const bool last_a = (kPasses & 1) != 0;
    k_walk_pass<T, true, true><<<sm_count() * pwl, kWalkThreads, 0, st>>>(
        v, last_a ? qa : qb, qn + 1 + kPasses, uint32_t(last_a ? cap_a : cap_b), 0, nullptr,
        nullptr, 0, out);
#ifdef RL_DEBUG_COUNTS
    {
      unsigned h[2 + kPasses];
      cudaMemcpyAsync(h, qn, sizeof h, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "counts n=%zu windows=%u near=%u", n, h[0], h[1]);
      for (int p = 0; p < kPasses; p++) fprintf(stderr, " after pass %d: %u", p, h[2 + p]);
      fprintf(stderr, "\n");
    }
#endif
    RL_CK(cudaFreeAsync(ws, st));
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
    out[i] = directional_cast(c, x[i], y[i], a[i], o);
  }
}

__global__ void k_single(CddtView c, double x, double y, double theta, int pair,
                         double* __restrict__ out) {
  const double th = normalize_angle_2pi(theta);
  const int a = direction_index(th, c.K);
  CastOut o;
  out[0] = directional_cast(c, x, y, a, o);
  if (pair) out[1] = directional_cast(c, x, y, (a + c.K / 2) % c.K, o);  // cddt.cpp:275-279
}

static int dir_blocks(size_t n) {
  size_t b = (n + 255) / 256;
  return int(std::max<size_t>(1, std::min(b, size_t(sm_count()) * 8)));
}

// ---------------------------------------------------------------------------
// K4: prune marking. One state per (free cell centre, direction); the
// resolving index and its near-side neighbour are marked (cddt.cpp:289-299).
__global__ void __launch_bounds__(256) k_prune_mark(CddtView c, uint8_t* __restrict__ marks) {
  const uint64_t total = uint64_t(c.w) * c.h * c.K;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t cell = i / c.K;
    const int a = int(i % c.K);
    if (__ldg(c.flags + cell) & kOcc) continue;  // occupied origins never consult bins
    const int cx = int(cell % c.w), cy = int(cell / c.w);
    CastOut o;
    directional_cast(c, double(cx) + 0.5, double(cy) + 0.5, a, o);
    if (o.res_idx < 0) continue;
    const uint32_t lo = c.row_off[o.res_g], n = c.row_off[o.res_g + 1] - lo;
    uint8_t* m = marks + lo;
    m[o.res_idx] = 1;
    if (a < c.S) {
      if (o.res_idx > 0) m[o.res_idx - 1] = 1;
    } else {
      if (uint32_t(o.res_idx) + 1 < n) m[o.res_idx + 1] = 1;
    }
  }
}

__global__ void k_widen(const uint8_t* __restrict__ in, uint32_t* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i <= n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = i < n ? uint32_t(in[i]) : 0u;
}

__global__ void k_compact(const float* __restrict__ zp, const uint8_t* __restrict__ marks,
                          const uint32_t* __restrict__ pos, float* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    if (marks[i]) out[pos[i]] = zp[i];
}

__global__ void k_remap_offsets(const uint32_t* __restrict__ old_off,
                                const uint32_t* __restrict__ pos, uint32_t* __restrict__ new_off,
                                size_t rows) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g <= rows;
       g += size_t(gridDim.x) * blockDim.x)
    new_off[g] = pos[old_off[g]];
}

int prune_structure(rl_cddt* c) {
  if (c->pruned) return RL_OK;
  cudaStream_t st = c->stream;
  const size_t n = c->zero_points;
  DevBuf<uint8_t> marks;
  RL_TRY(marks.alloc(n));
  RL_CK(cudaMemsetAsync(marks.p, 0, n ? n : 1, st));
  const uint64_t states = uint64_t(c->w) * c->h * c->K;
  k_prune_mark<<<int(std::max<uint64_t>(1, std::min<uint64_t>((states + 255) / 256,
                                                                 uint64_t(sm_count()) * 8))),
                 256, 0, st>>>(c->view(), marks.p);
  RL_CK(cudaGetLastError());
  DevBuf<uint32_t> wide, pos;
  RL_TRY(wide.alloc(n + 1));
  RL_TRY(pos.alloc(n + 1));
  k_widen<<<grid_blocks(n + 1, 256), 256, 0, st>>>(marks.p, wide.p, n);
  {
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, wide.p, pos.p, int(n + 1), st);
    DevBuf<uint8_t> tmp;
    RL_TRY(tmp.alloc(tmp_bytes));
    RL_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, wide.p, pos.p, int(n + 1), st));
  }
  uint32_t kept = 0;
  RL_CK(cudaMemcpyAsync(&kept, pos.p + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
  DevBuf<float> nzp;
  DevBuf<uint32_t> noff;
  RL_TRY(nzp.alloc(kept));
  RL_TRY(noff.alloc(c->rows + 1));
  k_compact<<<grid_blocks(n, 256), 256, 0, st>>>(c->zp.p, marks.p, pos.p, nzp.p, n);
  k_remap_offsets<<<grid_blocks(c->rows + 1, 256), 256, 0, st>>>(c->row_off.p, pos.p, noff.p,
                                                                  c->rows);
  RL_CK(cudaGetLastError());
  RL_CK(cudaStreamSynchronize(st));
  c->zp = std::move(nzp);
  c->row_off = std::move(noff);
  c->zero_points = kept;
  c->pruned = true;
  RL_TRY(refresh_row_hints(c));
  RL_CK(cudaStreamSynchronize(st));
  return RL_OK;
}

int create_handle(int32_t device, rl_cddt** out, rl_cddt** keep) {
  *out = nullptr;
  int ndev = 0;
  RL_CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("cddt: device %d not available (%d devices)", device, ndev);
    return RL_EINVAL;
  }
  rl_cddt* c = new rl_cddt();
  c->dev = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    set_error("cudaStreamCreate: %s", cudaGetErrorString(e));
    return RL_ECUDA;
  }
  *keep = c;
  return RL_OK;
}

}  // namespace rl

using namespace rl;

extern "C" {

const char* rl_last_error(void) { return g_err.c_str(); }

int rl_cddt_create(const uint8_t* grid, int32_t width, int32_t height, double resolution,
                   int32_t theta_disc, double max_range, int32_t prune, int32_t device,
                   rl_cddt** out) {
  if (!out) return RL_EINVAL;
  *out = nullptr;
  if (!grid || width <= 0 || height <= 0) {
    set_error("grid dimensions must be positive");  // grid.hpp:21
    return RL_EINVAL;
  }
  if (!(resolution > 0.0)) {
    set_error("resolution must be positive");  // grid.hpp:22
    return RL_EINVAL;
  }
  if (max_range < 0.0) {
    set_error("max_range must be >= 0");  // raycast.hpp:56
    return RL_EINVAL;
  }
  if (theta_disc < 4 || theta_disc % 2 != 0) {
    set_error("theta_disc must be even and >= 4");  // raycast.hpp:57-58
    return RL_EINVAL;
  }
  auto t0 = std::chrono::steady_clock::now();
  DeviceGuard guard(device);
  rl_cddt* c = nullptr;
  RL_TRY(create_handle(device, out, &c));
  c->w = width;
  c->h = height;
  c->K = theta_disc;
  c->resolution = resolution;
  c->max_range = max_range > 0.0 ? max_range
                                 : std::sqrt(double(width) * width + double(height) * height);
  const size_t wh = size_t(width) * height;
  c->grid_h.resize(wh);
  for (size_t i = 0; i < wh; i++) c->grid_h[i] = grid[i] ? 1 : 0;
  int st = init_geometry(c);
  if (st == RL_OK) st = build_structure(c);
  if (st == RL_OK && prune) st = prune_structure(c);
  if (st != RL_OK) {
    std::string msg = g_err;
    rl_cddt_destroy(c);
    g_err = msg;
    return st;
  }
  c->init_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = c;
  return RL_OK;
}

int rl_cddt_destroy(rl_cddt* c) {
  if (!c) return RL_OK;
  {
    DeviceGuard guard(c->dev);
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->flags.release();
    c->rowbits.release();
    c->row_off.release();
    c->zp.release();
    c->hints.release();
    c->d_slices.release();
    c->d_dirs.release();
    c->d_scalar.release();
    c->ws.release();
    c->upd_ws.release();
    c->zp_spare.release();
    c->off_spare.release();
    c->pf_ctl.release();
    if (c->pf_host) cudaFreeHost(c->pf_host);
    if (c->stream) cudaStreamDestroy(c->stream);
  }
  delete c;
  return RL_OK;
}

int rl_cddt_prune(rl_cddt* c) {
  if (!c) return RL_EINVAL;
  DeviceGuard guard(c->dev);
  return prune_structure(c);
}

int rl_cddt_info(const rl_cddt* c, rl_cddt_info_t* o) {
  if (!c || !o) return RL_EINVAL;
  o->width = c->w;
  o->height = c->h;
  o->theta_disc = c->K;
  o->slice_count = c->S;
  o->pruned = c->pruned;
  o->device = c->dev;
  o->max_range = c->max_range;
  o->resolution = c->resolution;
  o->rows = c->rows;
  o->zero_points = c->zero_points;
  const uint64_t wh = uint64_t(c->w) * c->h;
  o->memory_bytes = 4 * c->zero_points + (wh + 7) / 8 + uint64_t(c->S) * 48;  // cddt.hpp:200-203
  o->device_bytes = c->flags.bytes() + c->rowbits.bytes() + c->row_off.bytes() +
                    c->hints.bytes() + 4 * c->zero_points + c->d_slices.bytes() +
                    c->d_dirs.bytes();
  o->init_seconds = c->init_seconds;
  return RL_OK;
}

int rl_cddt_sync(rl_cddt* c) {
  if (!c) return RL_EINVAL;
  DeviceGuard guard(c->dev);
  RL_CK(cudaStreamSynchronize(c->stream));
  return RL_OK;
}

static int single(rl_cddt* c, double x, double y, double theta, int pair, double* o0,
                  double* o1) {
  std::lock_guard<std::mutex> lock(c->mu);
  DeviceGuard guard(c->dev);
  if (!c->d_scalar.p) RL_TRY(c->d_scalar.alloc(2));
  k_single<<<1, 1, 0, c->stream>>>(c->view(), x, y, theta, pair, c->d_scalar.p);
  RL_CK(cudaGetLastError());
  double r[2];
  RL_CK(cudaMemcpyAsync(r, c->d_scalar.p, sizeof(double) * (pair ? 2 : 1), cudaMemcpyDeviceToHost,
                        c->stream));
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
// both copy directions overlap the kernel.
int rl_cddt_cast_batch_host(rl_cddt* c, const float* x, const float* y, const float* theta,
                            float* out, size_t n) {
  if (!c || (n && (!x || !y || !theta || !out))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  DeviceGuard guard(c->dev);
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
  RL_CK(cudaEventRecord(ready, c->stream));  // order after pending structure work
  const size_t stride = lane_chunk;
  size_t k = 0;
  for (size_t off = 0; off < n; off += chunk, k++) {
    Lane& l = lanes[k % NSTREAM];
    const size_t m = std::min(chunk, n - off);
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
  }
  for (auto& l : lanes) RL_CK(cudaStreamSynchronize(l.s));
  cudaEventDestroy(ready);
  return RL_OK;
}

int rl_cddt_export(const rl_cddt* c, uint32_t* slice_row_base, uint64_t* row_off, float* zp,
                   uint8_t* membership, uint8_t* grid) {
  if (!c) return RL_EINVAL;
  DeviceGuard guard(c->dev);
  RL_CK(cudaStreamSynchronize(c->stream));
  if (slice_row_base) {
    for (int s = 0; s < c->S; s++) slice_row_base[s] = c->slices[s].row_base;
    slice_row_base[c->S] = uint32_t(c->rows);
  }
  if (row_off) {
    std::vector<uint32_t> o(c->rows + 1);
    RL_CK(cudaMemcpy(o.data(), c->row_off.p, sizeof(uint32_t) * (c->rows + 1),
                     cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i <= c->rows; i++) row_off[i] = o[i];
  }
  if (zp && c->zero_points)
    RL_CK(cudaMemcpy(zp, c->zp.p, sizeof(float) * c->zero_points, cudaMemcpyDeviceToHost));
  const size_t wh = size_t(c->w) * c->h;
  if (membership) std::memcpy(membership, c->member_h.data(), wh);
  if (grid) std::memcpy(grid, c->grid_h.data(), wh);
  return RL_OK;
}

}  // extern "C"
