// CDDT / PCDDT construction, pruning, handle lifecycle and export on sm_100a,
// behind the C ABI in include/rl_cddt.h (queries: rl_query.cu).
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

// Stream-ordered scratch (cudaMallocAsync) comes from a memory pool owned by
// this library, one per device, never from the device's default pool, whose
// settings the host application (e.g. PyTorch) may rely on. While any handle
// on the device is alive the pool keeps freed blocks reserved (release
// threshold UINT64_MAX), so steady-state allocations cost nothing and never
// synchronise; when the last handle on the device is destroyed the pool is
// trimmed to zero and the memory goes back to the driver (trim_pools).
namespace {
struct PoolSlot {
  cudaMemPool_t pool = nullptr;
  int live_handles = 0;
};
std::mutex g_pool_mu;
PoolSlot g_pools[64];
}  // namespace

static int pool_for(int dev, cudaMemPool_t* out) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  PoolSlot& ps = g_pools[dev & 63];
  if (!ps.pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    RL_CK(cudaMemPoolCreate(&ps.pool, &props));
    uint64_t keep = ~0ull;
    RL_CK(cudaMemPoolSetAttribute(ps.pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = ps.pool;
  return RL_OK;
}

int scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  RL_CK(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  RL_TRY(pool_for(dev, &pool));
  RL_CK(cudaMallocFromPoolAsync(p, bytes, pool, st));
  return RL_OK;
}

int scratch_free(void* p, cudaStream_t st) {
  RL_CK(cudaFreeAsync(p, st));
  return RL_OK;
}

void handle_opened(int dev) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  g_pools[dev & 63].live_handles++;
}

// the last handle on `dev` is gone: return the pool's reserved memory (after
// the device is idle, so no stream-ordered free is still pending)
void handle_closed(int dev) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  PoolSlot& ps = g_pools[dev & 63];
  if (--ps.live_handles > 0 || !ps.pool) return;
  ps.live_handles = 0;
  cudaDeviceSynchronize();
  cudaMemPoolTrimTo(ps.pool, 0);
}

// Checked builds: one zeroed {count, first code} pair per device, allocated
// on first use; every view carries it to the device assertions (RL_DCHECK).
unsigned long long* check_counter(int dev) {
#ifdef RL_CHECKED
  static unsigned long long* ctr[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  unsigned long long*& p = ctr[dev & 63];
  if (!p) {
    DeviceGuard guard(dev);
    if (cudaMalloc(&p, 16) != cudaSuccess || cudaMemset(p, 0, 16) != cudaSuccess) p = nullptr;
  }
  return p;
#else
  (void)dev;
  return nullptr;
#endif
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
  RL_TRY(c->d_pdirs.alloc(c->K));
  RL_TRY(c->d_rbase.alloc(c->S));
  std::vector<double4> pdirs(c->K);
  for (int a = 0; a < c->K; a++) {
    const int s = a < c->S ? a : a - c->S;
    pdirs[a] = make_double4(c->dcos[s], c->dsin[s], c->dcos[a], c->dsin[a]);
  }
  std::vector<uint32_t> rbase(c->S);
  for (int s = 0; s < c->S; s++) rbase[s] = c->slices[s].row_base;
  RL_CK(cudaMemcpyAsync(c->d_pdirs.p, pdirs.data(), sizeof(double4) * c->K, cudaMemcpyHostToDevice,
                        c->stream));
  RL_CK(cudaMemcpyAsync(c->d_rbase.p, rbase.data(), sizeof(uint32_t) * c->S,
                        cudaMemcpyHostToDevice, c->stream));
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
  c->zp_slots = total;  // dense rows
  c->gapped = false;

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
    directional_cast(c, double(cx) + 0.5, double(cy) + 0.5, a, o, false);  // resolving index only
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
  RL_TRY(densify_rows(c));  // prune reads dense rows (edits leave slack)
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
  c->zp_slots = kept;
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
  handle_opened(device);
  c->counted = true;
  *keep = c;
  return RL_OK;
}

}  // namespace rl

using namespace rl;

namespace rl {
// The host grid/membership mirrors after edits replayed on the device: one
// download of the flags (occupancy and membership bits).
int refresh_mirrors(const rl_cddt* cc) {
  rl_cddt* c = const_cast<rl_cddt*>(cc);
  if (!c->mirror_stale) return RL_OK;
  const size_t wh = size_t(c->w) * c->h;
  std::vector<uint8_t> fl(wh);
  RL_CK(cudaMemcpyAsync(fl.data(), c->flags.p, wh, cudaMemcpyDeviceToHost, c->stream));
  RL_CK(cudaStreamSynchronize(c->stream));
  c->grid_h.resize(wh);
  c->member_h.resize(wh);
  for (size_t i = 0; i < wh; i++) {
    c->grid_h[i] = (fl[i] & kOcc) ? 1 : 0;
    c->member_h[i] = (fl[i] & kMember) ? 1 : 0;
  }
  c->mirror_stale = false;
  return RL_OK;
}
}  // namespace rl

extern "C" {

const char* rl_last_error(void) { return g_err.c_str(); }

int rl_debug_checks(int32_t device, uint64_t* failures, uint32_t* first_code) {
  if (!failures || !first_code) return RL_EINVAL;
#ifdef RL_CHECKED
  unsigned long long* p = check_counter(device);
  unsigned long long h[2] = {0, 0};
  if (p) {
    DeviceGuard guard(device);
    RL_CK(cudaDeviceSynchronize());
    RL_CK(cudaMemcpy(h, p, sizeof h, cudaMemcpyDeviceToHost));
  }
  *failures = h[0];
  *first_code = uint32_t(h[1]);
  return RL_OK;
#else
  (void)device;
  *failures = 0;
  *first_code = 0xFFFFFFFFu;  // not a checked build
  return RL_OK;
#endif
}

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
    // casts may still run on caller streams (rl_cddt_cast_batch is async)
    cudaDeviceSynchronize();
    c->flags.release();
    c->rowbits.release();
    c->row_off.release();
    c->zp.release();
    c->hints.release();
    c->d_slices.release();
    c->d_dirs.release();
    c->d_pdirs.release();
    c->d_rbase.release();
    c->d_scalar.release();
    c->ws.release();
    c->sensor_ctl.release();
    c->upd_ws.release();
    c->zp_spare.release();
    c->off_spare.release();
    c->row_len.release();
    c->len_spare.release();
    c->row_cap.release();
    c->cap_spare.release();
    c->bkt.release();
    c->estamp.release();
    c->wstamp.release();
    c->pf_ctl.release();
    if (c->pf_host) cudaFreeHost(c->pf_host);
    if (c->host_small) cudaFreeHost(c->host_small);
    if (c->upd_host) cudaFreeHost(c->upd_host);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->counted) handle_closed(c->dev);
  }
  delete c;
  return RL_OK;
}

int rl_cddt_prune(rl_cddt* c) {
  if (!c) return RL_EINVAL;
  DeviceGuard guard(c->dev);
  RL_TRY(quiesce(c));  // casts queued on caller streams read the structure being replaced
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
                    c->hints.bytes() + 4 * (c->gapped ? c->zp.n : c->zero_points) + c->row_len.bytes() + c->row_cap.bytes() +
                    c->d_slices.bytes() +
                    c->d_dirs.bytes() + c->d_pdirs.bytes() + c->d_rbase.bytes();
  o->init_seconds = c->init_seconds;
  return RL_OK;
}

int rl_cddt_sync(rl_cddt* c) {
  if (!c) return RL_EINVAL;
  DeviceGuard guard(c->dev);
  RL_CK(cudaStreamSynchronize(c->stream));
  return RL_OK;
}

int rl_cddt_export(const rl_cddt* c, uint32_t* slice_row_base, uint64_t* row_off, float* zp,
                   uint8_t* membership, uint8_t* grid) {
  if (!c) return RL_EINVAL;
  DeviceGuard guard(c->dev);
  RL_CK(cudaStreamSynchronize(c->stream));
  if (membership || grid) RL_TRY(refresh_mirrors(c));
  if (slice_row_base) {
    for (int s = 0; s < c->S; s++) slice_row_base[s] = c->slices[s].row_base;
    slice_row_base[c->S] = uint32_t(c->rows);
  }
  if (c->gapped && (row_off || zp)) {  // slack rows: the dense CSR the reference defines
    std::vector<uint32_t> o(c->rows + 1), len(c->rows);
    std::vector<float> slots(c->zp_slots);
    RL_CK(cudaMemcpy(o.data(), c->row_off.p, sizeof(uint32_t) * (c->rows + 1),
                     cudaMemcpyDeviceToHost));
    RL_CK(cudaMemcpy(len.data(), c->row_len.p, sizeof(uint32_t) * c->rows,
                     cudaMemcpyDeviceToHost));
    if (zp && c->zp_slots)
      RL_CK(cudaMemcpy(slots.data(), c->zp.p, sizeof(float) * c->zp_slots,
                       cudaMemcpyDeviceToHost));
    uint64_t at = 0;
    for (uint64_t g = 0; g < c->rows; g++) {
      if (row_off) row_off[g] = at;
      if (zp) std::memcpy(zp + at, slots.data() + o[g], sizeof(float) * len[g]);
      at += len[g];
    }
    if (row_off) row_off[c->rows] = at;
  } else {
    if (row_off) {
      std::vector<uint32_t> o(c->rows + 1);
      RL_CK(cudaMemcpy(o.data(), c->row_off.p, sizeof(uint32_t) * (c->rows + 1),
                       cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i <= c->rows; i++) row_off[i] = o[i];
    }
    if (zp && c->zero_points)
      RL_CK(cudaMemcpy(zp, c->zp.p, sizeof(float) * c->zero_points, cudaMemcpyDeviceToHost));
  }
  const size_t wh = size_t(c->w) * c->h;
  if (membership) std::memcpy(membership, c->member_h.data(), wh);
  if (grid) std::memcpy(grid, c->grid_h.data(), wh);
  return RL_OK;
}

}  // extern "C"
