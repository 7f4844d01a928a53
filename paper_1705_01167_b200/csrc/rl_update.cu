// Incremental map updates: Cddt::set_occupancy (proj/src/cddt.cpp:332-377)
// applied to a batch of edits.
//
// The reference maintains the invariant that after any edit sequence the bins
// equal a fresh build of the final grid (proj/tests/test_cddt.cpp:578-604):
// membership is exactly the edge map, and each member pixel contributes
// float(project_x(centre)) to every row its square overlaps. A batch is
// therefore applied as a set difference against the current structure:
//   1. host: replay the edits in order on the host grid mirror (last writer
//      wins), collect cells whose occupancy changed;
//   2. host: recompute occupancy/clear/membership flags in the 1-cell dilation
//      of those cells; cells whose membership flipped are the delta pixels;
//   3. device: expand delta pixels to (row, value, +/-1) records over all
//      slices, counted per row; one scan gives both the new row offsets and
//      each row's bucket of delta records, which a second pass fills;
//   4. device: per-row merge of the old sorted row with its (unsorted)
//      deltas (unaffected rows are a straight copy).
// Only O(changed pixels * S) records are written; the copy is one pass over
// the zero-point array.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rl_common.cuh"

namespace rl {

// for_each_bin_of_pixel (cddt.cpp:118-134), as in rl_cddt.cu (device code is per-TU)
__device__ __forceinline__ void pixel_rows_u(const SliceParam& sp, int px, int py, int& r0,
                                             int& r1, float& v) {
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

// delta pixel (cell, sign) x slice -> per-row counts of added / removed points
__global__ void k_delta_count(const int32_t* __restrict__ cells, const int8_t* __restrict__ sign,
                              int n_cells, const SliceParam* __restrict__ slices, int S, int w,
                              int32_t* __restrict__ add_cnt, int32_t* __restrict__ rem_cnt) {
  const int total = n_cells * S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int k = i / S, s = i % S;
    const int cell = cells[k];
    const SliceParam sp = slices[s];
    int r0, r1;
    float v;
    pixel_rows_u(sp, cell % w, cell / w, r0, r1, v);
    int32_t* cnt = sign[k] > 0 ? add_cnt : rem_cnt;
    for (int r = r0; r <= r1; r++) atomicAdd(&cnt[sp.row_base + uint32_t(r)], 1);
  }
}

// Slots a row of `len` points is given when the rows are (re)laid out by an
// edit batch: room for later edits to merge in place (about 1/8 more).
__host__ __device__ __forceinline__ uint32_t slot_capacity(uint32_t len) {
  return len + (len >> 3) + 4u;
}

// packed[g] = (deltas of row g) << 32 | (slots of row g); packed[rows] = 0.
// One exclusive scan of it gives the new row offsets (low word) and the start
// of each row's delta bucket (high word). Also the new row lengths and their
// sum (the new zero-point count).
__global__ void k_pack_len(const uint32_t* __restrict__ off, const uint32_t* __restrict__ old_len,
                           const int32_t* __restrict__ add_cnt,
                           const int32_t* __restrict__ rem_cnt,
                           unsigned long long* __restrict__ packed, uint32_t* __restrict__ new_len,
                           uint32_t* __restrict__ new_cap, unsigned long long* __restrict__ total,
                           size_t rows) {
  unsigned long long sum = 0;
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g <= rows;
       g += size_t(gridDim.x) * blockDim.x) {
    if (g == rows) {
      packed[g] = 0ull;
      continue;
    }
    const uint32_t n0 = old_len ? old_len[g] : off[g + 1] - off[g];
    const uint32_t len = n0 + uint32_t(add_cnt[g]) - uint32_t(rem_cnt[g]);
    const uint32_t nd = uint32_t(add_cnt[g] + rem_cnt[g]);
    packed[g] = (static_cast<unsigned long long>(nd) << 32) | slot_capacity(len);
    new_len[g] = len;
    new_cap[g] = slot_capacity(len);
    sum += len;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(total, sum);
}

// the delta records into their rows' buckets (order within a bucket is
// arbitrary; the merge does not depend on it)
__global__ void k_delta_scatter(const int32_t* __restrict__ cells, const int8_t* __restrict__ sign,
                                int n_cells, const SliceParam* __restrict__ slices, int S, int w,
                                const unsigned long long* __restrict__ packed_off,
                                uint32_t* __restrict__ cursor, float* __restrict__ rec_v,
                                int8_t* __restrict__ rec_s) {
  const int total = n_cells * S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int k = i / S, s = i % S;
    const int cell = cells[k];
    const SliceParam sp = slices[s];
    int r0, r1;
    float v;
    pixel_rows_u(sp, cell % w, cell / w, r0, r1, v);
    for (int r = r0; r <= r1; r++) {
      const uint32_t g = sp.row_base + uint32_t(r);
      const uint32_t pos = uint32_t(packed_off[g] >> 32) + atomicAdd(&cursor[g], 1u);
      rec_v[pos] = v;
      rec_s[pos] = sign[k];
    }
  }
}

// first index in v[0, n) whose value is > x (upper) or >= x (lower)
__device__ __forceinline__ uint32_t row_bound(const float* __restrict__ v, uint32_t n, float x,
                                              bool upper) {
  uint32_t lo = 0, len = n;
  while (len > 0) {
    const uint32_t half = len >> 1, mid = lo + half;
    const float e = v[mid];
    if (upper ? !(x < e) : (e < x)) {
      lo = mid + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

// The row record of a merged row (cddt_device.cuh "Row records"): CSR range
// and the probes of its first search levels, read back from the new row.
__device__ __forceinline__ void write_row_record(float* __restrict__ hints, size_t g, uint32_t lo,
                                                 const float* __restrict__ v, uint32_t n) {
  float h[kHintFloats];
  int slot = 0;
  h[slot++] = __uint_as_float(lo);
  h[slot++] = __uint_as_float(n);
  for (int level = 0; level < kHintLevels; level++)
    for (uint32_t path = 0; path < (1u << level) && slot < kHintFloats; path++, slot++) {
      uint32_t idx;
      h[slot] = hint_index(n, level, path, &idx) ? v[idx] : 0.f;
    }
  for (; slot < kHintFloats; slot++) h[slot] = 0.f;
  for (int k = 0; k < kHintFloats; k += 4)
    reinterpret_cast<float4*>(hints + g * kHintFloats)[k / 4] =
        make_float4(h[k], h[k + 1], h[k + 2], h[k + 3]);
}

// Merge each row's delta records into its zero points, one warp per row
// (Cddt::add/remove_pixel_points: insert keeps the row sorted, remove drops
// one equal element; cddt.cpp:332-377, cddt.hpp:67-84). Equal values are
// identical floats, so the merged row is the sorted multiset
//   old - removed copies + added values,
// which a warp builds in parallel for rows with at most 32 records, in any
// order: every remove claims the next unclaimed copy of its value (ranked
// among the equal removes by lane); a kept old element lands at (its index -
// removed before it + adds smaller than it); an add lands after the kept
// copies <= its value, the smaller adds and the equal adds of lower lanes.
// Rows with more records: lane 0 sorts the bucket by value and merges
// sequentially. Also writes the new CSR offsets (low word of packed_off) and
// the row records: an unchanged row only moves (its record's lo), a merged
// row's record is rebuilt from the new row.
__global__ void k_merge_rows(const uint32_t* __restrict__ old_off,
                             const uint32_t* __restrict__ old_len, const float* __restrict__ old_zp,
                             const unsigned long long* __restrict__ packed_off,
                             uint32_t* __restrict__ new_off_out, float* __restrict__ new_zp,
                             const int32_t* __restrict__ add_cnt,
                             const int32_t* __restrict__ rem_cnt, float* __restrict__ rec_v,
                             int8_t* __restrict__ rec_s, size_t rows,
                             unsigned* __restrict__ unmatched, float* __restrict__ hints) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  const size_t warp = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;
  if (warp == 0 && lane == 0) new_off_out[rows] = uint32_t(packed_off[rows]);
  for (size_t g = warp; g < rows; g += nwarps) {
    const uint32_t a = old_off[g], b = old_len ? a + old_len[g] : old_off[g + 1];
    const unsigned long long po = packed_off[g];
    const uint32_t o = uint32_t(po);
    if (lane == 0) new_off_out[g] = o;
    const unsigned nd = unsigned(add_cnt[g] + rem_cnt[g]);
    if (nd == 0) {  // unchanged row: copy, four loads in flight per lane
      uint32_t i = a + lane;
      for (; i + 96 < b; i += 128) {
        const float v0 = __ldcs(old_zp + i), v1 = __ldcs(old_zp + i + 32);
        const float v2 = __ldcs(old_zp + i + 64), v3 = __ldcs(old_zp + i + 96);
        float* d = new_zp + o + (i - a);
        d[0] = v0;
        d[32] = v1;
        d[64] = v2;
        d[96] = v3;
      }
      for (; i < b; i += 32) new_zp[o + (i - a)] = __ldcs(old_zp + i);
      if (lane == 0) hints[g * kHintFloats] = __uint_as_float(o);  // the record's lo
      continue;
    }
    const unsigned j0 = unsigned(po >> 32);  // this row's delta bucket
    const uint32_t new_n = (b - a) + uint32_t(add_cnt[g]) - uint32_t(rem_cnt[g]);
    const float* __restrict__ row = old_zp + a;
    const uint32_t n = b - a;
    if (nd <= 32) {
      const bool has = lane < nd;
      const float dv = has ? rec_v[j0 + lane] : 0.f;
      const bool add = has && rec_s[j0 + lane] > 0, rem = has && !add;
      const unsigned add_mask = __ballot_sync(0xffffffffu, add);
      const unsigned rem_mask = __ballot_sync(0xffffffffu, rem);
      // removes: the k-th remove of value v drops old copy lower_bound(v) + k
      const unsigned same = __match_any_sync(0xffffffffu, __float_as_uint(dv)) & rem_mask;
      uint32_t ridx = 0xffffffffu;
      if (rem) {
        const uint32_t p = row_bound(row, n, dv, false) + __popc(same & lt);
        if (p < n && row[p] == dv)
          ridx = p;
        else
          atomicAdd(unmatched, 1u);
      }
      // adds: after the kept copies <= dv, the smaller adds and the equal adds of lower lanes
      unsigned rem_le = 0, adds_before = 0;
      for (unsigned l = 0; l < nd; l++) {
        const float dl = __shfl_sync(0xffffffffu, dv, l);
        rem_le += ((rem_mask >> l) & 1u) && !(dv < dl) ? 1u : 0u;
        adds_before += ((add_mask >> l) & 1u) && (dl < dv || (dl == dv && l < lane)) ? 1u : 0u;
      }
      if (add) new_zp[o + row_bound(row, n, dv, true) - rem_le + adds_before] = dv;
      // kept old elements, 32 at a time
      for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const float e = i < n ? row[i] : 0.f;
        bool removed = false;
        unsigned rb = 0, adds_lt = 0;
        for (unsigned l = 0; l < nd; l++) {
          const uint32_t rl = __shfl_sync(0xffffffffu, ridx, l);
          const float dl = __shfl_sync(0xffffffffu, dv, l);
          removed |= rl == i;
          rb += rl < i ? 1u : 0u;
          adds_lt += ((add_mask >> l) & 1u) && dl < e ? 1u : 0u;
        }
        if (i < n && !removed) new_zp[o + i - rb + adds_lt] = e;
      }
      __syncwarp();  // the warp's stores of the new row are visible to lane 0
      if (lane == 0) write_row_record(hints, g, o, new_zp + o, new_n);
      continue;
    }
    if (lane != 0) continue;
    // many records: sort the bucket by value (insertion sort; equal values in
    // any order give the same multiset), then merge sequentially
    float* bv = rec_v + j0;
    int8_t* bs = rec_s + j0;
    for (unsigned x = 1; x < nd; x++) {
      const float v = bv[x];
      const int8_t sg = bs[x];
      unsigned y = x;
      for (; y > 0 && v < bv[y - 1]; y--) {
        bv[y] = bv[y - 1];
        bs[y] = bs[y - 1];
      }
      bv[y] = v;
      bs[y] = sg;
    }
    unsigned j = 0;
    uint32_t i = a, w = o;
    unsigned miss = 0;
    while (i < b || j < nd) {
      if (j < nd) {
        const float dv = bv[j];
        if (i == b || dv < old_zp[i]) {
          if (bs[j] > 0)
            new_zp[w++] = dv;
          else
            miss++;
          j++;
          continue;
        }
        if (dv == old_zp[i]) {
          if (bs[j] > 0) {
            new_zp[w++] = dv;
          } else {
            i++;  // remove_one: drop one equal element
          }
          j++;
          continue;
        }
      }
      new_zp[w++] = old_zp[i++];
    }
    if (miss) atomicAdd(unmatched, miss);
    write_row_record(hints, g, o, new_zp + o, new_n);
  }
}

static int blocks_for(size_t work, int threads, int cap_per_sm = 16) {
  size_t b = (work + threads - 1) / threads;
  size_t cap = size_t(sm_count()) * cap_per_sm;
  return int(std::max<size_t>(1, std::min(b, cap)));
}

// ---- the batch replayed on the device ----
//
// Cddt::set_occupancy applied cell by cell in order (cddt.cpp:332-377) ends
// in the state of a fresh build of the final grid (the reference's invariant,
// proj/tests/test_cddt.cpp:578-604), so a batch reduces to: the final
// occupancy of every touched cell (the last edit of a cell wins), the flags
// of the changed cells' 3x3 dilation recomputed from it, and the membership
// flips there (the delta pixels, +1 joins / -1 leaves). Three small kernels;
// per-cell generation stamps pick the last edit and deduplicate the dilation
// without clearing anything between batches.

// control words of a batch (zeroed by its upload)
enum : int {
  kCtlRows = 0,      // touched-row list length (in place)
  kCtlStatus = 1,    // 1: a bucket overflowed, 2: the append area is exhausted
  kCtlMissed = 2,    // removals that found no stored point
  kCtlAppend = 3,    // append slots reserved
  kCtlNet = 4,       // net point change (i64, words 4-5)
  kCtlChanged = 6,   // cells whose occupancy changed
  kCtlDeltas = 7,    // delta pixels
  kCtlWords = 8
};
constexpr int kEditBits = 20;  // edit index bits of a stamp (batches go in chunks of 2^20)

// every edit stamps its cell with (generation, index): the largest index wins
__global__ void k_replay_stamp(const int32_t* __restrict__ xy, int n, int w,
                               uint32_t* __restrict__ stamp, uint32_t gen) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    atomicMax(&stamp[size_t(xy[2 * k + 1]) * w + xy[2 * k]], (gen << kEditBits) | uint32_t(k));
}

// the last edit of each cell sets its occupancy; changed cells are listed
__global__ void k_replay_apply(const int32_t* __restrict__ xy, const uint8_t* __restrict__ occ,
                               int n, int w, const uint32_t* __restrict__ stamp, uint32_t gen,
                               uint8_t* __restrict__ flags, int32_t* __restrict__ changed,
                               unsigned* __restrict__ ctl) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const size_t cell = size_t(xy[2 * k + 1]) * w + xy[2 * k];
    if (stamp[cell] != ((gen << kEditBits) | uint32_t(k))) continue;  // a later edit wins
    const uint8_t f = flags[cell];
    const bool o = occ[k] != 0;
    if (o == ((f & kOcc) != 0)) continue;
    flags[cell] = o ? uint8_t(f | kOcc) : uint8_t(f & ~kOcc);
    changed[atomicAdd(&ctl[kCtlChanged], 1u)] = int32_t(cell);
  }
}

// The 3x3 dilation of the changed cells (each cell once: the first thread to
// raise its stamp to this generation): occupancy / clear / membership flags
// from the final occupancy (is_edge_cell, grid.cpp:110-119; clear_around,
// cddt.cpp:173-180), the same bits in the query bitmaps, and the membership
// flips as delta pixels. Only clear/member bits are written here, so the
// occupancy bits other threads read are final.
__global__ void k_replay_flags(const int32_t* __restrict__ changed, int w, int h, int wpr,
                               uint32_t* __restrict__ wstamp, uint32_t gen,
                               uint8_t* __restrict__ flags, uint2* __restrict__ bits,
                               int32_t* __restrict__ dcells, int8_t* __restrict__ dsign,
                               unsigned* __restrict__ ctl) {
  const unsigned m = ctl[kCtlChanged] * 9u;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int32_t c0 = changed[i / 9];
    const int x = c0 % w + int(i % 9) % 3 - 1, y = c0 / w + int(i % 9) / 3 - 1;
    if (x < 0 || y < 0 || x >= w || y >= h) continue;
    const size_t q = size_t(y) * w + x;
    if (atomicMax(&wstamp[q], gen) >= gen) continue;  // another thread has this cell
    const uint8_t old = flags[q];
    const bool o = (old & kOcc) != 0;
    bool any_occ = false, any_free = false;
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        if (dx == 0 && dy == 0) continue;
        const int nx = x + dx, ny = y + dy;
        if (nx < 0 || ny < 0 || nx >= w || ny >= h || !(flags[size_t(ny) * w + nx] & kOcc))
          any_free = true;
        else
          any_occ = true;
      }
    const bool member = o && any_free;
    const bool clear = !o && !any_occ;
    uint8_t f = o ? kOcc : 0;
    if (clear) f |= kClear;
    if (member) f |= kMember;
    flags[q] = f;
    unsigned* word = reinterpret_cast<unsigned*>(bits + size_t(y) * wpr + (x >> 5));
    const unsigned bit = 1u << (x & 31);
    if (o)
      atomicOr(word, bit);
    else
      atomicAnd(word, ~bit);
    if (clear)
      atomicOr(word + 1, bit);
    else
      atomicAnd(word + 1, ~bit);
    if (member != ((old & kMember) != 0)) {
      const unsigned d = atomicAdd(&ctl[kCtlDeltas], 1u);
      dcells[d] = int32_t(q);
      dsign[d] = member ? int8_t(1) : int8_t(-1);
    }
  }
}

// The batch's membership deltas on the device: pixels and +1 (joins) / -1
// (leaves); *n_dev their count (the host learns it as `n` only when the
// relayout needs it).
struct EditBatch {
  const int32_t* cells;
  const int8_t* sign;
  const unsigned* n_dev;
  int n_bound;  // upper bound on the count (launch sizing)
  int n;        // the count, when known on the host
};
static int edits_relayout(rl_cddt* c, const EditBatch& e);
static int edits_in_place(rl_cddt* c, const EditBatch& e, unsigned* ctl, bool* applied);

// Apply edits [0, n) (already validated) to the structure, in order: chunks
// of 2^20 edits (the stamp's index field), each replayed on the device.
static int apply_chunk(rl_cddt* c, const int32_t* xy, const uint8_t* occ, size_t n);
static int apply_edits(rl_cddt* c, const int32_t* xy, const uint8_t* occ, size_t n) {
  constexpr size_t kChunk = size_t(1) << kEditBits;
  for (size_t off = 0; off < n; off += kChunk)
    RL_TRY(apply_chunk(c, xy + 2 * off, occ + off, std::min(kChunk, n - off)));
  return RL_OK;
}

static int apply_chunk(rl_cddt* c, const int32_t* xy, const uint8_t* occ, size_t n) {
  cudaStream_t st = c->stream;
  const size_t wh = size_t(c->w) * c->h;
  if (c->estamp.n != wh || c->wstamp.n != wh || c->edit_gen + 1 >= (1u << (32 - kEditBits))) {
    if (c->estamp.n != wh) RL_TRY(c->estamp.alloc(wh));
    if (c->wstamp.n != wh) RL_TRY(c->wstamp.alloc(wh));
    RL_CK(cudaMemsetAsync(c->estamp.p, 0, 4 * wh, st));
    RL_CK(cudaMemsetAsync(c->wstamp.p, 0, 4 * wh, st));
    c->edit_gen = 0;
  }
  const uint32_t gen = ++c->edit_gen;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  // one upload through pinned staging: xy | occ | control words (zeroed)
  const size_t up_sizes[] = {8 * n, n, 4 * kCtlWords};
  size_t up = 0;
  for (size_t b : up_sizes) up += al(b);
  if (c->upd_host_n < up) {
    if (c->upd_host) cudaFreeHost(c->upd_host);
    c->upd_host = nullptr;
    c->upd_host_n = 0;
    RL_CK(cudaMallocHost(&c->upd_host, up + up / 4));
    c->upd_host_n = up + up / 4;
  }
  // device scratch: the upload | changed cells (n) | delta cells (9n) | delta signs (9n)
  const size_t dev_sizes[] = {up, 4 * n, 36 * n, 9 * n};
  size_t need = 0;
  for (size_t b : dev_sizes) need += al(b);
  if (c->upd_up.n < need) RL_TRY(c->upd_up.alloc(need + need / 4));
  uint8_t* hbuf = static_cast<uint8_t*>(c->upd_host);
  std::memcpy(hbuf, xy, 8 * n);
  std::memcpy(hbuf + al(8 * n), occ, n);
  std::memset(hbuf + al(8 * n) + al(n), 0, 4 * kCtlWords);
  RL_CK(cudaMemcpyAsync(c->upd_up.p, hbuf, up, cudaMemcpyHostToDevice, st));
  const int32_t* d_xy = reinterpret_cast<const int32_t*>(c->upd_up.p);
  const uint8_t* d_occ = c->upd_up.p + al(8 * n);
  unsigned* ctl = reinterpret_cast<unsigned*>(c->upd_up.p + al(8 * n) + al(n));
  int32_t* changed = reinterpret_cast<int32_t*>(c->upd_up.p + up);
  int32_t* dcells = reinterpret_cast<int32_t*>(c->upd_up.p + up + al(4 * n));
  int8_t* dsign = reinterpret_cast<int8_t*>(c->upd_up.p + up + al(4 * n) + al(36 * n));
  const int nb = blocks_for(n, 256, 4);
  k_replay_stamp<<<nb, 256, 0, st>>>(d_xy, int(n), c->w, c->estamp.p, gen);
  k_replay_apply<<<nb, 256, 0, st>>>(d_xy, d_occ, int(n), c->w, c->estamp.p, gen, c->flags.p,
                                     changed, ctl);
  k_replay_flags<<<blocks_for(9 * n, 256, 4), 256, 0, st>>>(changed, c->w, c->h, c->wpr,
                                                            c->wstamp.p, gen, c->flags.p,
                                                            c->rowbits.p, dcells, dsign, ctl);
  RL_CK(cudaGetLastError());
  c->mirror_stale = true;
  EditBatch e{dcells, dsign, ctl + kCtlDeltas, int(9 * n), -1};
  if (c->gapped) {  // the touched rows only
    bool applied = false;
    RL_TRY(edits_in_place(c, e, ctl, &applied));
    if (applied) return finish(c, nullptr);
  } else {
    uint32_t* hs = nullptr;
    RL_TRY(host_small(c, &hs));
    RL_CK(cudaMemcpyAsync(hs, ctl, 4 * kCtlWords, cudaMemcpyDeviceToHost, st));
    RL_CK(cudaStreamSynchronize(st));
  }
  uint32_t* hs = nullptr;
  RL_TRY(host_small(c, &hs));
  e.n = int(hs[kCtlDeltas]);
  if (e.n) RL_TRY(edits_relayout(c, e));
  return finish(c, nullptr);
}

// All rows to fresh slots (slot_capacity) with the batch's deltas merged:
// the first batch on a dense structure, and any batch a row outgrows its
// slots in (or with more than kBucket records for one row).
static int edits_relayout(rl_cddt* c, const EditBatch& e) {
#ifdef RL_EDIT_PROFILE
  fprintf(stderr, "relayout: %zu slots in use of %zu\n", size_t(c->zp_slots), size_t(c->zp.n));
#endif
  cudaStream_t st = c->stream;
  const size_t rows = c->rows;
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (unsigned long long*)nullptr,
                                (unsigned long long*)nullptr, int(rows + 1), st);
  const size_t cap = size_t(e.n) * c->S * 3;  // a unit square spans at most 3 rows
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  // one persistent workspace, carved in 256-byte aligned pieces
  const size_t sizes[] = {12 * rows, 8 * (rows + 1), 8 * (rows + 1), 4 * cap, cap, 16, scan_tmp};
  size_t need = 0;
  for (size_t b : sizes) need += al(b);
  if (c->upd_ws.n < need) RL_TRY(c->upd_ws.alloc(need + need / 4));
  uint8_t* cur = c->upd_ws.p;
  auto take = [&](size_t b) {
    uint8_t* p = cur;
    cur += al(b);
    return p;
  };
  int32_t* add_cnt = reinterpret_cast<int32_t*>(take(sizes[0]));  // add | rem | cursor
  int32_t* rem_cnt = add_cnt + rows;
  uint32_t* cursor = reinterpret_cast<uint32_t*>(rem_cnt + rows);
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(take(sizes[1]));
  unsigned long long* packed_off = reinterpret_cast<unsigned long long*>(take(sizes[2]));
  float* rec_v = reinterpret_cast<float*>(take(sizes[3]));
  int8_t* rec_s = reinterpret_cast<int8_t*>(take(sizes[4]));
  unsigned long long* ctl = reinterpret_cast<unsigned long long*>(take(sizes[5]));  // total | unmatched
  void* tmp = take(sizes[6]);

  // per-row delta counts -> one scan (new offsets | delta buckets) -> records into buckets
  RL_CK(cudaMemsetAsync(add_cnt, 0, 12 * rows, st));
  RL_CK(cudaMemsetAsync(ctl, 0, 16, st));
  if (c->len_spare.n < rows) RL_TRY(c->len_spare.alloc(rows));
  if (c->cap_spare.n < rows) RL_TRY(c->cap_spare.alloc(rows));
  const int db = blocks_for(size_t(e.n) * c->S, 256);
  k_delta_count<<<db, 256, 0, st>>>(e.cells, e.sign, e.n, c->d_slices.p, c->S, c->w, add_cnt,
                                    rem_cnt);
  k_pack_len<<<blocks_for(rows + 1, 256), 256, 0, st>>>(
      c->row_off.p, c->gapped ? c->row_len.p : nullptr, add_cnt, rem_cnt, packed, c->len_spare.p,
      c->cap_spare.p, ctl, rows);
  RL_CK(cub::DeviceScan::ExclusiveSum(tmp, scan_tmp, packed, packed_off, int(rows + 1), st));
  k_delta_scatter<<<db, 256, 0, st>>>(e.cells, e.sign, e.n, c->d_slices.p, c->S, c->w, packed_off,
                                      cursor, rec_v, rec_s);
  RL_CK(cudaGetLastError());
  // merge into the spare buffers (the new offsets too), then swap
  if (c->off_spare.n < rows + 1) RL_TRY(c->off_spare.alloc(rows + 1));
  const size_t pts = c->zero_points + cap;  // bound on the new point count
  const size_t slots_ub = pts + pts / 8 + 4 * rows;
  if (slots_ub >= (size_t(1) << 31)) {
    set_error("cddt: %zu zero-point slots exceed the 31-bit CSR offset", slots_ub);
    return RL_EINVAL;
  }
  // plus an append area for rows that outgrow their slots in later batches
  // (RL_EDIT_APPEND_SLOTS overrides its size: a test hook for the exhausted-area path)
  static const long long append_env = [] {
    const char* v = std::getenv("RL_EDIT_APPEND_SLOTS");
    return (v && *v) ? std::atoll(v) : -1ll;
  }();
  const size_t append = std::max(slots_ub / 4, size_t(1) << 20);
  const size_t slots_buf = std::min(slots_ub + append, (size_t(1) << 31) - 1);
  // (with headroom: a structure that keeps growing would otherwise reallocate
  // - a synchronous free and malloc of the whole array - at every relayout)
  if (c->zp_spare.n < slots_buf)
    RL_TRY(c->zp_spare.alloc(std::min(slots_buf + slots_buf / 4, (size_t(1) << 31) - 1)));
  k_merge_rows<<<blocks_for(rows * 32, 256, 32), 256, 0, st>>>(
      c->row_off.p, c->gapped ? c->row_len.p : nullptr, c->zp.p, packed_off, c->off_spare.p,
      c->zp_spare.p, add_cnt, rem_cnt, rec_v, rec_s, rows,
      reinterpret_cast<unsigned*>(ctl + 1), c->hints.p);
  RL_CK(cudaGetLastError());
  uint32_t* hs = nullptr;  // pinned: {slots, -, total points (u64), missed removals}
  RL_TRY(host_small(c, &hs));
  RL_CK(cudaMemcpyAsync(&hs[0], packed_off + rows, 4, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaMemcpyAsync(&hs[2], ctl, 12, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
  uint64_t total = 0;
  std::memcpy(&total, &hs[2], 8);
  if (hs[4]) {
    set_error("cddt: %u zero-point removals found no stored point (structure inconsistent)",
              hs[4]);
    return RL_ELOGIC;
  }
  std::swap(c->zp, c->zp_spare);
  std::swap(c->row_off, c->off_spare);  // the row records were rewritten by k_merge_rows
  std::swap(c->row_len, c->len_spare);
  std::swap(c->row_cap, c->cap_spare);
  c->zero_points = total;
  c->zp_slots = hs[0];
  c->slot_limit = append_env >= 0 ? std::min<uint64_t>(c->zp.n, c->zp_slots + append_env)
                                  : c->zp.n;
  c->gapped = true;
  return RL_OK;
}

// ---- in place: only the touched rows ----
//
// Each touched row is merged where it lies when the merged row fits its slots
// and the moved middle fits the warp's registers; otherwise it is rewritten
// into fresh slots from the append area past zp_slots (and its record, offset
// and capacity follow it). Only when the append area is exhausted, or a row
// receives more than kBucket records, does the batch fall back to
// edits_relayout — decided before anything is written.

constexpr int kBucket = 32;               // delta records per row and batch (the warp merge's width)
#ifndef RL_MID_REGS
#define RL_MID_REGS 8
#endif
constexpr int kMidRegs = RL_MID_REGS;     // middle elements per lane held in registers
constexpr int kMidMax = 32 * kMidRegs;    // longest middle merged in place
constexpr int kMergeWarps = 4;            // warps per CTA of the plan and merge kernels

// bkt layout (c->bkt): counts[rows] (zero between batches) | values[rows][kBucket] |
// kinds[rows][kBucket] | planned positions[rows][kBucket] | touched-row list[rows] |
// plan per list entry. The control words live in the batch's upload (zeroed).
struct BucketView {
  uint32_t* cnt;
  float* val;
  int8_t* sgn;     // +1 add, -1 remove; the plan sets 0 for a remove with no stored copy
  uint32_t* pos;   // planned: a remove's claimed index, an add's insert position
  uint32_t* list;
  uint4* span;     // planned: {pmin, pend, net, new first slot or ~0u (in place)}
  unsigned* ctl;   // the batch's control words (kCtl*)
  long long* net;
};

// every (delta pixel, slice, row) record into its row's bucket; the first
// record of a row lists the row
__global__ void k_bucket(EditBatch e, const SliceParam* __restrict__ slices, int S, int w,
                         BucketView b) {
  const unsigned total = *e.n_dev * unsigned(S);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += gridDim.x * blockDim.x) {
    const int k = int(i / S), s = int(i % S);
    const int cell = e.cells[k];
    const SliceParam sp = slices[s];
    int r0, r1;
    float v;
    pixel_rows_u(sp, cell % w, cell / w, r0, r1, v);
    for (int r = r0; r <= r1; r++) {
      const uint32_t g = sp.row_base + uint32_t(r);
      const uint32_t slot = atomicAdd(&b.cnt[g], 1u);
      if (slot == 0) b.list[atomicAdd(&b.ctl[kCtlRows], 1u)] = g;
      if (slot < kBucket) {
        b.val[size_t(g) * kBucket + slot] = v;
        b.sgn[size_t(g) * kBucket + slot] = e.sign[k];
      } else {
        atomicOr(&b.ctl[kCtlStatus], 1u);
      }
    }
  }
}

// Where a row's bucket lands (the order-free merge of k_merge_rows, per
// lane = per record): a remove claims old copy lower_bound(v) + its rank among
// the equal removes; an add goes in at upper_bound(v). Old elements before
// the first claimed/insert position keep their index, those from `pend` on
// all shift by `net`; only the middle [pmin, pend) moves irregularly.
struct MergePlan {
  float dv;
  bool add, rem;       // rem: a remove that found its copy
  uint32_t pos;        // rem: the claimed index; add: the insert position
  unsigned add_mask, rem_mask;
  uint32_t pmin, pend;
  int net;
};

// new index of old element i (value x) of the middle; false: removed
__device__ __forceinline__ bool middle_dest(const MergePlan& p, uint32_t i, float x,
                                            uint32_t* dst) {
  bool removed = false;
  unsigned rb = 0, adds_lt = 0;
  for (unsigned any = p.add_mask | p.rem_mask; any; any &= any - 1) {  // warp-uniform
    const unsigned l = __ffs(any) - 1;
    const uint32_t pl = __shfl_sync(0xffffffffu, p.pos, l);
    const float dl = __shfl_sync(0xffffffffu, p.dv, l);
    if ((p.rem_mask >> l) & 1u) {
      removed |= pl == i;
      rb += pl < i ? 1u : 0u;
    } else {
      adds_lt += dl < x ? 1u : 0u;
    }
  }
  *dst = i - rb + adds_lt;
  return !removed;
}

// new index of this lane's add: after the kept copies <= dv, the smaller adds
// and the equal adds of lower lanes (call from every lane: it shuffles)
__device__ __forceinline__ uint32_t add_dest(const MergePlan& p) {
  const unsigned lane = threadIdx.x & 31;
  unsigned rem_lt = 0, adds_before = 0;
  for (unsigned any = p.add_mask | p.rem_mask; any; any &= any - 1) {  // warp-uniform
    const unsigned l = __ffs(any) - 1;
    const uint32_t pl = __shfl_sync(0xffffffffu, p.pos, l);
    const float dl = __shfl_sync(0xffffffffu, p.dv, l);
    if ((p.rem_mask >> l) & 1u)
      rem_lt += pl < p.pos ? 1u : 0u;
    else
      adds_before += (dl < p.dv || (dl == p.dv && l < lane)) ? 1u : 0u;
  }
  return p.pos - rem_lt + adds_before;
}

// Per touched row (one warp): the record positions, the middle, and whether
// the row merges in place or into fresh slots from the append area. All
// reservations are made here, so an exhausted append area is known before
// anything is written.
__global__ void __launch_bounds__(32 * kMergeWarps) k_bucket_plan(
    BucketView b, const uint32_t* __restrict__ off, const uint32_t* __restrict__ cap,
    const uint32_t* __restrict__ len, const float* __restrict__ zp, uint32_t append_base,
    uint32_t slots_total) {
  const unsigned lane = threadIdx.x & 31, lt = (1u << lane) - 1;
  const unsigned m = b.ctl[kCtlRows];
  if (b.ctl[kCtlStatus]) return;  // a bucket overflowed: relayout
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
  for (unsigned j = warp; j < m; j += nwarps) {
    const uint32_t g = b.list[j];
    const unsigned nd = b.cnt[g];
    const uint32_t n = len[g];
    const float* __restrict__ row = zp + off[g];
    const size_t r0 = size_t(g) * kBucket;
    const bool has = lane < nd;
    const float dv = has ? b.val[r0 + lane] : 0.f;
    const bool add = has && b.sgn[r0 + lane] > 0;
    bool rem = has && !add;
    const unsigned rem_all = __ballot_sync(0xffffffffu, rem);
    const unsigned same = __match_any_sync(0xffffffffu, __float_as_uint(dv)) & rem_all;
    uint32_t pos = 0;
    if (rem) {
      const uint32_t q = row_bound(row, n, dv, false) + __popc(same & lt);
      if (q < n && row[q] == dv) {
        pos = q;
      } else {
        rem = false;
        b.sgn[r0 + lane] = 0;  // missed: reported by the merge
      }
    }
    if (add) pos = row_bound(row, n, dv, true);
    if (has) b.pos[r0 + lane] = pos;
    const int net = __popc(__ballot_sync(0xffffffffu, add)) - __popc(__ballot_sync(0xffffffffu, rem));
    uint32_t lo = (add || rem) ? pos : 0xffffffffu;
    uint32_t hi = rem ? pos + 1 : (add ? pos : 0u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const uint32_t pmin = lo == 0xffffffffu ? n : lo, pend = hi < pmin ? pmin : hi;
    if (lane == 0) {
      const uint32_t nn = uint32_t(int(n) + net);
      uint32_t target = ~0u;
      if (nn > cap[g] || pend - pmin > uint32_t(kMidMax)) {
        const uint32_t need = slot_capacity(nn);
        const uint32_t at = atomicAdd(&b.ctl[kCtlAppend], need);
        if (uint64_t(append_base) + at + need > slots_total)
          atomicOr(&b.ctl[kCtlStatus], 2u);
        else
          target = append_base + at;
      }
      b.span[j] = make_uint4(pmin, pend, uint32_t(net), target);
    }
  }
}

// One warp per touched row: the planned merge, in place or into its fresh
// slots; then the row's record, length (offset and capacity when it moved).
// With a status flag set nothing is written (the batch goes to
// edits_relayout); the counts are zeroed either way.
__global__ void __launch_bounds__(32 * kMergeWarps) k_merge_touched(
    BucketView b, uint32_t* __restrict__ off, uint32_t* __restrict__ cap,
    uint32_t* __restrict__ len, float* __restrict__ zp, float* __restrict__ hints) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned m = b.ctl[kCtlRows];
  const bool skip = b.ctl[kCtlStatus] != 0;
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nwarps = (gridDim.x * blockDim.x) >> 5;
  long long net = 0;
  unsigned missed = 0;
  for (unsigned j = warp; j < m; j += nwarps) {
    const uint32_t g = b.list[j];
    if (skip) {
      if (lane == 0) b.cnt[g] = 0;
      continue;
    }
    const unsigned nd = b.cnt[g];
    const uint32_t lo = off[g], n = len[g];
    const float* row = zp + lo;
    const uint4 sp = b.span[j];
    const size_t r0 = size_t(g) * kBucket;
    MergePlan p;
    const bool has = lane < nd;
    const int8_t kind = has ? b.sgn[r0 + lane] : int8_t(0);
    p.dv = has ? b.val[r0 + lane] : 0.f;
    p.pos = has ? b.pos[r0 + lane] : 0u;
    p.add = kind > 0;
    p.rem = kind < 0;
    missed += (has && kind == 0) ? 1u : 0u;
    p.add_mask = __ballot_sync(0xffffffffu, p.add);
    p.rem_mask = __ballot_sync(0xffffffffu, p.rem);
    p.pmin = sp.x;
    p.pend = sp.y;
    p.net = int(sp.z);
    const uint32_t target = sp.w;
    const uint32_t nn = uint32_t(int(n) + p.net);
    if (target != ~0u) {  // fresh slots: no overlap, straight copies around the middle
      float* dst = zp + target;
      for (uint32_t i = lane; i < p.pmin; i += 32) dst[i] = row[i];
      for (uint32_t i = p.pend + lane; i < n; i += 32) dst[int(i) + p.net] = row[i];
      for (uint32_t base = p.pmin; base < p.pend; base += 32) {  // warp-uniform trips
        const uint32_t i = base + lane;
        const float x = i < p.pend ? row[i] : 0.f;
        uint32_t d;
        const bool keep = middle_dest(p, i, x, &d);
        if (i < p.pend && keep) dst[d] = x;
      }
      const uint32_t ad = add_dest(p);  // every lane: add_dest shuffles
      if (p.add) dst[ad] = p.dv;
    } else {
      float* dst = zp + lo;
      // the middle into registers before anything moves
      float mid[kMidRegs];
#pragma unroll
      for (int k = 0; k < kMidRegs; k++) {
        const uint32_t i = p.pmin + lane + 32u * k;
        mid[k] = i < p.pend ? row[i] : 0.f;
      }
      // the tail [pend, n) shifts by net, kTailGroup chunks of 32 per round
      // trip: groups from the far end when it grows, from the near end when it
      // shrinks (each group is read before it is written)
      if (p.net != 0 && p.pend < n) {
        constexpr uint32_t kG = 32u * kMidRegs;
        const uint32_t span = n - p.pend, groups = (span + kG - 1) / kG;
        for (uint32_t q = 0; q < groups; q++) {
          const uint32_t g0 = p.pend + (p.net > 0 ? (groups - 1 - q) : q) * kG;
          float t[kMidRegs];
#pragma unroll
          for (int k = 0; k < kMidRegs; k++) {
            const uint32_t i = g0 + lane + 32u * k;
            t[k] = i < n ? row[i] : 0.f;
          }
          __syncwarp();
#pragma unroll
          for (int k = 0; k < kMidRegs; k++) {
            const uint32_t i = g0 + lane + 32u * k;
            if (i < n) dst[int(i) + p.net] = t[k];
          }
          __syncwarp();
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kMidRegs; k++) {
        const uint32_t i = p.pmin + lane + 32u * k;
        if (p.pmin + 32u * k >= p.pend) break;  // warp-uniform
        uint32_t d;
        const bool keep = middle_dest(p, i, mid[k], &d);
        if (i < p.pend && keep) dst[d] = mid[k];
      }
      const uint32_t ad = add_dest(p);  // every lane: add_dest shuffles
      if (p.add) dst[ad] = p.dv;
    }
    __syncwarp();  // the warp's stores of the new row are visible to lane 0
    if (lane == 0) {
      const uint32_t at = target != ~0u ? target : lo;
      write_row_record(hints, g, at, zp + at, nn);
      len[g] = nn;
      if (target != ~0u) {
        off[g] = target;
        cap[g] = slot_capacity(nn);
      }
      b.cnt[g] = 0;
      net += (long long)nn - (long long)n;
    }
  }
  if (lane == 0 && net)
    atomicAdd(reinterpret_cast<unsigned long long*>(b.net), static_cast<unsigned long long>(net));
  if (missed) atomicAdd(&b.ctl[kCtlMissed], missed);
}

static int edits_in_place(rl_cddt* c, const EditBatch& e, unsigned* ctl, bool* applied) {
  *applied = false;
  cudaStream_t st = c->stream;
  const size_t rows = c->rows;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t sizes[] = {4 * rows, 4 * rows * kBucket, rows * kBucket, 4 * rows * kBucket,
                          4 * rows, 16 * rows};
  size_t need = 0;
  for (size_t s : sizes) need += al(s);
  if (c->bkt.n < need) {
    RL_TRY(c->bkt.alloc(need));
    RL_CK(cudaMemsetAsync(c->bkt.p, 0, al(sizes[0]), st));  // counts start (and stay) zero
  }
  uint8_t* cur = c->bkt.p;
  auto take = [&](size_t s) {
    uint8_t* p = cur;
    cur += al(s);
    return p;
  };
  BucketView b;
  b.cnt = reinterpret_cast<uint32_t*>(take(sizes[0]));
  b.val = reinterpret_cast<float*>(take(sizes[1]));
  b.sgn = reinterpret_cast<int8_t*>(take(sizes[2]));
  b.pos = reinterpret_cast<uint32_t*>(take(sizes[3]));
  b.list = reinterpret_cast<uint32_t*>(take(sizes[4]));
  b.span = reinterpret_cast<uint4*>(take(sizes[5]));
  b.ctl = ctl;
  b.net = reinterpret_cast<long long*>(ctl + kCtlNet);
  k_bucket<<<blocks_for(size_t(e.n_bound) * c->S, 256), 256, 0, st>>>(e, c->d_slices.p, c->S,
                                                                       c->w, b);
  // latency-bound warps (a chain of dependent loads per row): fill the GPU
  static const int plan_ctas = [] {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bucket_plan, 32 * kMergeWarps, 0);
    return sm_count() * std::max(per_sm, 1);
  }();
  static const int merge_ctas = [] {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_merge_touched, 32 * kMergeWarps, 0);
    return sm_count() * std::max(per_sm, 1);
  }();
  k_bucket_plan<<<plan_ctas, 32 * kMergeWarps, 0, st>>>(b, c->row_off.p, c->row_cap.p, c->row_len.p,
                                                 c->zp.p, uint32_t(c->zp_slots),
                                                 uint32_t(c->slot_limit));
  k_merge_touched<<<merge_ctas, 32 * kMergeWarps, 0, st>>>(b, c->row_off.p, c->row_cap.p, c->row_len.p,
                                                   c->zp.p, c->hints.p);
  RL_CK(cudaGetLastError());
  uint32_t* hs = nullptr;
  RL_TRY(host_small(c, &hs));
  RL_CK(cudaMemcpyAsync(hs, ctl, 4 * kCtlWords, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
#ifdef RL_EDIT_PROFILE
  fprintf(stderr, "in-place status %u rows %u appended %u of %zu free\n", hs[kCtlStatus], hs[kCtlRows], hs[kCtlAppend],
          size_t(c->zp.n - c->zp_slots));
#endif
  if (hs[kCtlStatus]) return RL_OK;  // nothing written: relayout
  if (hs[kCtlMissed]) {
    set_error("cddt: %u zero-point removals found no stored point (structure inconsistent)",
              hs[kCtlMissed]);
    return RL_ELOGIC;
  }
  long long net = 0;
  std::memcpy(&net, hs + kCtlNet, 8);
  c->zero_points = uint64_t((long long)c->zero_points + net);
  c->zp_slots += hs[kCtlAppend];
  *applied = true;
  return RL_OK;
}

// Slack rows back to dense CSR (before prune): one scan of the row lengths,
// one warp per row copying it down.
__global__ void k_len_wide(const uint32_t* __restrict__ len, uint32_t* __restrict__ out,
                           size_t rows) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g <= rows;
       g += size_t(gridDim.x) * blockDim.x)
    out[g] = g < rows ? len[g] : 0u;
}
__global__ void k_copy_rows(const uint32_t* __restrict__ off, const uint32_t* __restrict__ len,
                            const float* __restrict__ zp, const uint32_t* __restrict__ noff,
                            float* __restrict__ nzp, size_t rows) {
  const unsigned lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;
  for (size_t g = warp; g < rows; g += nwarps)
    for (uint32_t i = lane; i < len[g]; i += 32) nzp[noff[g] + i] = zp[off[g] + i];
}

}  // namespace rl

namespace rl {
int densify_rows(rl_cddt* c) {
  if (!c->gapped) return RL_OK;
  cudaStream_t st = c->stream;
  const size_t rows = c->rows;
  DevBuf<uint32_t> wide, noff;
  DevBuf<float> nzp;
  RL_TRY(wide.alloc(rows + 1));
  RL_TRY(noff.alloc(rows + 1));
  RL_TRY(nzp.alloc(c->zero_points));
  k_len_wide<<<blocks_for(rows + 1, 256), 256, 0, st>>>(c->row_len.p, wide.p, rows);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, wide.p, noff.p, int(rows + 1), st);
  DevBuf<uint8_t> tmp;
  RL_TRY(tmp.alloc(tmp_bytes));
  RL_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, wide.p, noff.p, int(rows + 1), st));
  k_copy_rows<<<blocks_for(rows * 32, 256, 32), 256, 0, st>>>(c->row_off.p, c->row_len.p,
                                                               c->zp.p, noff.p, nzp.p, rows);
  RL_CK(cudaGetLastError());
  RL_CK(cudaStreamSynchronize(st));
  c->zp = std::move(nzp);
  c->row_off = std::move(noff);
  c->row_len.release();
  c->len_spare.release();
  c->row_cap.release();
  c->cap_spare.release();
  c->zp_spare.release();
  c->off_spare.release();
  c->zp_slots = c->zero_points;
  c->gapped = false;
  RL_TRY(refresh_row_hints(c));
  RL_CK(cudaStreamSynchronize(st));
  return RL_OK;
}
}  // namespace rl

using namespace rl;

extern "C" {

int rl_cddt_set_occupancy_batch(rl_cddt* c, const int32_t* xy, const uint8_t* occupied,
                                size_t n) {
  if (!c || (n && (!xy || !occupied))) return RL_EINVAL;
  if (n == 0) return RL_OK;
  if (c->pruned) {
    set_error("cddt: incremental updates are disabled after prune");  // cddt.cpp:333
    return RL_ELOGIC;
  }
  size_t valid = n;
  for (size_t k = 0; k < n; k++) {
    const int x = xy[2 * k], y = xy[2 * k + 1];
    if (x < 0 || y < 0 || x >= c->w || y >= c->h) {
      valid = k;
      break;
    }
  }
  DeviceGuard guard(c->dev);
  if (valid) RL_TRY(quiesce(c));  // casts queued on caller streams read the rows being merged
  RL_TRY(apply_edits(c, xy, occupied, valid));
  if (valid < n) {
    set_error("cddt: cell outside the grid");  // cddt.cpp:334
    return RL_ERANGE;
  }
  return RL_OK;
}

int rl_cddt_set_occupancy(rl_cddt* c, int32_t x, int32_t y, int32_t occupied) {
  int32_t xy[2] = {x, y};
  uint8_t o = occupied ? 1 : 0;
  return rl_cddt_set_occupancy_batch(c, xy, &o, 1);
}

}  // extern "C"
