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

// packed[g] = (deltas of row g) << 32 | (new length of row g); packed[rows] = 0.
// One exclusive scan of it gives the new CSR offsets (low word) and the start
// of each row's delta bucket (high word).
__global__ void k_pack_len(const uint32_t* __restrict__ off, const int32_t* __restrict__ add_cnt,
                           const int32_t* __restrict__ rem_cnt,
                           unsigned long long* __restrict__ packed, size_t rows) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g <= rows;
       g += size_t(gridDim.x) * blockDim.x) {
    if (g == rows) {
      packed[g] = 0ull;
      continue;
    }
    const uint32_t len = (off[g + 1] - off[g]) + uint32_t(add_cnt[g]) - uint32_t(rem_cnt[g]);
    const uint32_t nd = uint32_t(add_cnt[g] + rem_cnt[g]);
    packed[g] = (static_cast<unsigned long long>(nd) << 32) | len;
  }
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
__global__ void k_merge_rows(const uint32_t* __restrict__ old_off, const float* __restrict__ old_zp,
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
    const uint32_t a = old_off[g], b = old_off[g + 1];
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

__global__ void k_set_flags(const int32_t* __restrict__ cells, const uint8_t* __restrict__ f,
                            int n, uint8_t* __restrict__ flags) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    flags[cells[i]] = f[i];
}

static int blocks_for(size_t work, int threads, int cap_per_sm = 16) {
  size_t b = (work + threads - 1) / threads;
  size_t cap = size_t(sm_count()) * cap_per_sm;
  return int(std::max<size_t>(1, std::min(b, cap)));
}

// Apply edits [0, n) (already validated) to the structure.
static int apply_edits(rl_cddt* c, const int32_t* xy, const uint8_t* occ, size_t n) {
  const int w = c->w, h = c->h;
  auto at = [&](int x, int y) { return c->grid_h[size_t(y) * w + x] != 0; };
  auto inb = [&](int x, int y) { return x >= 0 && y >= 0 && x < w && y < h; };
  // 1. the touched cells' original states, then replay in order (last writer
  //    wins); changed = touched cells whose final state differs
  std::vector<int32_t> touched(n);
  for (size_t k = 0; k < n; k++) touched[k] = xy[2 * k + 1] * w + xy[2 * k];
  std::sort(touched.begin(), touched.end());
  touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
  std::vector<uint8_t> orig(touched.size());
  for (size_t k = 0; k < touched.size(); k++) orig[k] = c->grid_h[touched[k]];
  for (size_t k = 0; k < n; k++) c->grid_h[size_t(xy[2 * k + 1]) * w + xy[2 * k]] = occ[k] ? 1 : 0;
  std::vector<int32_t> changed;
  for (size_t k = 0; k < touched.size(); k++)
    if (orig[k] != c->grid_h[touched[k]]) changed.push_back(touched[k]);
  if (changed.empty()) return RL_OK;
  // 2. flags in the dilation; membership deltas
  std::vector<int32_t> window;
  window.reserve(changed.size() * 9);
  for (int32_t cell : changed) {
    const int x = cell % w, y = cell / w;
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++)
        if (inb(x + dx, y + dy)) window.push_back((y + dy) * w + (x + dx));
  }
  std::sort(window.begin(), window.end());
  window.erase(std::unique(window.begin(), window.end()), window.end());
  std::vector<int32_t> wcells, dcells;
  std::vector<uint8_t> wflags;
  std::vector<int8_t> dsign;
  wcells.reserve(window.size());
  for (const int32_t cell : window) {
    const int x = cell % w, y = cell / w;
    const bool o = at(x, y);
    bool any_occ = false, any_free = false;
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        if (dx == 0 && dy == 0) continue;
        const int nx = x + dx, ny = y + dy;
        if (!inb(nx, ny) || !at(nx, ny))
          any_free = true;
        else
          any_occ = true;
      }
    const bool member = o && any_free;  // is_edge_cell (grid.cpp:110-119)
    uint8_t f = 0;
    if (o) f |= kOcc;
    if (!o && !any_occ) f |= kClear;  // clear_around (cddt.cpp:173-180)
    if (member) f |= kMember;
    wcells.push_back(cell);
    wflags.push_back(f);
    if (member != (c->member_h[cell] != 0)) {
      dcells.push_back(cell);
      dsign.push_back(member ? 1 : -1);
      c->member_h[cell] = member ? 1 : 0;
    }
  }
  cudaStream_t st = c->stream;
  const size_t nw = wcells.size();
  const int nd = int(dcells.size());
  const size_t rows = c->rows;
  size_t scan_tmp = 0;
  if (nd)
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, int(rows + 1), st);
  const size_t cap = size_t(nd) * c->S * 3;  // a unit square spans at most 3 rows
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  // uploads wcells | wflags | dcells | dsign, staged through pinned memory so
  // they go as one truly asynchronous copy
  const size_t up_sizes[] = {4 * nw, nw, 4 * size_t(nd), size_t(nd)};
  size_t up = 0;
  for (size_t b : up_sizes) up += al(b);
  // one persistent workspace, carved in 256-byte aligned pieces
  const size_t sizes[] = {up, 12 * rows, 8 * (rows + 1), 8 * (rows + 1), 4 * cap, cap, 8, scan_tmp};
  size_t need = 0;
  for (size_t b : sizes) need += al(b);
  if (c->upd_ws.n < need) RL_TRY(c->upd_ws.alloc(need + need / 4));
  if (c->upd_host_n < up) {
    if (c->upd_host) cudaFreeHost(c->upd_host);
    c->upd_host = nullptr;
    c->upd_host_n = 0;
    RL_CK(cudaMallocHost(&c->upd_host, up + up / 4));
    c->upd_host_n = up + up / 4;
  }
  uint8_t* cur = c->upd_ws.p;
  auto take = [&](size_t b) {
    uint8_t* p = cur;
    cur += al(b);
    return p;
  };
  uint8_t* d_up = take(sizes[0]);
  int32_t* add_cnt = reinterpret_cast<int32_t*>(take(sizes[1]));  // add | rem | cursor
  int32_t* rem_cnt = add_cnt + rows;
  uint32_t* cursor = reinterpret_cast<uint32_t*>(rem_cnt + rows);
  unsigned long long* packed = reinterpret_cast<unsigned long long*>(take(sizes[2]));
  unsigned long long* packed_off = reinterpret_cast<unsigned long long*>(take(sizes[3]));
  float* rec_v = reinterpret_cast<float*>(take(sizes[4]));
  int8_t* rec_s = reinterpret_cast<int8_t*>(take(sizes[5]));
  unsigned* d_unmatched = reinterpret_cast<unsigned*>(take(sizes[6]));
  void* tmp = take(sizes[7]);
  size_t up_off[4];
  {
    uint8_t* hbuf = static_cast<uint8_t*>(c->upd_host);
    const void* src[] = {wcells.data(), wflags.data(), dcells.data(), dsign.data()};
    size_t o = 0;
    for (int k = 0; k < 4; k++) {
      up_off[k] = o;
      if (up_sizes[k]) std::memcpy(hbuf + o, src[k], up_sizes[k]);
      o += al(up_sizes[k]);
    }
    RL_CK(cudaMemcpyAsync(d_up, hbuf, up, cudaMemcpyHostToDevice, st));
  }
  const int32_t* d_wcells = reinterpret_cast<const int32_t*>(d_up + up_off[0]);
  const uint8_t* d_wflags = d_up + up_off[1];
  const int32_t* d_dcells = reinterpret_cast<const int32_t*>(d_up + up_off[2]);
  const int8_t* d_dsign = reinterpret_cast<const int8_t*>(d_up + up_off[3]);
  k_set_flags<<<blocks_for(nw, 256), 256, 0, st>>>(d_wcells, d_wflags, int(nw), c->flags.p);
  RL_CK(cudaGetLastError());
  RL_TRY(refresh_query_bits(c));
  if (nd == 0) return finish(c, nullptr);

  // 3. per-row delta counts -> one scan (new offsets | delta buckets) -> records into buckets
  RL_CK(cudaMemsetAsync(add_cnt, 0, 12 * rows, st));
  RL_CK(cudaMemsetAsync(d_unmatched, 0, 4, st));
  const int db = blocks_for(size_t(nd) * c->S, 256);
  k_delta_count<<<db, 256, 0, st>>>(d_dcells, d_dsign, nd, c->d_slices.p, c->S, w, add_cnt,
                                    rem_cnt);
  k_pack_len<<<blocks_for(rows + 1, 256), 256, 0, st>>>(c->row_off.p, add_cnt, rem_cnt, packed,
                                                        rows);
  RL_CK(cub::DeviceScan::ExclusiveSum(tmp, scan_tmp, packed, packed_off, int(rows + 1), st));
  k_delta_scatter<<<db, 256, 0, st>>>(d_dcells, d_dsign, nd, c->d_slices.p, c->S, w, packed_off,
                                      cursor, rec_v, rec_s);
  RL_CK(cudaGetLastError());
  // 4. merge into the spare buffers (the new offsets too), then swap
  if (c->off_spare.n < rows + 1) RL_TRY(c->off_spare.alloc(rows + 1));
  const size_t zp_need = c->zero_points + cap;
  if (c->zp_spare.n < zp_need) RL_TRY(c->zp_spare.alloc(zp_need + zp_need / 8));
  k_merge_rows<<<blocks_for(rows * 32, 256, 32), 256, 0, st>>>(
      c->row_off.p, c->zp.p, packed_off, c->off_spare.p, c->zp_spare.p, add_cnt, rem_cnt, rec_v,
      rec_s, rows, d_unmatched, c->hints.p);
  RL_CK(cudaGetLastError());
  uint32_t* total_miss = nullptr;  // pinned: {new zero-point total, missed removals}
  RL_TRY(host_small(c, &total_miss));
  RL_CK(cudaMemcpyAsync(&total_miss[0], packed_off + rows, 4, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaMemcpyAsync(&total_miss[1], d_unmatched, 4, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
  if (total_miss[1]) {
    set_error("cddt: %u zero-point removals found no stored point (structure inconsistent)",
              total_miss[1]);
    return RL_ELOGIC;
  }
  std::swap(c->zp, c->zp_spare);
  std::swap(c->row_off, c->off_spare);  // the row records were rewritten by k_merge_rows
  c->zero_points = total_miss[0];
  return finish(c, nullptr);
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
