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
//      slices, radix-sort them by (row, value);
//   4. device: new row lengths -> scan -> per-row merge of the old sorted row
//      with its sorted deltas (unaffected rows are a straight copy).
// Only O(changed pixels * S) records are sorted; the copy is one pass over
// the zero-point array.
#include <cub/cub.cuh>

#include <algorithm>
#include <unordered_map>

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

// order-preserving map f32 -> u32 (negatives flipped)
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// delta pixel (cell, sign) x slice -> records key = row<<32 | f2key(v), val = sign
__global__ void k_delta_records(const int32_t* __restrict__ cells, const int8_t* __restrict__ sign,
                                int n_cells, const SliceParam* __restrict__ slices, int S, int w,
                                unsigned long long* __restrict__ keys, int8_t* __restrict__ vals,
                                unsigned* __restrict__ count, int32_t* __restrict__ add_cnt,
                                int32_t* __restrict__ rem_cnt) {
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
      unsigned pos = atomicAdd(count, 1u);
      keys[pos] = (static_cast<unsigned long long>(g) << 32) | f2key(v);
      vals[pos] = sign[k];
      if (sign[k] > 0)
        atomicAdd(&add_cnt[g], 1);
      else
        atomicAdd(&rem_cnt[g], 1);
    }
  }
}

__global__ void k_new_len(const uint32_t* __restrict__ off, const int32_t* __restrict__ add_cnt,
                          const int32_t* __restrict__ rem_cnt, uint32_t* __restrict__ len,
                          size_t rows) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g <= rows;
       g += size_t(gridDim.x) * blockDim.x)
    len[g] = g < rows ? (off[g + 1] - off[g]) + uint32_t(add_cnt[g]) - uint32_t(rem_cnt[g]) : 0u;
}

__device__ __forceinline__ float key2f(unsigned long long key) {
  const uint32_t k = uint32_t(key);
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
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

// Merge each row's sorted delta records into its zero points, one warp per
// row (Cddt::add/remove_pixel_points: insert keeps the row sorted, remove
// drops one equal element; cddt.cpp:332-377, cddt.hpp:67-84). Equal values are
// identical floats, so the merged row is the sorted multiset
//   old - removed copies + added values,
// which a warp builds in parallel for rows with at most 32 records: every
// remove claims the next unclaimed copy of its value; a kept old element
// lands at (its index - removed before it + adds smaller than it); an add
// lands after the kept copies <= its value and the adds before it. Rows with
// more records fall back to a sequential merge by lane 0.
__global__ void k_merge_rows(const uint32_t* __restrict__ old_off, const float* __restrict__ old_zp,
                             const uint32_t* __restrict__ new_off, float* __restrict__ new_zp,
                             const int32_t* __restrict__ add_cnt,
                             const int32_t* __restrict__ rem_cnt,
                             const unsigned long long* __restrict__ keys,
                             const int8_t* __restrict__ vals, unsigned n_rec, size_t rows,
                             unsigned* __restrict__ unmatched) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  const size_t warp = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * blockDim.x) >> 5;
  for (size_t g = warp; g < rows; g += nwarps) {
    const uint32_t a = old_off[g], b = old_off[g + 1];
    const uint32_t o = new_off[g];
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
      continue;
    }
    // delta range of row g: lower_bound of g<<32 in the sorted keys (lane 0)
    unsigned j0 = 0;
    if (lane == 0) {
      const unsigned long long lo_key = static_cast<unsigned long long>(g) << 32;
      unsigned lo = 0, len = n_rec;
      while (len > 0) {
        const unsigned half = len >> 1, mid = lo + half;
        if (keys[mid] < lo_key) {
          lo = mid + 1;
          len -= half + 1;
        } else {
          len = half;
        }
      }
      j0 = lo;
    }
    j0 = __shfl_sync(0xffffffffu, j0, 0);
    const float* __restrict__ row = old_zp + a;
    const uint32_t n = b - a;
    if (nd <= 32) {
      const bool has = lane < nd;
      const float dv = has ? key2f(keys[j0 + lane]) : 0.f;
      const bool add = has && vals[j0 + lane] > 0, rem = has && !add;
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
      // adds: after the kept copies <= dv and the adds sorted before this one
      unsigned rem_le = 0;  // removed copies with value <= dv
      for (unsigned l = 0; l < nd; l++) {
        const float dl = __shfl_sync(0xffffffffu, dv, l);
        rem_le += ((rem_mask >> l) & 1u) && !(dv < dl) ? 1u : 0u;
      }
      if (add) new_zp[o + row_bound(row, n, dv, true) - rem_le + __popc(add_mask & lt)] = dv;
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
      continue;
    }
    if (lane != 0) continue;
    // sequential merge for rows with many records
    unsigned j = j0;
    const unsigned jend = j0 + nd;
    uint32_t i = a, w = o;
    unsigned miss = 0;
    while (i < b || j < jend) {
      if (j < jend) {
        const float dv = key2f(keys[j]);
        if (i == b || dv < old_zp[i]) {
          if (vals[j] > 0)
            new_zp[w++] = dv;
          else
            miss++;
          j++;
          continue;
        }
        if (dv == old_zp[i]) {
          if (vals[j] > 0) {
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
  // 1. replay in order; remember each touched cell's original state
  std::unordered_map<int32_t, uint8_t> orig;
  orig.reserve(n * 2);
  for (size_t k = 0; k < n; k++) {
    const int32_t cell = xy[2 * k + 1] * w + xy[2 * k];
    orig.emplace(cell, c->grid_h[cell]);
    c->grid_h[cell] = occ[k] ? 1 : 0;
  }
  std::vector<int32_t> changed;
  for (auto& kv : orig)
    if (kv.second != c->grid_h[kv.first]) changed.push_back(kv.first);
  if (changed.empty()) return RL_OK;
  // 2. flags in the dilation; membership deltas
  std::unordered_map<int32_t, uint8_t> window;
  for (int32_t cell : changed) {
    const int x = cell % w, y = cell / w;
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++)
        if (inb(x + dx, y + dy)) window.emplace((y + dy) * w + (x + dx), 0);
  }
  std::vector<int32_t> wcells, dcells;
  std::vector<uint8_t> wflags;
  std::vector<int8_t> dsign;
  wcells.reserve(window.size());
  for (auto& kv : window) {
    const int32_t cell = kv.first;
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
  const size_t cap = size_t(nd) * c->S * 3;  // a unit square spans at most 3 rows
  const size_t rows = c->rows;
  // one persistent workspace, carved in 256-byte aligned pieces
  size_t sort_tmp = 0, scan_tmp = 0;
  if (nd) {
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, (int8_t*)nullptr,
                                    (int8_t*)nullptr, int(cap), 0, 64, st);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  int(rows + 1), st);
  }
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t sizes[] = {4 * nw, nw, 4 * size_t(nd), size_t(nd), 4 * rows, 4 * rows, 8 * cap,
                          cap, 8 * cap, cap, 8, 4 * (rows + 1), std::max(sort_tmp, scan_tmp)};
  size_t need = 0;
  for (size_t b : sizes) need += al(b);
  if (c->upd_ws.n < need) RL_TRY(c->upd_ws.alloc(need + need / 4));
  uint8_t* cur = c->upd_ws.p;
  auto take = [&](size_t b) {
    uint8_t* p = cur;
    cur += al(b);
    return p;
  };
  int32_t* d_wcells = reinterpret_cast<int32_t*>(take(sizes[0]));
  uint8_t* d_wflags = take(sizes[1]);
  int32_t* d_dcells = reinterpret_cast<int32_t*>(take(sizes[2]));
  int8_t* d_dsign = reinterpret_cast<int8_t*>(take(sizes[3]));
  int32_t* add_cnt = reinterpret_cast<int32_t*>(take(sizes[4]));
  int32_t* rem_cnt = reinterpret_cast<int32_t*>(take(sizes[5]));
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(take(sizes[6]));
  int8_t* vals = reinterpret_cast<int8_t*>(take(sizes[7]));
  unsigned long long* keys_sorted = reinterpret_cast<unsigned long long*>(take(sizes[8]));
  int8_t* vals_sorted = reinterpret_cast<int8_t*>(take(sizes[9]));
  unsigned* d_count = reinterpret_cast<unsigned*>(take(sizes[10]));
  uint32_t* len = reinterpret_cast<uint32_t*>(take(sizes[11]));
  void* tmp = take(sizes[12]);

  RL_CK(cudaMemcpyAsync(d_wcells, wcells.data(), 4 * nw, cudaMemcpyHostToDevice, st));
  RL_CK(cudaMemcpyAsync(d_wflags, wflags.data(), nw, cudaMemcpyHostToDevice, st));
  k_set_flags<<<blocks_for(nw, 256), 256, 0, st>>>(d_wcells, d_wflags, int(nw), c->flags.p);
  RL_CK(cudaGetLastError());
  RL_TRY(refresh_query_bits(c));
  if (nd == 0) return finish(c, nullptr);

  // 3. delta records; unused key slots stay at UINT64_MAX and sort last, so
  //    the fixed-size sort needs no host round trip for the record count
  RL_CK(cudaMemcpyAsync(d_dcells, dcells.data(), 4 * size_t(nd), cudaMemcpyHostToDevice, st));
  RL_CK(cudaMemcpyAsync(d_dsign, dsign.data(), size_t(nd), cudaMemcpyHostToDevice, st));
  RL_CK(cudaMemsetAsync(add_cnt, 0, 4 * rows, st));
  RL_CK(cudaMemsetAsync(rem_cnt, 0, 4 * rows, st));
  RL_CK(cudaMemsetAsync(d_count, 0, 8, st));
  RL_CK(cudaMemsetAsync(keys, 0xFF, 8 * cap, st));
  k_delta_records<<<blocks_for(size_t(nd) * c->S, 256), 256, 0, st>>>(
      d_dcells, d_dsign, nd, c->d_slices.p, c->S, w, keys, vals, d_count, add_cnt, rem_cnt);
  RL_CK(cudaGetLastError());
  // keys are row<<32 | value; the unused slots (all ones) must sort last, so
  // the sort covers the value bits and enough row bits that no row is all ones
  int row_bits = 1;
  while ((size_t(1) << row_bits) <= rows) row_bits++;
  RL_CK(cub::DeviceRadixSort::SortPairs(tmp, sort_tmp, keys, keys_sorted, vals, vals_sorted,
                                        int(cap), 0, 32 + row_bits, st));
  // 4. new offsets and merge into the spare buffers, then swap
  if (c->off_spare.n < rows + 1) RL_TRY(c->off_spare.alloc(rows + 1));
  const size_t zp_need = c->zero_points + cap;
  if (c->zp_spare.n < zp_need) RL_TRY(c->zp_spare.alloc(zp_need + zp_need / 8));
  uint32_t* new_off = c->off_spare.p;
  k_new_len<<<blocks_for(rows + 1, 256), 256, 0, st>>>(c->row_off.p, add_cnt, rem_cnt, len, rows);
  RL_CK(cub::DeviceScan::ExclusiveSum(tmp, scan_tmp, len, new_off, int(rows + 1), st));
  k_merge_rows<<<blocks_for(rows * 32, 256, 32), 256, 0, st>>>(
      c->row_off.p, c->zp.p, new_off, c->zp_spare.p, add_cnt, rem_cnt, keys_sorted, vals_sorted,
      unsigned(cap), rows, d_count + 1);
  RL_CK(cudaGetLastError());
  uint32_t* total_miss = nullptr;  // pinned: {new zero-point total, missed removals}
  RL_TRY(host_small(c, &total_miss));
  RL_CK(cudaMemcpyAsync(&total_miss[0], new_off + rows, 4, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaMemcpyAsync(&total_miss[1], d_count + 1, 4, cudaMemcpyDeviceToHost, st));
  RL_CK(cudaStreamSynchronize(st));
  if (total_miss[1]) {
    set_error("cddt: %u zero-point removals found no stored point (structure inconsistent)",
              total_miss[1]);
    return RL_ELOGIC;
  }
  std::swap(c->zp, c->zp_spare);
  std::swap(c->row_off, c->off_spare);
  RL_TRY(refresh_row_hints(c));
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
