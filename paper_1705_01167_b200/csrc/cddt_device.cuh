// Device-side CDDT query: the exact FP64 restatement of Cddt::directional_cast
// (proj/src/cddt.cpp:207-269) and detail::RayWalker
// (proj/include/rangelib/detail/ray_walker.hpp:21-104) for sm_100a.
//
// Bit-exactness contract: every TU including this header is
// compiled with -fmad=false so no FP64 multiply-add is contracted; the
// direction lattice cos/sin comes from the host (glibc) and is uploaded;
// division, floor, ceil, fmod and conversions are IEEE-exact on the device.
#pragma once

#include <cstdint>

namespace rl {

constexpr double kTwoPi = 6.283185307179586476925286766559;  // raycast.hpp:12
constexpr double kNearField = 0.75;                           // cddt.cpp:19
constexpr double kVerifyHalf = 0.7072;                        // cddt.cpp:25
constexpr double kLatticeEps = 1e-9;                          // cddt.cpp:26
constexpr double kWalkNone = -1.0;                            // ray_walker.hpp:23
constexpr double kWalkExit = -2.0;                            // ray_walker.hpp:24

// per-cell flag byte
constexpr uint8_t kOcc = 1;     // occupied
constexpr uint8_t kClear = 2;   // cell and all in-bounds 8-neighbours free (cddt.cpp:173-180)
constexpr uint8_t kMember = 4;  // edge cell with stored zero points (grid.cpp:110-119)

// Per-slice projection (SliceProjection, cddt.hpp:22-33) packed for one
// 32-byte load: cos, sin, y_offset, bin_count, global row base.
struct __align__(32) SliceParam {
  double cos_t, sin_t, y_offset;
  int32_t bin_count;
  uint32_t row_base;
};

// Read-only view of one device-resident structure, passed by value.
// Occupancy for queries lives in 8x8-cell tiles: tiles[(y>>3)*tw + (x>>3)] =
// {occupied bits, clear bits}, bit (y&7)*8 + (x&7). A ray walk crosses a tile
// boundary every ~8 cells, so one 8-byte load serves several DDA steps.
struct CddtView {
  const uint8_t* __restrict__ flags;      // w*h (build / update bookkeeping)
  const ulonglong2* __restrict__ tiles;   // tw*th occupancy + clear tiles
  int tw;
  const uint2* __restrict__ rowbits;      // h*wpr {occupied, clear} bits, 32 cells per word
  int wpr;
  const uint32_t* __restrict__ row_off;   // rows+1, CSR into zp
  const float* __restrict__ zp;           // zero points, ascending per row
  const float* __restrict__ zs;           // zs[j] = zp[16 j]: a search guide over the CSR
  const SliceParam* __restrict__ slices;  // S
  const double4* __restrict__ dirs;       // K (cos, sin, 1/cos, 1/sin), axis-snapped (cddt.cpp:30-42)
  int w, h, K, S;
  double max_range;
  size_t zp_bytes;
};

__host__ __device__ __forceinline__ double fmin_std(double a, double b) { return (b < a) ? b : a; }
__host__ __device__ __forceinline__ double fmax_std(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ long iround(double v) { return (long)ceil(v - 0.5); }  // raycast.hpp:17

// Exact double <-> int helpers that stay off the XU (conversion) pipe, which
// the cast kernel otherwise saturates (profiles/r01/ncu_k_cast_v3.txt):
// floor via the 1.5*2^52 rounding constant (RN(v) lands in the low mantissa
// bits, then one compare corrects to floor), int -> double via the 2^52 + 2^31
// bias. Both are exact for |v| < 2^30; anything else takes the IEEE path.
struct Floor {
  int i;
  double d;
};
#ifndef RL_NOXU_FLOOR
#define RL_NOXU_FLOOR 0
#endif
#ifndef RL_NOXU_I2D
#define RL_NOXU_I2D 0
#endif
__device__ __forceinline__ Floor floor2(double v) {
  if (!RL_NOXU_FLOOR || !(fabs(v) < 1073741824.0)) {
    const double f = floor(v);
    return Floor{(int)f, f};
  }
  const double t = v + 6755399441055744.0;
  int i = __double2loint(t);
  double r = t - 6755399441055744.0;  // RN(v), exact
  if (r > v) {
    i -= 1;
    r -= 1.0;
  }
  return Floor{i, r};
}
__device__ __forceinline__ double i2d(int v) {
  if (!RL_NOXU_I2D) return (double)v;
  return __hiloint2double(0x43300000, v ^ (int)0x80000000) - 4503601774854144.0;
}

__device__ __forceinline__ double normalize_angle_2pi(double t) {  // raycast.hpp:20-25
  if (t >= 0.0 && t < kTwoPi) return t;  // fmod(t, 2pi) == t exactly here
  t = fmod(t, kTwoPi);
  if (t < 0) t += kTwoPi;
  if (t >= kTwoPi) t = 0.0;
  return t;
}

__device__ __forceinline__ double div_rn(double a, double d, double r);
constexpr double kInvTwoPi = 1.0 / kTwoPi;  // RN(1/2pi), folded at compile time

__device__ __forceinline__ int direction_index(double theta, int K) {  // raycast.hpp:36-40
  // iround(theta * K / 2pi) % K; the quotient is the correctly rounded one
  const double t = div_rn(theta * (double)K, kTwoPi, kInvTwoPi) - 0.5;
  const Floor f = floor2(-t);  // ceil(t) = -floor(-t)
  const int ci = -f.i;
  if (ci >= 0 && ci <= K && fabs(t) < 1073741824.0)  // theta in [0, 2pi): no modulo
    return ci == K ? 0 : ci;
  long i = (long)ceil(t) % K;
  if (i < 0) i += K;
  return (int)i;
}

__device__ __forceinline__ int tile_of(const CddtView& c, int x, int y) {
  return (y >> 3) * c.tw + (x >> 3);
}
__device__ __forceinline__ int bit_of(int x, int y) { return ((y & 7) << 3) | (x & 7); }

#ifndef RL_TILES
#define RL_TILES 0
#endif
#ifndef RL_ROWBITS
#define RL_ROWBITS 1
#endif

// Register-resident copy of the last occupancy tile touched by a query.
struct OccCache {
  int tile = -1;
  unsigned long long word = 0;
  __device__ __forceinline__ bool occ(const CddtView& c, int x, int y) {
#if RL_ROWBITS
    return (__ldg(&c.rowbits[y * c.wpr + (x >> 5)].x) >> (x & 31)) & 1u;
#elif !RL_TILES
    return (__ldg(c.flags + (size_t)y * c.w + x) & kOcc) != 0;
#endif
    const int t = tile_of(c, x, y);
    if (t != tile) {
      tile = t;
      word = __ldg(&c.tiles[t].x);
    }
    return (word >> bit_of(x, y)) & 1ull;
  }
};
__device__ __forceinline__ bool in_bounds(const CddtView& c, int x, int y) {
  return (unsigned)x < (unsigned)c.w && (unsigned)y < (unsigned)c.h;
}

#ifndef RL_FAST_DIV
#define RL_FAST_DIV 1
#endif

// a / d correctly rounded, given r = RN(1/d) (host-computed per direction):
// q0 = RN(a r) is within one ulp of a/d and the FMA residual a - d q0 is
// exact, so RN(q0 + (a - d q0) r) = RN(a/d) (Markstein's theorem; valid here
// because |a| <= grid extent and |d| >= sin(2pi/theta_disc) keep every
// intermediate far from overflow and the subnormal range). Replaces the
// ~30-instruction IEEE division sequence with 3 FP64 operations; checked
// bit-for-bit against IEEE division by tests/test_fast_div.py.
__device__ __forceinline__ double div_rn(double a, double d, double r) {  // NOLINT
#if RL_FAST_DIV
  const double q0 = __dmul_rn(a, r);
  const double e = fma(-d, q0, a);
  return fma(e, r, q0);
#else
  return a / d;
#endif
}

__device__ __forceinline__ double boundary_t(double d, double o, int cc, double r) {  // ray_walker.hpp:75-79
  if (d > 0) return div_rn(i2d(cc) + 1.0 - o, d, r);
  if (d < 0) return div_rn(i2d(cc) - o, d, r);
  return __longlong_as_double(0x7ff0000000000000ll);
}

#ifndef RL_WALK_BRANCHFREE
#define RL_WALK_BRANCHFREE 1
#endif

// RayWalker (ray_walker.hpp:21-104). The per-axis sign logic of boundary_t
// and advance() is hoisted into per-query constants (step sign, boundary
// bias 1.0/0.0, axis-parallel flag), so a walker step is straight-line code
// with selects: lanes walking in different directions no longer diverge.
// Each boundary value is still ((double)c + 1.0 - o) / d or ((double)c - o)/d
// rounded exactly as the reference computes it.
struct Walker {
  double ox, oy, dx, dy, rx, ry, t, tnx, tny;
  int cx, cy;
#if RL_WALK_BRANCHFREE
  double bx, by;   // 1.0 when the axis direction is positive, else 0.0
  int sx, sy;      // cell step along each axis
  bool zx, zy;     // axis-parallel: boundary parameter is +inf

  __device__ __forceinline__ double bnd_x(int c) const {
    const double v = div_rn((i2d(c) + bx) - ox, dx, rx);
    return zx ? __longlong_as_double(0x7ff0000000000000ll) : v;
  }
  __device__ __forceinline__ double bnd_y(int c) const {
    const double v = div_rn((i2d(c) + by) - oy, dy, ry);
    return zy ? __longlong_as_double(0x7ff0000000000000ll) : v;
  }
  __device__ __forceinline__ void place(double tt) {  // ray_walker.hpp:62-73
    t = tt;
    double px = ox + tt * dx, py = oy + tt * dy;
    const Floor fx = floor2(px), fy = floor2(py);
    cx = fx.i - ((dx < 0 && px == fx.d) ? 1 : 0);
    cy = fy.i - ((dy < 0 && py == fy.d) ? 1 : 0);
    tnx = bnd_x(cx);
    tny = bnd_y(cy);
  }
  __device__ __forceinline__ void init(double x, double y, const double4& dir) {
    ox = x;
    oy = y;
    dx = dir.x;
    dy = dir.y;
    rx = dir.z;
    ry = dir.w;
    bx = dx > 0 ? 1.0 : 0.0;
    by = dy > 0 ? 1.0 : 0.0;
    sx = dx > 0 ? 1 : -1;
    sy = dy > 0 ? 1 : -1;
    zx = !(dx > 0) && !(dx < 0);
    zy = !(dy > 0) && !(dy < 0);
    place(0.0);
  }
  // emplace + seek(tt): place() resets the whole state, so one place at max(0, tt)
  __device__ __forceinline__ void init_at(double x, double y, const double4& dir, double tt) {
    ox = x;
    oy = y;
    dx = dir.x;
    dy = dir.y;
    rx = dir.z;
    ry = dir.w;
#if RL_WALK_BRANCHFREE
    bx = dx > 0 ? 1.0 : 0.0;
    by = dy > 0 ? 1.0 : 0.0;
    sx = dx > 0 ? 1 : -1;
    sy = dy > 0 ? 1 : -1;
    zx = !(dx > 0) && !(dx < 0);
    zy = !(dy > 0) && !(dy < 0);
#endif
    place(tt > 0.0 ? tt : 0.0);
  }
  __device__ __forceinline__ void seek(double tt) {  // ray_walker.hpp:36-38
    if (tt > t) place(tt);
  }
  __device__ __forceinline__ void advance() {  // ray_walker.hpp:81-97
    // equal parameters: exact corner crossing, both axes step (diagonal)
    const bool stx = tnx <= tny, sty = tny <= tnx;
    t = stx ? tnx : tny;
    const int ncx = cx + sx, ncy = cy + sy;
    const double ntx = bnd_x(ncx), nty = bnd_y(ncy);
    if (stx) {
      cx = ncx;
      tnx = ntx;
    }
    if (sty) {
      cy = ncy;
      tny = nty;
    }
  }
#else
  __device__ __forceinline__ void place(double tt) {  // ray_walker.hpp:62-73
    t = tt;
    double px = ox + tt * dx, py = oy + tt * dy;
    const Floor fx = floor2(px), fy = floor2(py);
    cx = fx.i;
    cy = fy.i;
    if (dx < 0 && px == fx.d) cx--;
    if (dy < 0 && py == fy.d) cy--;
    tnx = boundary_t(dx, ox, cx, rx);
    tny = boundary_t(dy, oy, cy, ry);
  }
  __device__ __forceinline__ void init(double x, double y, const double4& dir) {
    ox = x;
    oy = y;
    dx = dir.x;
    dy = dir.y;
    rx = dir.z;
    ry = dir.w;
    place(0.0);
  }
  // emplace + seek(tt): place() resets the whole state, so one place at max(0, tt)
  __device__ __forceinline__ void init_at(double x, double y, const double4& dir, double tt) {
    ox = x;
    oy = y;
    dx = dir.x;
    dy = dir.y;
    rx = dir.z;
    ry = dir.w;
#if RL_WALK_BRANCHFREE
    bx = dx > 0 ? 1.0 : 0.0;
    by = dy > 0 ? 1.0 : 0.0;
    sx = dx > 0 ? 1 : -1;
    sy = dy > 0 ? 1 : -1;
    zx = !(dx > 0) && !(dx < 0);
    zy = !(dy > 0) && !(dy < 0);
#endif
    place(tt > 0.0 ? tt : 0.0);
  }
  __device__ __forceinline__ void seek(double tt) {  // ray_walker.hpp:36-38
    if (tt > t) place(tt);
  }
  __device__ __forceinline__ void advance() {  // ray_walker.hpp:81-97
    if (tnx == tny) {
      t = tnx;
      cx += dx > 0 ? 1 : -1;
      cy += dy > 0 ? 1 : -1;
      tnx = boundary_t(dx, ox, cx, rx);
      tny = boundary_t(dy, oy, cy, ry);
    } else if (tnx < tny) {
      t = tnx;
      cx += dx > 0 ? 1 : -1;
      tnx = boundary_t(dx, ox, cx, rx);
    } else {
      t = tny;
      cy += dy > 0 ? 1 : -1;
      tny = boundary_t(dy, oy, cy, ry);
    }
  }
#endif
  __device__ __forceinline__ double scan_to(const CddtView& c, OccCache& oc, double lim) {  // :51-59
    for (;;) {
      if (!in_bounds(c, cx, cy)) return kWalkExit;
      if (oc.occ(c, cx, cy)) return t;
      double tn = tnx < tny ? tnx : tny;
      if (tn > lim) return kWalkNone;
      advance();
    }
  }
};

#ifndef RL_SEARCH
#define RL_SEARCH 2
#endif

// Number of leading elements e of v[0, n) with pred(e): e <= xq (forward,
// i.e. !(xq < e), upper_bound) or e < xq (backward, lower_bound).
//
// Comparisons run in the float domain, exactly: for a float e,
//   double(e) <= xq  <=>  e <= RD_f32(xq)     and     double(e) < xq  <=>  e < RU_f32(xq)
// (no float lies strictly between RD_f32(xq) and RU_f32(xq)).
__device__ __forceinline__ uint32_t partition_point(const float* __restrict__ v, uint32_t n,
                                                    double xq, bool forward) {
  const float xlo = __double2float_rd(xq), xhi = __double2float_ru(xq);
#define RL_PRED(e) (forward ? ((e) <= xlo) : ((e) < xhi))
#if RL_SEARCH == 8
  // 8-way search: each level issues 7 independent pivot loads, so a row of
  // length n costs ~log8(n) dependent load rounds instead of log2(n).
  uint32_t base = 0, len = n;  // partition point lies in [base, base + len]
  while (len > 8) {
    const uint32_t s = len >> 3;
    float pv[7];
#pragma unroll
    for (int j = 0; j < 7; j++) pv[j] = __ldg(v + base + (j + 1) * s - 1);
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < 7; j++) cnt += RL_PRED(pv[j]) ? 1u : 0u;
    if (cnt == 7) {
      base += 7 * s;
      len -= 7 * s;
    } else {
      base += cnt * s;
      len = s - 1;
    }
  }
  float tv[8];
#pragma unroll
  for (int j = 0; j < 8; j++) tv[j] = (uint32_t)j < len ? __ldg(v + base + j) : 0.0f;
  uint32_t cnt = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) cnt += ((uint32_t)j < len && RL_PRED(tv[j])) ? 1u : 0u;
  return base + cnt;
#else
  // libstdc++'s halving sequence
  uint32_t first = 0, len = n;
  while (len > 0) {
    uint32_t half = len >> 1, mid = first + half;
    if (RL_PRED(__ldg(v + mid))) {
      first = mid + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return first;
#endif
#undef RL_PRED
}

#ifndef RL_SAMPLED_SEARCH
#define RL_SAMPLED_SEARCH 0
#endif
constexpr int kSampleShift = 4;  // one guide key per 16 zero points

// partition_point over the row zp[lo, hi) using the guide keys zs[j] =
// zp[16 j] that fall inside the row: a search over those (a few entries of a
// small, L2-resident array) picks the 16-element block holding the partition
// point, then one search inside the block. Two dependent rounds instead of
// log2(n); the returned index is the same (a partition point is unique).
__device__ __forceinline__ uint32_t partition_point_guided(const CddtView& c, uint32_t lo,
                                                           uint32_t hi, double xq, bool forward) {
  const uint32_t j0 = (lo + 15) >> kSampleShift;
  const uint32_t j1 = hi > 0 ? (hi - 1) >> kSampleShift : 0;
  if (hi <= lo || j0 > j1) return partition_point(c.zp + lo, hi - lo, xq, forward);
  // number of guide keys in [j0, j1] satisfying the predicate
  const uint32_t k = partition_point(c.zs + j0, j1 - j0 + 1, xq, forward);
  uint32_t a, b;  // the partition point lies in [a, b] (global indices)
  if (k == 0) {
    a = lo;
    b = j0 << kSampleShift;
  } else {
    a = ((j0 + k - 1) << kSampleShift) + 1;
    b = k <= j1 - j0 ? (j0 + k) << kSampleShift : hi;
  }
  return (a - lo) + partition_point(c.zp + a, b - a, xq, forward);
}

// Outcome of one query beyond the range: the occupied cell that settled it
// and the resolving zero point (what MarkSink::mark receives, cddt.cpp:249,259).
struct CastOut {
  int32_t hit;      // y*w+x or -1
  uint32_t res_g;   // global row of the resolving zero point
  int32_t res_idx;  // index within the row, -1 when no zero point resolved
};

// Cddt::directional_cast (cddt.cpp:207-269).
__device__ __forceinline__ double directional_cast(const CddtView& c, double x, double y, int a,
                                                   CastOut& o) {
  o.hit = -1;
  o.res_idx = -1;
  o.res_g = 0;
  const int cxi = floor2(x).i, cyi = floor2(y).i;
  if (!in_bounds(c, cxi, cyi)) return c.max_range;
  OccCache oc;
  // Issue the independent gathers of this query together: the origin cell's
  // bits and the row offsets do not depend on each other, so the row offsets
  // are requested before the origin test resolves (they are simply unused when
  // the origin is occupied).
  const bool forward = a < c.S;
  const int s = forward ? a : a - c.S;
  const SliceParam sp = c.slices[s];
  const double xq = x * sp.cos_t + y * sp.sin_t;                 // cddt.hpp:31
  const double yq = -x * sp.sin_t + y * sp.cos_t + sp.y_offset;  // cddt.hpp:32
  int row = floor2(yq).i;  // == int(yq) after the clamp below (differs only for yq < 0)
  if (row < 0) row = 0;
  if (row >= sp.bin_count) row = sp.bin_count - 1;
  const uint32_t g = sp.row_base + (uint32_t)row;
  const uint32_t lo = __ldg(c.row_off + g), hi = __ldg(c.row_off + g + 1);
#if RL_ROWBITS
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {
    o.hit = cyi * c.w + cxi;
    return 0.0;
  }
  const bool clear0 = (w0.y >> (cxi & 31)) & 1u;
#elif RL_TILES
  oc.tile = tile_of(c, cxi, cyi);
  const ulonglong2 t0 = __ldg(c.tiles + oc.tile);
  oc.word = t0.x;
  const int b0 = bit_of(cxi, cyi);
  if ((t0.x >> b0) & 1ull) {
    o.hit = cyi * c.w + cxi;
    return 0.0;
  }
  const bool clear0 = (t0.y >> b0) & 1ull;
#else
  const uint8_t f0 = __ldg(c.flags + (size_t)cyi * c.w + cxi);
  if (f0 & kOcc) {
    o.hit = cyi * c.w + cxi;
    return 0.0;
  }
  const bool clear0 = (f0 & kClear) != 0;
#endif
  const double4 dir = c.dirs[a];
  const double dx = dir.x, dy = dir.y;

  Walker wk;
  bool have_walker = false;
  if (!clear0) {
    wk.init(x, y, dir);
    have_walker = true;
    double r = wk.scan_to(c, oc, kNearField);
    if (r >= 0.0) {
      o.hit = wk.cy * c.w + wk.cx;
      return (c.max_range < r) ? c.max_range : r;
    }
    if (r == kWalkExit) return c.max_range;
  }

  double result = c.max_range;
  const double gw = (double)c.w, gh = (double)c.h;
  const float* __restrict__ v = c.zp + lo;
  // std::upper_bound (forward, xq < double(v)) / std::lower_bound (backward,
  // double(v) < xq): the partition point of a monotone predicate over the
  // sorted row (cddt.hpp:106-131); any search order yields the same index.
#if RL_SAMPLED_SEARCH
  const uint32_t first = partition_point_guided(c, lo, hi, xq, forward);
#else
  const uint32_t first = partition_point(v, hi - lo, xq, forward);
#endif
  const int n = (int)(hi - lo);
  int idx = forward ? (int)first : (int)first - 1;
  const int step = forward ? 1 : -1;
  for (; idx >= 0 && idx < n; idx += step) {
    const double vv = (double)__ldg(v + idx);
    const double d = forward ? vv - xq : xq - vv;
    if (d >= c.max_range) break;
    // landing-cell probe (cddt.cpp:239-253)
    const double px = x + d * dx, py = y + d * dy;
    if (px >= 0.0 && py >= 0.0 && px < gw && py < gh) {
      const Floor flx = floor2(px), fly = floor2(py);  // px, py >= 0: int() == floor
      const int hx = flx.i, hy = fly.i;
      const double fx = px - flx.d, fy = py - fly.d;
      if (fx > kLatticeEps && fx < 1.0 - kLatticeEps && fy > kLatticeEps &&
          fy < 1.0 - kLatticeEps && oc.occ(c, hx, hy)) {
        o.hit = hy * c.w + hx;
        o.res_g = g;
        o.res_idx = idx;
        result = d;
        break;
      }
    }
    // verification window around the candidate (cddt.cpp:254-261)
#ifdef RL_DEBUG_NOWALK  // timing experiment only: results are wrong
    continue;
#endif
    if (!have_walker) {
      wk.init(x, y, dir);
      have_walker = true;
    }
    wk.seek(d - kVerifyHalf);
    double r = wk.scan_to(c, oc, d + kVerifyHalf);
    if (r == kWalkExit) break;
    if (r < 0.0) continue;
    o.hit = wk.cy * c.w + wk.cx;
    o.res_g = g;
    o.res_idx = idx;
    result = d;
    break;
  }
  return result;
}

}  // namespace rl

namespace rl {

// First phase of directional_cast for the two-phase batch kernel: everything
// up to and including the first candidate's landing-cell probe, with no
// RayWalker. Returns true with *result set when the query is settled there
// (off-map or occupied origin, no candidate, candidate beyond max_range, or
// an interior landing hit) — exactly where cddt.cpp:207-269 would return —
// and false when the exact answer needs the walker (a non-clear origin's
// near field, or a candidate whose landing probe does not settle it); the
// caller then runs the full directional_cast for that query.
__device__ __forceinline__ bool directional_cast_fast(const CddtView& c, double x, double y,
                                                      int a, double* result) {
  const int cxi = floor2(x).i, cyi = floor2(y).i;
  if (!in_bounds(c, cxi, cyi)) {
    *result = c.max_range;
    return true;
  }
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {
    *result = 0.0;
    return true;
  }
  if (!((w0.y >> (cxi & 31)) & 1u)) return false;  // near field needs the walker
  const bool forward = a < c.S;
  const int s = forward ? a : a - c.S;
  const SliceParam sp = c.slices[s];
  const double xq = x * sp.cos_t + y * sp.sin_t;
  const double yq = -x * sp.sin_t + y * sp.cos_t + sp.y_offset;
  int row = floor2(yq).i;  // == int(yq) after the clamp below (differs only for yq < 0)
  if (row < 0) row = 0;
  if (row >= sp.bin_count) row = sp.bin_count - 1;
  const uint32_t g = sp.row_base + (uint32_t)row;
  const uint32_t lo = __ldg(c.row_off + g), hi = __ldg(c.row_off + g + 1);
#if RL_SAMPLED_SEARCH
  const uint32_t first = partition_point_guided(c, lo, hi, xq, forward);
#else
  const uint32_t first = partition_point(c.zp + lo, hi - lo, xq, forward);
#endif
  const int n = (int)(hi - lo);
  const int idx = forward ? (int)first : (int)first - 1;
  if (idx < 0 || idx >= n) {
    *result = c.max_range;
    return true;
  }
  const double vv = (double)__ldg(c.zp + lo + idx);
  const double d = forward ? vv - xq : xq - vv;
  if (d >= c.max_range) {
    *result = c.max_range;
    return true;
  }
  const double4 dir = c.dirs[a];
  const double px = x + d * dir.x, py = y + d * dir.y;
  if (px >= 0.0 && py >= 0.0 && px < (double)c.w && py < (double)c.h) {
    const Floor flx = floor2(px), fly = floor2(py);
    const int hx = flx.i, hy = fly.i;
    const double fx = px - flx.d, fy = py - fly.d;
    if (fx > kLatticeEps && fx < 1.0 - kLatticeEps && fy > kLatticeEps &&
        fy < 1.0 - kLatticeEps &&
        ((__ldg(&c.rowbits[hy * c.wpr + (hx >> 5)].x) >> (hx & 31)) & 1u)) {
      *result = d;
      return true;
    }
  }
  return false;
}

}  // namespace rl

namespace rl {

// ---- split form of directional_cast for the deferred-walk batch kernel ----
// Phase 1 runs cddt.cpp:207-269 up to the first point where a RayWalker is
// needed: a non-clear origin (near-field walk) or a candidate whose landing
// probe does not settle it (verification window). Phase 2 resumes exactly
// there. Split and unsplit runs take the same decisions in the same order.
struct WalkDefer {
  uint32_t lo, n;  // CSR row of the query
  int idx;         // candidate whose window walk is pending; -1: near field
};

__device__ __forceinline__ bool directional_cast_p1(const CddtView& c, double x, double y, int a,
                                                    double* result, WalkDefer* def) {
  const Floor fcx = floor2(x), fcy = floor2(y);
  const int cxi = fcx.i, cyi = fcy.i;
  if (!in_bounds(c, cxi, cyi)) {
    *result = c.max_range;
    return true;
  }
  const bool forward = a < c.S;
  const int s = forward ? a : a - c.S;
  const SliceParam sp = c.slices[s];
  const double xq = x * sp.cos_t + y * sp.sin_t;
  const double yq = -x * sp.sin_t + y * sp.cos_t + sp.y_offset;
  int row = floor2(yq).i;
  if (row < 0) row = 0;
  if (row >= sp.bin_count) row = sp.bin_count - 1;
  const uint32_t g = sp.row_base + (uint32_t)row;
  const uint32_t lo = __ldg(c.row_off + g), hi = __ldg(c.row_off + g + 1);
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {
    *result = 0.0;
    return true;
  }
  def->lo = lo;
  def->n = hi - lo;
  if (!((w0.y >> (cxi & 31)) & 1u)) {
    def->idx = -1;  // near field needs the walker: phase 2 redoes the whole query
    return false;
  }
#if RL_SAMPLED_SEARCH
  const uint32_t first = partition_point_guided(c, lo, hi, xq, forward);
#else
  const uint32_t first = partition_point(c.zp + lo, hi - lo, xq, forward);
#endif
  const int n = (int)(hi - lo);
  const int step = forward ? 1 : -1;
  const double4 dir = c.dirs[a];
  const double gw = (double)c.w, gh = (double)c.h;
  OccCache oc;
  for (int idx = forward ? (int)first : (int)first - 1; idx >= 0 && idx < n; idx += step) {
    const double vv = (double)__ldg(c.zp + lo + idx);
    const double d = forward ? vv - xq : xq - vv;
    if (d >= c.max_range) break;
    const double px = x + d * dir.x, py = y + d * dir.y;
    if (px >= 0.0 && py >= 0.0 && px < gw && py < gh) {
      const Floor flx = floor2(px), fly = floor2(py);
      const double fx = px - flx.d, fy = py - fly.d;
      if (fx > kLatticeEps && fx < 1.0 - kLatticeEps && fy > kLatticeEps &&
          fy < 1.0 - kLatticeEps && oc.occ(c, flx.i, fly.i)) {
        *result = d;
        return true;
      }
    }
    def->idx = idx;  // first verification window: hand over to phase 2
    return false;
  }
  *result = c.max_range;
  return true;
}

// Phase 2 for a deferred window: the walker does not exist yet (the origin
// was clear), so emplace + seek(d - kVerifyHalf) is one place() at
// max(0, d - kVerifyHalf); then the reference's candidate loop continues.
__device__ __forceinline__ double directional_cast_resume(const CddtView& c, double x, double y,
                                                          int a, const WalkDefer& def) {
  const bool forward = a < c.S;
  const int s = forward ? a : a - c.S;
  const SliceParam sp = c.slices[s];
  const double xq = x * sp.cos_t + y * sp.sin_t;
  const double4 dir = c.dirs[a];
  const double dx = dir.x, dy = dir.y;
  const double gw = (double)c.w, gh = (double)c.h;
  const float* __restrict__ v = c.zp + def.lo;
  const int n = (int)def.n, step = forward ? 1 : -1;
  OccCache oc;
  Walker wk;
  bool first = true;
  for (int idx = def.idx; idx >= 0 && idx < n; idx += step) {
    const double vv = (double)__ldg(v + idx);
    const double d = forward ? vv - xq : xq - vv;
    if (d >= c.max_range) break;
    if (!first) {  // landing probe (phase 1 already ran it for def.idx)
      const double px = x + d * dx, py = y + d * dy;
      if (px >= 0.0 && py >= 0.0 && px < gw && py < gh) {
        const Floor flx = floor2(px), fly = floor2(py);
        const double fx = px - flx.d, fy = py - fly.d;
        if (fx > kLatticeEps && fx < 1.0 - kLatticeEps && fy > kLatticeEps &&
            fy < 1.0 - kLatticeEps && oc.occ(c, flx.i, fly.i))
          return d;
      }
      wk.seek(d - kVerifyHalf);
    } else {
      wk.init_at(x, y, dir, d - kVerifyHalf);
      first = false;
    }
    const double r = wk.scan_to(c, oc, d + kVerifyHalf);
    if (r == kWalkExit) break;
    if (r < 0.0) continue;
    return d;
  }
  return c.max_range;
}

}  // namespace rl
