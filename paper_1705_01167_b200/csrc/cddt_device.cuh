// Device-side CDDT query: the exact FP64 restatement of Cddt::directional_cast
// (proj/src/cddt.cpp:207-269) and detail::RayWalker
// (proj/include/rangelib/detail/ray_walker.hpp:21-104) for sm_100a.
//
// Bit-exactness contract: every TU including this header is
// compiled with -fmad=false so no FP64 multiply-add is contracted; the
// direction lattice cos/sin comes from the host (glibc) and is uploaded;
// floor, ceil, fmod and conversions are IEEE-exact on the device, and the two
// divisions of the path use a proven-exact reciprocal form (div_rn below).
#pragma once

#include <cstdint>

namespace rl {

constexpr double kTwoPi = 6.283185307179586476925286766559;  // raycast.hpp:12
constexpr double kInvTwoPi = 1.0 / kTwoPi;                    // RN(1/2pi), folded at compile time
constexpr double kNearField = 0.75;                           // cddt.cpp:19
constexpr double kVerifyHalf = 0.7072;                        // cddt.cpp:25
constexpr double kLatticeEps = 1e-9;                          // cddt.cpp:26
constexpr double kWalkNone = -1.0;                            // ray_walker.hpp:23
constexpr double kWalkExit = -2.0;                            // ray_walker.hpp:24

// per-cell flag byte (construction and edits)
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

// Read-only view of one device-resident structure, passed by value. Queries
// read occupancy from `rowbits`: per 32-cell run of a grid row one uint2 of
// {occupied bits, clear bits} (4 MB at 4000x4000, so it stays L2-resident).
struct CddtView {
  const uint8_t* __restrict__ flags;      // w*h (build / prune / edit bookkeeping)
  const uint2* __restrict__ rowbits;      // h*wpr {occupied, clear} bits
  int wpr;                                // words per grid row
  const uint32_t* __restrict__ row_off;   // rows+1, CSR into zp
  const float* __restrict__ zp;           // zero points, ascending per row
  const float* __restrict__ hints;        // rows x kHintFloats: row records (CSR range + probes)
  const SliceParam* __restrict__ slices;  // S
  const double4* __restrict__ dirs;       // K (cos, sin, 1/cos, 1/sin), axis-snapped (cddt.cpp:30-42)
  const double4* __restrict__ pdirs;      // K (slice cos, slice sin, direction cos, direction sin)
  const uint32_t* __restrict__ rbase;     // S: slice row bases (4 B each: a few lines in all)
  int w, h, K, S;
  double max_range;
  // checked builds (-DRL_CHECKED): bounds of the arrays above and the
  // violation counter {count, first code} the device assertions bump
  unsigned long long* chk;
  uint32_t n_rows, n_zp;
};

// Device bounds assertions of the checked build (RL_CHECKED; compute-sanitizer
// is unavailable on the GPU pool): a failed check bumps c.chk[0] and records
// its site code in c.chk[1]; rl_debug_checks() reads them back. Compiled out
// otherwise.
#ifdef RL_CHECKED
static __device__ __noinline__ void rl_check_fail(unsigned long long* chk, unsigned code) {
  if (chk && atomicAdd(chk, 1ull) == 0ull) chk[1] = code;
}
#define RL_DCHECK(view, cond, code)                          \
  do {                                                       \
    if (!(cond)) ::rl::rl_check_fail((view).chk, (code));    \
  } while (0)
#else
#define RL_DCHECK(view, cond, code) ((void)0)
#endif

__host__ __device__ __forceinline__ double fmin_std(double a, double b) { return (b < a) ? b : a; }
__host__ __device__ __forceinline__ double fmax_std(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ long iround(double v) { return (long)ceil(v - 0.5); }  // raycast.hpp:17


// a / d correctly rounded, given r = RN(1/d) (host IEEE division).
// Markstein's theorem: if q is a faithful rounding of a/d (within one ulp)
// and r = RN(1/d), the FMA residual e = a - d q is exact and RN(q + e r) =
// RN(a/d) — barring overflow and subnormals, which the walker's and
// direction_index's operands never reach (|a| < 2^16; |d| >= sin(2pi/K), far
// above the subnormal range for any usable K).
// q0 = RN(a r) alone is NOT always faithful (|q0 - a/d| can reach ~2 ulp at
// the top of a binade), so one correction step first makes it faithful:
//   q1 = RN(q0 + RN(a - d q0) r):  |q1 - a/d| <= 1/2 ulp + 2 ulp * 2^-52 < 1 ulp,
// and the second step rounds correctly. Five FP64 operations instead of the
// ~30-instruction IEEE division sequence; tests/fast_div_check.c also checks
// it bit for bit against IEEE division on the walker's operand distribution
// (float and f64 origins, cell centres, lattice-adjacent origins).
__device__ __forceinline__ double div_rn(double a, double d, double r) {
  const double q0 = __dmul_rn(a, r);
  const double q1 = fma(fma(-d, q0, a), r, q0);
#ifdef RL_DIV_ONE_STEP  // A/B only: round 1's single correction (empirically, not provably, exact)
  return q1;
#else
  return fma(fma(-d, q1, a), r, q1);
#endif
}

__device__ __forceinline__ double normalize_angle_2pi(double t) {  // raycast.hpp:20-25
  if (t >= 0.0 && t < kTwoPi) return t;  // fmod(t, 2pi) == t exactly here
  // fmod is exact: on [2pi, 4pi) it is t - 2pi (Sterbenz, so the subtraction
  // is exact too); on (-2pi, 0) it is t itself, then the reference adds 2pi.
  if (t >= kTwoPi && t < 2.0 * kTwoPi) return t - kTwoPi;
  if (t < 0.0 && t > -kTwoPi) {
    t += kTwoPi;
    return t >= kTwoPi ? 0.0 : t;
  }
  t = fmod(t, kTwoPi);
  if (t < 0) t += kTwoPi;
  if (t >= kTwoPi) t = 0.0;
  return t;
}

__device__ __forceinline__ int direction_index(double theta, int K) {  // raycast.hpp:36-40
  // iround(theta * K / 2pi) % K with the quotient correctly rounded
  const double v = ceil(div_rn(theta * (double)K, kTwoPi, kInvTwoPi) - 0.5);
  if (v >= 0.0 && v <= (double)K) {  // theta in [0, 2pi): no modulo needed
    const int i = (int)v;
    return i == K ? 0 : i;
  }
  long i = (long)v % K;
  if (i < 0) i += K;
  return (int)i;
}

__device__ __forceinline__ bool in_bounds(const CddtView& c, int x, int y) {
  return (unsigned)x < (unsigned)c.w && (unsigned)y < (unsigned)c.h;
}
__device__ __forceinline__ bool occupied(const CddtView& c, int x, int y) {
  RL_DCHECK(c, unsigned(x) < unsigned(c.w) && unsigned(y) < unsigned(c.h), 1);
  return (__ldg(&c.rowbits[y * c.wpr + (x >> 5)].x) >> (x & 31)) & 1u;
}

// RayWalker (ray_walker.hpp:21-104). Every boundary parameter is the
// reference's ((double)c + 1 - o) / d or ((double)c - o) / d, rounded exactly.
//
// kBranchFree hoists the per-axis sign logic of boundary_t/advance into
// per-query constants (step, bias 1.0/0.0, axis-parallel flag) and computes
// both next boundaries with selects, so lanes walking in different directions
// do not diverge. It costs registers and one extra division per step: it pays
// in the dedicated walk kernels (k_walk_pass, every lane walking) and not
// in the monolithic kernels, which use the branchy form.
template <bool kBranchFree>
struct Walker {
  double ox, oy, dx, dy, rx, ry, t, tnx, tny;
  int cx, cy;
  double bx, by;  // kBranchFree: 1.0 when the axis direction is positive, else 0.0
  int sx, sy;     // kBranchFree: cell step per axis
  bool zx, zy;    // kBranchFree: axis-parallel (boundary parameter +inf)

  __device__ __forceinline__ static double inf() {
    return __longlong_as_double(0x7ff0000000000000ll);
  }
  __device__ __forceinline__ double bnd_x(int c) const {
    if (kBranchFree) {
      const double v = div_rn(((double)c + bx) - ox, dx, rx);
      return zx ? inf() : v;
    }
    if (dx > 0) return div_rn((double)c + 1.0 - ox, dx, rx);
    if (dx < 0) return div_rn((double)c - ox, dx, rx);
    return inf();
  }
  __device__ __forceinline__ double bnd_y(int c) const {
    if (kBranchFree) {
      const double v = div_rn(((double)c + by) - oy, dy, ry);
      return zy ? inf() : v;
    }
    if (dy > 0) return div_rn((double)c + 1.0 - oy, dy, ry);
    if (dy < 0) return div_rn((double)c - oy, dy, ry);
    return inf();
  }
  __device__ __forceinline__ void place(double tt) {  // ray_walker.hpp:62-73
    t = tt;
    const double px = ox + tt * dx, py = oy + tt * dy;
    const double fx = floor(px), fy = floor(py);
    // a point exactly on a boundary moving in the negative direction enters
    // the lower cell
    cx = (int)fx - ((dx < 0 && px == fx) ? 1 : 0);
    cy = (int)fy - ((dy < 0 && py == fy) ? 1 : 0);
    tnx = bnd_x(cx);
    tny = bnd_y(cy);
  }
  // walker.emplace(...) (place(0)) followed by seek(tt): place() resets the
  // whole state, so this is one place at max(0, tt)
  __device__ __forceinline__ void init_params(double x, double y, const double4& dir) {
    ox = x;
    oy = y;
    dx = dir.x;
    dy = dir.y;
    rx = dir.z;
    ry = dir.w;
    if (kBranchFree) {
      bx = dx > 0 ? 1.0 : 0.0;
      by = dy > 0 ? 1.0 : 0.0;
      sx = dx > 0 ? 1 : -1;
      sy = dy > 0 ? 1 : -1;
      zx = !(dx > 0) && !(dx < 0);
      zy = !(dy > 0) && !(dy < 0);
    }
  }
  __device__ __forceinline__ void init_at(double x, double y, const double4& dir, double tt) {
    init_params(x, y, dir);
    place(tt > 0.0 ? tt : 0.0);
  }
  // the state a previous scan left (tnx/tny are bnd_x(cx)/bnd_y(cy) always)
  __device__ __forceinline__ void restore(double x, double y, const double4& dir, int ccx,
                                          int ccy, double tt) {
    init_params(x, y, dir);
    t = tt;
    cx = ccx;
    cy = ccy;
    tnx = bnd_x(cx);
    tny = bnd_y(cy);
  }
  __device__ __forceinline__ void seek(double tt) {  // ray_walker.hpp:36-38
    if (tt > t) place(tt);
  }
  __device__ __forceinline__ void advance() {  // ray_walker.hpp:81-97
    if (kBranchFree) {
      // equal parameters: exact lattice-corner crossing, both axes step
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
      return;
    }
    if (tnx == tny) {
      t = tnx;
      cx += dx > 0 ? 1 : -1;
      cy += dy > 0 ? 1 : -1;
      tnx = bnd_x(cx);
      tny = bnd_y(cy);
    } else if (tnx < tny) {
      t = tnx;
      cx += dx > 0 ? 1 : -1;
      tnx = bnd_x(cx);
    } else {
      t = tny;
      cy += dy > 0 ? 1 : -1;
      tny = bnd_y(cy);
    }
  }
  // Advance until entering an occupied cell (returns its entry t), past
  // t_limit (kWalkNone) or off the grid (kWalkExit).  ray_walker.hpp:51-59
  __device__ __forceinline__ double scan_to(const CddtView& c, double lim) {
    for (;;) {
      if (!in_bounds(c, cx, cy)) return kWalkExit;
      if (occupied(c, cx, cy)) return t;
      const double tn = tnx < tny ? tnx : tny;
      if (tn > lim) return kWalkNone;
      advance();
    }
  }
};

// Row records: one 32-byte sector per row with the CSR range and the zero
// points the row's binary search probes first, so a query's first three
// search steps arrive with its row instead of one round trip each:
//   lo, n (u32 bits), L1, L2(0), L2(1), L3(00), L3(01), L3(10)
// indexed by the decisions taken so far (1 = the probe passed, the search
// moved right); L3(11) falls back to a zero-point load. Derived from row_off
// and zp after every structure change (refresh_row_hints).
constexpr int kHintLevels = 3, kHintFloats = 8;
#ifndef RL_LINEAR_TAIL
#define RL_LINEAR_TAIL 4
#endif
constexpr int kLinearTail = RL_LINEAR_TAIL;  // rows searched by one parallel load at the end

// index probed at `level` (0-based) after the decisions `path` (level bits,
// first decision most significant); false when the search ended earlier
__host__ __device__ __forceinline__ bool hint_index(uint32_t n, int level, uint32_t path,
                                                   uint32_t* idx) {
  uint32_t first = 0, len = n;
  for (int l = 0;; l++) {
    if (len == 0) return false;
    const uint32_t half = len >> 1;
    if (l == level) {
      *idx = first + half;
      return true;
    }
    if ((path >> (level - 1 - l)) & 1u) {
      first += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
}

// Number of leading elements e of v[0, n) with double(e) <= xq (forward:
// !(xq < e), std::upper_bound) or double(e) < xq (backward, std::lower_bound),
// with libstdc++'s halving sequence (cddt.hpp:106-131). The comparisons run in
// the float domain, exactly: for a float e,
//   double(e) <= xq  <=>  e <= RD_f32(xq)     and     double(e) < xq  <=>  e < RU_f32(xq)
// (no float lies strictly between RD_f32(xq) and RU_f32(xq)). The first
// kHintLevels steps are taken from the row record: the same index sequence
// and comparisons, so the same result. It also
// reports the first candidate's zero point when the search probed it (the
// forward candidate is the leftmost failing probe, the backward one the
// rightmost passing probe), which saves that load for short rows.
struct RowSearch {
  uint32_t first;  // partition point
  uint32_t kidx;   // index whose value is kval (~0u: none)
  float kval;
};

__device__ __forceinline__ RowSearch partition_point_hinted(const float* __restrict__ v,
                                                            uint32_t n, double xq, bool forward,
                                                            float4 h, float4 h2) {
  RowSearch r{0, ~0u, 0.f};
  // one strict threshold for both directions: for a float e,
  //   e <= RD_f32(xq)  <=>  e < nextup(RD_f32(xq))      (forward)
  //   e <  RU_f32(xq)                                    (backward)
  const float thr = forward ? nextafterf(__double2float_rd(xq), __int_as_float(0x7f800000))
                            : __double2float_ru(xq);
  uint32_t len = n, path = 0;
#pragma unroll
  for (int l = 0; l < kHintLevels; l++) {
    if (len == 0) return r;
    const uint32_t half = len >> 1, mid = r.first + half;
    float e;
    if (l == 0) {
      e = h.z;
    } else if (l == 1) {
      e = path ? h2.x : h.w;
    } else {
      e = path == 0 ? h2.y : path == 1 ? h2.z : path == 2 ? h2.w : __ldg(v + mid);
    }
    const bool pass = e < thr;
    if (pass != forward) {
      r.kidx = mid;
      r.kval = e;
    }
    if (pass) {
      r.first = mid + 1;
      len -= half + 1;
    } else {
      len = half;
    }
    path = (path << 1) | (pass ? 1u : 0u);
  }
  while (len > kLinearTail) {
    const uint32_t half = len >> 1, mid = r.first + half;
    const float e = __ldg(v + mid);
    const bool pass = e < thr;
    if (pass != forward) {
      r.kidx = mid;
      r.kval = e;
    }
    if (pass) {
      r.first = mid + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  if (kLinearTail > 0 && len > 0) {
    // the last <= kLinearTail elements in one round trip: the partition point
    // is the count of passing elements (the predicate is monotone); slots
    // past the row hold +inf, which never passes
    float e[kLinearTail > 0 ? kLinearTail : 1];
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kLinearTail; k++) {
      e[k] = uint32_t(k) < len ? __ldg(v + r.first + k) : __int_as_float(0x7f800000);
      cnt += e[k] < thr ? 1u : 0u;
    }
    // the first candidate: forward e[cnt], backward e[cnt - 1], when in range
    const int ci = forward ? int(cnt) : int(cnt) - 1;
    float cv = e[0];
#pragma unroll
    for (int k = 1; k < kLinearTail; k++) cv = ci == k ? e[k] : cv;
    if (ci >= 0 && uint32_t(ci) < len) {
      r.kidx = r.first + uint32_t(ci);
      r.kval = cv;
    }
    r.first += cnt;
  }
  return r;
}

// Outcome of one query beyond the range: the occupied cell that settled it
// and the resolving zero point (what MarkSink::mark receives, cddt.cpp:249,259).
struct CastOut {
  int32_t hit;      // y*w+x or -1
  uint32_t res_g;   // global row of the resolving zero point
  int32_t res_idx;  // index within the row, -1 when no zero point resolved
};

struct __align__(32) RowRecord {
  float4 a, b;
};

// Per-query geometry shared by the whole and the split forms.
struct QueryRow {
  bool forward;
  double xq;        // projected x' of the query (cddt.hpp:31)
  uint32_t g;       // global row
  uint32_t lo, hi;  // CSR range of the row
  float4 hint, hint2;  // the row record
};
__device__ __forceinline__ QueryRow query_row(const CddtView& c, double x, double y, int a) {
  QueryRow q;
  q.forward = a < c.S;
  const int s = q.forward ? a : a - c.S;
  const SliceParam sp = c.slices[s];
  q.xq = x * sp.cos_t + y * sp.sin_t;                            // cddt.hpp:31
  const double yq = -x * sp.sin_t + y * sp.cos_t + sp.y_offset;  // cddt.hpp:32
  int row = (int)yq;
  if (row < 0) row = 0;
  if (row >= sp.bin_count) row = sp.bin_count - 1;
  q.g = sp.row_base + (uint32_t)row;
  RL_DCHECK(c, s >= 0 && s < c.S && q.g < c.n_rows, 2);
  // requested together with the origin cell's bits: the two are independent
  // one 32-byte load (LDG.256) rather than two 16-byte ones: one L1 wavefront per lane
  // not allocated in L1: a random row's record is read once per query, and L1
  // is worth more to the direction tables, bitmaps and search tails (-0.8 %)
  RowRecord rec;
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(rec.a.x), "=f"(rec.a.y), "=f"(rec.a.z), "=f"(rec.a.w), "=f"(rec.b.x), "=f"(rec.b.y),
        "=f"(rec.b.z), "=f"(rec.b.w)
      : "l"(reinterpret_cast<const RowRecord*>(c.hints) + q.g));

  q.hint = rec.a;
  q.hint2 = rec.b;
  q.lo = __float_as_uint(q.hint.x);
  q.hi = q.lo + __float_as_uint(q.hint.y);
  RL_DCHECK(c, q.lo <= q.hi && q.hi <= c.n_zp, 4);  // every zero-point read lies in [lo, hi)
  return q;
}

// SliceProjection::make's offset and bin count (cddt.cpp:44-60), recomputed
// from the slice's cos/sin with the host's operations (init_geometry), so
// bit-identical to the table values.
__device__ __forceinline__ void slice_extent(const CddtView& c, double cs, double sn,
                                             double* y_offset, int* bin_count) {
  const double A = 0.0, B = -double(c.w) * sn, C = double(c.h) * cs, D = B + C;
  const double lo = fmin_std(fmin_std(A, B), fmin_std(C, D));
  const double hi = fmax_std(fmax_std(A, B), fmax_std(C, D));
  *y_offset = -lo;
  *bin_count = int(ceil(hi - lo)) + 1;
}

// The query's slice row and its record: one 32-byte per-direction entry
// (slice cos/sin and the direction's cos/sin) rather than the slice and
// direction records, the slice's offset and bin count recomputed, the row
// base from the 4-byte-per-slice table. Returns the direction in *dir.
__device__ __forceinline__ QueryRow query_row(const CddtView& c, double x, double y, int a,
                                                 double2* dir) {
  QueryRow q;
  q.forward = a < c.S;
  const int s = q.forward ? a : a - c.S;
  double4 pd;  // one 256-bit load: a single L1 wavefront per lane
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(pd.x), "=d"(pd.y), "=d"(pd.z), "=d"(pd.w)
      : "l"(c.pdirs + a));
  *dir = make_double2(pd.z, pd.w);
  double y_offset;
  int bin_count;
  slice_extent(c, pd.x, pd.y, &y_offset, &bin_count);
  q.xq = x * pd.x + y * pd.y;                            // cddt.hpp:31
  const double yq = -x * pd.y + y * pd.x + y_offset;     // cddt.hpp:32
  int row = (int)yq;
  if (row < 0) row = 0;
  if (row >= bin_count) row = bin_count - 1;
  q.g = __ldg(c.rbase + s) + uint32_t(row);
  RL_DCHECK(c, a >= 0 && a < c.K && q.g < c.n_rows, 3);
  // not allocated in L1: a random row's record is read once per query, and L1
  // is worth more to the direction tables, bitmaps and search tails (-0.8 %)
  RowRecord rec;
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(rec.a.x), "=f"(rec.a.y), "=f"(rec.a.z), "=f"(rec.a.w), "=f"(rec.b.x), "=f"(rec.b.y),
        "=f"(rec.b.z), "=f"(rec.b.w)
      : "l"(reinterpret_cast<const RowRecord*>(c.hints) + q.g));

  q.hint = rec.a;
  q.hint2 = rec.b;
  q.lo = __float_as_uint(q.hint.x);
  q.hi = q.lo + __float_as_uint(q.hint.y);
  RL_DCHECK(c, q.lo <= q.hi && q.hi <= c.n_zp, 4);  // every zero-point read lies in [lo, hi)
  return q;
}

// Landing-cell probe (cddt.cpp:239-253): the point at distance d settles the
// candidate when it lies strictly inside an occupied cell.
__device__ __forceinline__ bool landing_hit(const CddtView& c, double px, double py,
                                            int32_t* cell) {
  if (!(px >= 0.0 && py >= 0.0 && px < (double)c.w && py < (double)c.h)) return false;
  const int hx = (int)px, hy = (int)py;
  const double fx = px - (double)hx, fy = py - (double)hy;
  if (fx > kLatticeEps && fx < 1.0 - kLatticeEps && fy > kLatticeEps && fy < 1.0 - kLatticeEps &&
      occupied(c, hx, hy)) {
    *cell = hy * c.w + hx;
    return true;
  }
  return false;
}

// A second probe of a verification window [t0, lim] = [max(0, d - 0.7072),
// d + 0.7072] (cddt.cpp:254-261), near its far end: if the ray point at
// d + kProbeAhead lies strictly inside an occupied cell (landing_hit's
// margin), the reference's walker enters that cell - it covers the segment
// cell by cell, and a cell holding a point of the segment strictly inside is
// never one touched at a corner only - or an earlier occupied cell, and it
// cannot leave the grid first (the grid is convex and both the origin and
// that cell lie in it). So the window hits and the cast is d, decided
// without a walker. The far end is where a ray that entered an obstacle
// within the window is most likely still inside it: measured at config 3,
// this one probe settles 57 % of the first windows (a probe at d +- 0.5: 46 %).
#ifndef RL_WIN_PROBE
#define RL_WIN_PROBE 1
#endif
// where the probe is used (A/B switches). Kept: phase 1 (config 3 -7 %),
// the near-field kernel, the sensor model's casts (config 4 -1.4 %). Not
// kept: the window passes (+1 % there: their windows mostly come clean) and
// the single-kernel batch cast (+10 % at 100 k queries: longer divergent
// lanes in a one-wave launch).
#ifndef RL_PROBE_P1
#define RL_PROBE_P1 RL_WIN_PROBE
#endif
#ifndef RL_PROBE_PASS
#define RL_PROBE_PASS 0
#endif
#ifndef RL_PROBE_NEAR
#define RL_PROBE_NEAR RL_WIN_PROBE
#endif
#ifndef RL_PROBE_MONO
#define RL_PROBE_MONO 0
#endif
#ifndef RL_PROBE_SENSOR
#define RL_PROBE_SENSOR RL_WIN_PROBE
#endif
constexpr double kProbeAhead = 0.7071;  // < kVerifyHalf: inside the window
__device__ __forceinline__ bool window_probe_hit(const CddtView& c, double x, double y,
                                                 double dx, double dy, double d) {
  const double tp = d + kProbeAhead;
  int32_t cell;
  return landing_hit(c, x + tp * dx, y + tp * dy, &cell);
}

// Cddt::directional_cast (cddt.cpp:207-269).
// exact_hit_cell: o.hit must be the cell the reference's walker enters
// first (the hit-cell outputs); otherwise a window may be settled by
// window_probe_hit, whose cell can be a later one (same range and resolving
// index).
__device__ __forceinline__ double directional_cast(const CddtView& c, double x, double y, int a,
                                                   CastOut& o, bool exact_hit_cell = true) {
  o.hit = -1;
  o.res_idx = -1;
  o.res_g = 0;
  const int cxi = (int)floor(x), cyi = (int)floor(y);
  if (!in_bounds(c, cxi, cyi)) return c.max_range;  // cddt.cpp:209
  double2 d2;  // the direction's cos/sin; the walker's full entry is read when one is needed
  const QueryRow q = query_row(c, x, y, a, &d2);
  RL_DCHECK(c, unsigned(cxi) < unsigned(c.w) && unsigned(cyi) < unsigned(c.h), 5);
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {  // cddt.cpp:210
    o.hit = cyi * c.w + cxi;
    return 0.0;
  }
  Walker<false> wk;
  bool have_walker = false;
  if (!((w0.y >> (cxi & 31)) & 1u)) {
    // something occupied within one cell: resolve the near field exactly (cddt.cpp:225-232)
    wk.init_at(x, y, c.dirs[a], 0.0);
    have_walker = true;
    const double r = wk.scan_to(c, kNearField);
    if (r >= 0.0) {
      o.hit = wk.cy * c.w + wk.cx;
      return (c.max_range < r) ? c.max_range : r;
    }
    if (r == kWalkExit) return c.max_range;
  }
  const float* __restrict__ v = c.zp + q.lo;
  const RowSearch rs =
      partition_point_hinted(v, q.hi - q.lo, q.xq, q.forward, q.hint, q.hint2);
  const int n = (int)(q.hi - q.lo);
  const int step = q.forward ? 1 : -1;
  for (int idx = q.forward ? (int)rs.first : (int)rs.first - 1; idx >= 0 && idx < n;
       idx += step) {
    // consider(v, index), cddt.cpp:236-262
    const double vv = (double)(uint32_t(idx) == rs.kidx ? rs.kval : __ldg(v + idx));
    const double d = q.forward ? vv - q.xq : q.xq - vv;
    if (d >= c.max_range) break;
    int32_t cell;
    if (landing_hit(c, x + d * d2.x, y + d * d2.y, &cell)) {
      o.hit = cell;
      o.res_g = q.g;
      o.res_idx = idx;
      return d;
    }
    // verification window around the candidate (cddt.cpp:254-261)
#if RL_PROBE_MONO
    if (!exact_hit_cell && window_probe_hit(c, x, y, d2.x, d2.y, d)) {
      o.hit = -2;  // an occupied cell of the window, not necessarily the walker's first
      o.res_g = q.g;
      o.res_idx = idx;
      return d;
    }
#endif
    if (!have_walker) {
      wk.init_at(x, y, c.dirs[a], d - kVerifyHalf);
      have_walker = true;
    } else {
      wk.seek(d - kVerifyHalf);
    }
    const double r = wk.scan_to(c, d + kVerifyHalf);
    if (r == kWalkExit) break;
    if (r < 0.0) continue;
    o.hit = wk.cy * c.w + wk.cx;
    o.res_g = q.g;
    o.res_idx = idx;
    return d;
  }
  return c.max_range;
}

// ---- split form for the deferred-walk batch kernels (rl_query.cu) ----
// Phase 1 runs cddt.cpp:207-269 up to the first point where a RayWalker is
// needed: a non-clear origin (near-field walk) or a candidate whose landing
// probe does not settle it (verification window). Phase 2 resumes exactly
// there. Split and unsplit runs take the same decisions in the same order.
struct WalkDefer {
  uint32_t lo, n;  // CSR row of the query
  int idx;         // candidate whose window walk is pending; -1: near field
  float cval;      // its zero point (phase 1 loaded it)
};

// Register diet (32 registers, no spills, so 2048 resident threads per SM
// instead of 1536; -1 % per step): the query enters as floats and its doubles
// are rebuilt (exactly) after the row search; the direction and the projected
// x' are not kept across the search either - the 32-byte per-direction entry
// is read again (an L1 hit) and x' recomputed with the same operations.
__device__ __forceinline__ bool directional_cast_p1(const CddtView& c, float xf, float yf, int a,
                                                    double* result, WalkDefer* def) {
  double x = double(xf), y = double(yf);
  const int cxi = (int)floor(x), cyi = (int)floor(y);
  if (!in_bounds(c, cxi, cyi)) {
    *result = c.max_range;
    return true;
  }
  double2 dir;
  const QueryRow q = query_row(c, x, y, a, &dir);
  RL_DCHECK(c, unsigned(cxi) < unsigned(c.w) && unsigned(cyi) < unsigned(c.h), 5);
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {
    *result = 0.0;
    return true;
  }
  def->lo = q.lo;
  def->n = q.hi - q.lo;
  if (!((w0.y >> (cxi & 31)) & 1u)) {
    def->idx = -1;  // near field needs the walker: phase 2 redoes the whole query
    def->cval = 0.f;
    return false;
  }
  const RowSearch rs =
      partition_point_hinted(c.zp + q.lo, q.hi - q.lo, q.xq, q.forward, q.hint, q.hint2);
  const int n = (int)(q.hi - q.lo);
  const bool forward = a < c.S;
  const int step = forward ? 1 : -1;
  for (int idx = forward ? (int)rs.first : (int)rs.first - 1; idx >= 0 && idx < n;
       idx += step) {
    const float fv = uint32_t(idx) == rs.kidx ? rs.kval : __ldg(c.zp + q.lo + idx);
    const double vv = (double)fv;
    // the barrier keeps the compiler from holding the first conversion's doubles
    asm volatile("" : "+f"(xf), "+f"(yf));
    x = double(xf);
    y = double(yf);
    double pcs, psn;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(pcs), "=d"(psn), "=d"(dir.x), "=d"(dir.y)
                 : "l"(c.pdirs + a));
    const double xq = x * pcs + y * psn;  // cddt.hpp:31, as in query_row
    const double d = forward ? vv - xq : xq - vv;
    if (d >= c.max_range) break;
    int32_t cell;
    if (landing_hit(c, x + d * dir.x, y + d * dir.y, &cell)) {
      *result = d;
      return true;
    }
#if RL_PROBE_P1
    if (window_probe_hit(c, x, y, dir.x, dir.y, d)) {
      *result = d;
      return true;
    }
#endif
    def->idx = idx;  // first verification window: hand over to phase 2
    def->cval = fv;
    return false;
  }
  *result = c.max_range;
  return true;
}

// Phase 2 for a deferred window. The origin was clear, so no walker exists
// yet: emplace + seek(d - kVerifyHalf) is one place(); then the reference's
// candidate loop continues. A query may need many windows (rays grazing a
// wall meet one failing candidate per wall cell), so the walk kernels scan
// at most `cap` windows and hand the rest on: WinState is everything the
// candidate loop carries between iterations (the walker's cell and entry
// parameter; its boundary parameters are functions of the cell).
struct WinState {
  uint32_t lo, n;  // CSR row of the query
  int idx;         // next candidate
  int cx, cy;      // walker cell and entry parameter (continuations)
  double t;
  float cval;      // FRESH: the zero point of candidate idx, from phase 1
};

// FRESH: s.idx is phase 1's candidate (landing probe done, no walker yet);
// otherwise s continues a previous pass (walker restored, s.idx not probed).
// true: settled, *result set. false: `cap` windows scanned and candidates
// remain; s continues at s.idx.
template <bool FRESH>
__device__ __forceinline__ bool resume_windows(const CddtView& c, double x, double y, int a,
                                               WinState& s, int cap, double* result) {
  const bool forward = a < c.S;
  // a forward direction is its slice's own direction (the same glibc cos/sin),
  // so only backward queries read the slice record
  const double4 dir = c.dirs[a];
  double cs = dir.x, sn = dir.y;
  if (!forward) {
    const double2 sl = __ldg(reinterpret_cast<const double2*>(c.slices + (a - c.S)));
    cs = sl.x;
    sn = sl.y;
  }
  const double xq = x * cs + y * sn;
  const float* __restrict__ v = c.zp + s.lo;
  const int n = (int)s.n, step = forward ? 1 : -1;
  RL_DCHECK(c, uint64_t(s.lo) + s.n <= c.n_zp && a >= 0 && a < c.K, 6);
  Walker<true> wk;
  int idx = s.idx, windows = 0;
  if (FRESH) {
    const double vv = (double)s.cval;
    const double d = forward ? vv - xq : xq - vv;
    *result = c.max_range;
    if (d >= c.max_range) return true;
    wk.init_at(x, y, dir, d - kVerifyHalf);
    const double r = wk.scan_to(c, d + kVerifyHalf);
    if (r == kWalkExit) return true;
    if (r >= 0.0) {
      *result = d;
      return true;
    }
    windows = 1;
    idx += step;
  } else {
    wk.restore(x, y, dir, s.cx, s.cy, s.t);
  }
  for (; idx >= 0 && idx < n; idx += step) {
    if (windows == cap) {
      s.idx = idx;
      s.cx = wk.cx;
      s.cy = wk.cy;
      s.t = wk.t;
      return false;
    }
    const double vv = (double)__ldg(v + idx);
    const double d = forward ? vv - xq : xq - vv;
    if (d >= c.max_range) break;
    int32_t cell;
    if (landing_hit(c, x + d * dir.x, y + d * dir.y, &cell)
#if RL_PROBE_PASS
        || window_probe_hit(c, x, y, dir.x, dir.y, d)
#endif
    ) {
      *result = d;
      return true;
    }
    wk.seek(d - kVerifyHalf);
    const double r = wk.scan_to(c, d + kVerifyHalf);
    windows++;
    if (r == kWalkExit) break;
    if (r < 0.0) continue;
    *result = d;
    return true;
  }
  *result = c.max_range;
  return true;
}


// Near-field records (origin not clear): the near-field walk, the row search
// and the candidate loop up to the first verification window. A query that
// needs one leaves with the candidate loop's state (the walker exists), for
// resume_windows<false>; its landing probe is repeated there (same answer).
// Phase 1 already established the origin is in bounds and unoccupied.
__device__ __forceinline__ bool near_cast_p1(const CddtView& c, double x, double y, int a,
                                             double* result, WinState* s) {
  const QueryRow q = query_row(c, x, y, a);
  const double4 dir = c.dirs[a];
  Walker<true> wk;
  wk.init_at(x, y, dir, 0.0);
  const double r = wk.scan_to(c, kNearField);  // cddt.cpp:225-232
  if (r >= 0.0) {
    *result = (c.max_range < r) ? c.max_range : r;
    return true;
  }
  *result = c.max_range;
  if (r == kWalkExit) return true;
  const RowSearch rs =
      partition_point_hinted(c.zp + q.lo, q.hi - q.lo, q.xq, q.forward, q.hint, q.hint2);
  const int n = (int)(q.hi - q.lo);
  const int step = q.forward ? 1 : -1;
  for (int idx = q.forward ? (int)rs.first : (int)rs.first - 1; idx >= 0 && idx < n;
       idx += step) {
    const double vv =
        (double)(uint32_t(idx) == rs.kidx ? rs.kval : __ldg(c.zp + q.lo + idx));
    const double d = q.forward ? vv - q.xq : q.xq - vv;
    if (d >= c.max_range) break;
    int32_t cell;
    if (landing_hit(c, x + d * dir.x, y + d * dir.y, &cell)
#if RL_PROBE_NEAR
        || window_probe_hit(c, x, y, dir.x, dir.y, d)
#endif
    ) {
      *result = d;
      return true;
    }
    *s = WinState{q.lo, uint32_t(n), idx, wk.cx, wk.cy, wk.t, 0.f};
    return false;
  }
  return true;
}

// ---- long casts: the candidate loop evaluated a warp at a time ----
//
// A ray grazing a wall meets one failing candidate per wall cell, so a few
// casts run tens of verification windows while their warp and CTA wait: in a
// launch that fits the GPU in one wave (a config-2 sensor update, a config-1
// batch) those casts decide the kernel time. Each candidate's verdict is a pure function of the
// candidate: its landing probe, and the cells of its window [d - 0.7072,
// d + 0.7072] (cddt.cpp:236-262). The reference's single walker covers each
// window from max(its position, d - 0.7072); the cells between d - 0.7072 and
// that position were already entered and found free by the earlier windows
// or the near-field walk, so a fresh walker placed at d - 0.7072 reaches the
// same verdict (hit, clean, or leaving the grid). The first non-clean verdict
// in candidate order decides the cast exactly as the sequential loop does —
// so 32 lanes can evaluate 32 consecutive candidates at once.
//
// Phase A (every thread, its own items) stops a cast after RL_COOP_WCAP
// windows and queues it in shared memory {pose, direction, next candidate,
// output slot}; phase B hands each queued cast to a whole warp (resume_coop).
#ifndef RL_COOP_WCAP
#define RL_COOP_WCAP 4  // windows a thread scans before handing its cast to a warp
#endif
constexpr int kLongQueue = 64;  // queued casts per CTA (beyond: the thread finishes alone)

struct LongCast {
  double x, y;
  int32_t a, idx;
  uint32_t slot, pad;
};

// directional_cast (cddt.cpp:207-269) that stops after `cap` verification
// windows: returns false with *next = the next candidate when it stopped
// (cap < 0: no cap).
__device__ __forceinline__ bool directional_cast_capped(const CddtView& c, double x, double y,
                                                        int a, int cap, double* res, int* next) {
  const int cxi = (int)floor(x), cyi = (int)floor(y);
  *res = c.max_range;
  if (!in_bounds(c, cxi, cyi)) return true;  // cddt.cpp:209
  const QueryRow q = query_row(c, x, y, a);
  RL_DCHECK(c, unsigned(cxi) < unsigned(c.w) && unsigned(cyi) < unsigned(c.h), 5);
  const uint2 w0 = __ldg(&c.rowbits[cyi * c.wpr + (cxi >> 5)]);
  if ((w0.x >> (cxi & 31)) & 1u) {  // cddt.cpp:210
    *res = 0.0;
    return true;
  }
  const double4 dir = c.dirs[a];
  Walker<false> wk;
  bool have_walker = false;
  if (!((w0.y >> (cxi & 31)) & 1u)) {  // near field, cddt.cpp:225-232
    wk.init_at(x, y, dir, 0.0);
    have_walker = true;
    const double r = wk.scan_to(c, kNearField);
    if (r >= 0.0) {
      *res = (c.max_range < r) ? c.max_range : r;
      return true;
    }
    if (r == kWalkExit) return true;
  }
  const float* __restrict__ v = c.zp + q.lo;
  const int n = (int)(q.hi - q.lo);
  const RowSearch rs = partition_point_hinted(v, uint32_t(n), q.xq, q.forward, q.hint, q.hint2);
  const int step = q.forward ? 1 : -1;
  int windows = 0;
  for (int idx = q.forward ? (int)rs.first : (int)rs.first - 1; idx >= 0 && idx < n;
       idx += step) {
    const double vv = (double)(uint32_t(idx) == rs.kidx ? rs.kval : __ldg(v + idx));
    const double d = q.forward ? vv - q.xq : q.xq - vv;
    if (d >= c.max_range) break;
    int32_t cell;
    if (landing_hit(c, x + d * dir.x, y + d * dir.y, &cell)
#if RL_PROBE_SENSOR
        || window_probe_hit(c, x, y, dir.x, dir.y, d)
#endif
    ) {
      *res = d;
      return true;
    }
    if (windows == cap) {
      *next = idx;  // this candidate's window is the first one not scanned
      return false;
    }
    if (!have_walker) {
      wk.init_at(x, y, dir, d - kVerifyHalf);
      have_walker = true;
    } else {
      wk.seek(d - kVerifyHalf);
    }
    const double r = wk.scan_to(c, d + kVerifyHalf);
    windows++;
    if (r == kWalkExit) break;
    if (r < 0.0) continue;
    *res = d;
    return true;
  }
  return true;
}

// The rest of a cast from candidate idx0 on, by all 32 lanes of a warp (the
// arguments are warp-uniform): lane k takes candidate idx0 +- (32 j + k).
__device__ __forceinline__ double resume_coop(const CddtView& c, double x, double y, int a,
                                              int idx0) {
  const QueryRow q = query_row(c, x, y, a);
  const double4 dir = c.dirs[a];
  const float* __restrict__ v = c.zp + q.lo;
  const int n = (int)(q.hi - q.lo);
  const int lane = threadIdx.x & 31, step = q.forward ? 1 : -1;
  for (int base = idx0;; base += 32 * step) {
    const int idx = base + lane * step;
    int verdict = 0;  // 0: clean window, 1: settled at d, 2: the cast ends at max_range
    double d = 0.0;
    if (idx < 0 || idx >= n) {
      verdict = 2;  // past the row's last candidate
    } else {
      const double vv = (double)__ldg(v + idx);
      d = q.forward ? vv - q.xq : q.xq - vv;
      int32_t cell;
      if (d >= c.max_range) {
        verdict = 2;
      } else if (landing_hit(c, x + d * dir.x, y + d * dir.y, &cell)
#if RL_PROBE_SENSOR
                 || window_probe_hit(c, x, y, dir.x, dir.y, d)
#endif
      ) {
        verdict = 1;
      } else {
        Walker<true> wk;
        wk.init_at(x, y, dir, d - kVerifyHalf);
        const double r = wk.scan_to(c, d + kVerifyHalf);
        verdict = r == kWalkExit ? 2 : (r >= 0.0 ? 1 : 0);
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, verdict != 0);
    if (m) {
      const int first = __ffs(m) - 1;
      const int vf = __shfl_sync(0xffffffffu, verdict, first);
      const double df = __shfl_sync(0xffffffffu, d, first);
      return vf == 1 ? df : c.max_range;
    }
  }
}

}  // namespace rl
