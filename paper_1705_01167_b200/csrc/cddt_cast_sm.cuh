// Batched CDDT queries as a per-lane state machine.
//
// Cddt::directional_cast (proj/src/cddt.cpp:207-269) is a chain of dependent
// gathers with data-dependent trip counts: an optional near-field grid walk,
// a row search, a candidate loop, and per candidate an optional verification
// walk (RayWalker::seek + scan_to, ray_walker.hpp:36-59). Written as nested
// loops, a warp waits at every loop exit for its slowest lane and runs the
// walker with ~3 of 32 lanes active (profiles/r01/ncu_k_cast_v1.txt).
//
// Here every lane owns a stream of queries (grid-stride) and one loop
// iteration advances each lane by one step of whatever phase it is in:
//   NEW  -> fetch the next query, origin checks, projection
//   ROW  -> row offsets + search for the first candidate
//   CAND -> next candidate: range cut-off, landing probe, walker seek
//   WALK -> one cell of scan_to (bounds, occupancy, window limit, advance)
// A lane that finishes a query starts the next one immediately instead of
// idling until the warp's slowest query ends, and all lanes that are walking
// step together. The arithmetic and the order of decisions per query are
// exactly the reference's, so results stay bit-identical.
#pragma once

#include "cddt_device.cuh"

namespace rl {

enum : int { PH_NEW = 0, PH_ROW = 1, PH_CAND = 2, PH_WALK = 3, PH_EXIT = 4 };
enum : int { WM_NEAR = 0, WM_WINDOW = 1 };

// RayWalker state without the origin/direction copies (those live in the
// per-query registers x, y, dx, dy): t, next x/y boundary parameters, cell.
struct WalkState {
  double t, tnx, tny;
  int cx, cy;
  __device__ __forceinline__ void place(double x, double y, double dx, double dy, double rx,
                                        double ry, double tt) {
    t = tt;  // ray_walker.hpp:62-73
    const double px = x + tt * dx, py = y + tt * dy;
    const Floor fx = floor2(px), fy = floor2(py);
    cx = fx.i;
    cy = fy.i;
    if (dx < 0 && px == fx.d) cx--;
    if (dy < 0 && py == fy.d) cy--;
    tnx = boundary_t(dx, x, cx, rx);
    tny = boundary_t(dy, y, cy, ry);
  }
  __device__ __forceinline__ void advance(double x, double y, double dx, double dy, double rx,
                                          double ry) {
    if (tnx == tny) {  // ray_walker.hpp:81-97
      t = tnx;
      cx += dx > 0 ? 1 : -1;
      cy += dy > 0 ? 1 : -1;
      tnx = boundary_t(dx, x, cx, rx);
      tny = boundary_t(dy, y, cy, ry);
    } else if (tnx < tny) {
      t = tnx;
      cx += dx > 0 ? 1 : -1;
      tnx = boundary_t(dx, x, cx, rx);
    } else {
      t = tny;
      cy += dy > 0 ? 1 : -1;
      tny = boundary_t(dy, y, cy, ry);
    }
  }
};

template <class T, bool HIT, bool RES>
__device__ __forceinline__ void cast_stream(const CddtView& c, const T* __restrict__ qx,
                                            const T* __restrict__ qy, const T* __restrict__ qt,
                                            T* __restrict__ out, int32_t* __restrict__ hit,
                                            int64_t* __restrict__ res_row,
                                            int32_t* __restrict__ res_idx, size_t i0,
                                            size_t stride, size_t n) {
  size_t i = i0;
  int phase = i < n ? PH_NEW : PH_EXIT;
  // per-query state
  double x = 0, y = 0, dx = 0, dy = 0, rx = 0, ry = 0, xq = 0, dcur = 0, result = 0, lim = 0;
  bool forward = true, have_walker = false, resolved = false;
  int wmode = WM_NEAR, idx = 0, n_row = 0;
  uint32_t lo = 0, g = 0;
  int32_t hcell = -1;
  WalkState wk;
  wk.t = wk.tnx = wk.tny = 0;
  wk.cx = wk.cy = 0;
  OccCache oc;
  const double gw = (double)c.w, gh = (double)c.h;

  while (phase != PH_EXIT) {
    bool done = false;
    if (phase == PH_NEW) {
      x = double(__ldcs(qx + i));
      y = double(__ldcs(qy + i));
      const double th = normalize_angle_2pi(double(__ldcs(qt + i)));  // raycast.hpp:47
      const int a = direction_index(th, c.K);
      hcell = -1;
      resolved = false;
      result = c.max_range;
      have_walker = false;
      oc.tile = -1;
      const int cxi = (int)floor(x), cyi = (int)floor(y);
      if (!in_bounds(c, cxi, cyi)) {  // cddt.cpp:209
        done = true;
      } else {
        const uint8_t f0 = __ldg(c.flags + (size_t)cyi * c.w + cxi);
        if (f0 & kOcc) {  // cddt.cpp:210
          result = 0.0;
          hcell = cyi * c.w + cxi;
          done = true;
        } else {
          forward = a < c.S;
          const int s = forward ? a : a - c.S;
          const SliceParam sp = c.slices[s];
          const double4 dir = c.dirs[a];
          dx = dir.x;
          dy = dir.y;
          rx = dir.z;
          ry = dir.w;
          xq = x * sp.cos_t + y * sp.sin_t;                              // cddt.hpp:31
          const double yq = -x * sp.sin_t + y * sp.cos_t + sp.y_offset;  // cddt.hpp:32
          int row = (int)yq;
          if (row < 0) row = 0;
          if (row >= sp.bin_count) row = sp.bin_count - 1;
          g = sp.row_base + (uint32_t)row;
          if (!(f0 & kClear)) {
            // near field resolved exactly by the walker (cddt.cpp:225-232)
            wk.place(x, y, dx, dy, rx, ry, 0.0);
            have_walker = true;
            lim = kNearField;
            wmode = WM_NEAR;
            phase = PH_WALK;
          } else {
            phase = PH_ROW;
          }
        }
      }
    }
    if (phase == PH_ROW && !done) {
      lo = __ldg(c.row_off + g);
      const uint32_t hi = __ldg(c.row_off + g + 1);
      n_row = (int)(hi - lo);
      const uint32_t first = partition_point(c.zp + lo, hi - lo, xq, forward);
      idx = forward ? (int)first : (int)first - 1;
      phase = PH_CAND;
    }
    if (phase == PH_CAND && !done) {
      // consider(v, idx) (cddt.cpp:236-262) up to the verification walk
      if (idx < 0 || idx >= n_row) {
        done = true;
      } else {
        const double vv = (double)__ldg(c.zp + lo + idx);
        dcur = forward ? vv - xq : xq - vv;
        if (dcur >= c.max_range) {
          done = true;
        } else {
          const double px = x + dcur * dx, py = y + dcur * dy;
          bool landed = false;
          if (px >= 0.0 && py >= 0.0 && px < gw && py < gh) {
            const int hx = (int)px, hy = (int)py;
            const double fx = px - (double)hx, fy = py - (double)hy;
            if (fx > kLatticeEps && fx < 1.0 - kLatticeEps && fy > kLatticeEps &&
                fy < 1.0 - kLatticeEps && oc.occ(c, hx, hy)) {
              hcell = hy * c.w + hx;
              landed = true;
            }
          }
          if (landed) {
            result = dcur;
            resolved = true;
            done = true;
          } else {
            // walker.emplace (place(0)) then seek(d - kVerifyHalf): place() resets
            // the whole state, so a fresh walker is placed once, at the later t
            const double t0 = dcur - kVerifyHalf;
            if (!have_walker) {
              wk.place(x, y, dx, dy, rx, ry, t0 > 0.0 ? t0 : 0.0);
              have_walker = true;
            } else if (t0 > wk.t) {
              wk.place(x, y, dx, dy, rx, ry, t0);
            }
            lim = dcur + kVerifyHalf;
            wmode = WM_WINDOW;
            phase = PH_WALK;
          }
        }
      }
    }
    if (phase == PH_WALK && !done) {
      // one iteration of RayWalker::scan_to (ray_walker.hpp:51-59)
      int outcome = 0;  // 0 continue, 1 hit, 2 window exhausted, 3 left the grid
      if (!in_bounds(c, wk.cx, wk.cy)) {
        outcome = 3;
      } else if (oc.occ(c, wk.cx, wk.cy)) {
        outcome = 1;
      } else {
        const double tn = wk.tnx < wk.tny ? wk.tnx : wk.tny;
        if (tn > lim)
          outcome = 2;
        else
          wk.advance(x, y, dx, dy, rx, ry);
      }
      if (outcome == 1) {
        hcell = wk.cy * c.w + wk.cx;
        if (wmode == WM_NEAR) {
          result = (c.max_range < wk.t) ? c.max_range : wk.t;
        } else {
          result = dcur;
          resolved = true;
        }
        done = true;
      } else if (outcome == 3) {
        done = true;  // result stays max_range
      } else if (outcome == 2) {
        if (wmode == WM_NEAR) {
          phase = PH_ROW;
        } else {
          idx += forward ? 1 : -1;
          phase = PH_CAND;
        }
      }
    }
    if (done) {
      if (out) __stcs(out + i, T(result));
      if (HIT) hit[i] = hcell;
      if (RES) {
        res_row[i] = resolved ? int64_t(g) : -1;
        res_idx[i] = resolved ? idx : -1;
      }
      i += stride;
      phase = i < n ? PH_NEW : PH_EXIT;
    }
  }
}

}  // namespace rl
