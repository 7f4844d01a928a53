/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, CPU restatement of the reference rangelib CDDT path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. Nothing in the product path (paper_1705_01167_b200/) may link,
 * import or call this file.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to the reference tree, proj/...). Compiled with -O2 -ffp-contract=off so
 * the FP64 expression order and rounding match the reference built without
 * FMA contraction.
 *
 * Parity of this restatement is pinned against the unmodified reference
 * compiled from its own sources into oracle/_ref/ (oracle/Makefile) and
 * against the golden vectors in tests/golden/ (tests/test_oracle_golden.py).
 *
 * Beyond the reference it reports, per query, the hit cell, the resolving
 * (row, index) and the number of distinct 32-byte sectors the query touches
 * under the device layout.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define K_TWO_PI 6.283185307179586476925286766559 /* raycast.hpp:12 */
#define K_NEAR_FIELD 0.75                         /* cddt.cpp:19 */
#define K_VERIFY_HALF 0.7072                      /* cddt.cpp:25 */
#define K_LATTICE_EPS 1e-9                        /* cddt.cpp:26 */
#define W_NONE (-1.0)                             /* ray_walker.hpp:23 */
#define W_EXIT (-2.0)                             /* ray_walker.hpp:24 */

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ELOGIC = 2, ORC_ERANGE = 3, ORC_ENOMEM = 5 };

/* ---- angle helpers: proj/include/rangelib/raycast.hpp:17-40 ---- */
static inline long orc_iround(double v) { return (long)ceil(v - 0.5); }

double orc_normalize_angle_2pi(double t) {
  t = fmod(t, K_TWO_PI);
  if (t < 0) t += K_TWO_PI;
  if (t >= K_TWO_PI) t = 0.0;
  return t;
}

int orc_direction_index(double theta, int K) {
  long i = orc_iround(theta * (double)K / K_TWO_PI) % K;
  if (i < 0) i += K;
  return (int)i;
}

/* proj/src/cddt.cpp:30-42 */
void orc_direction_components(int i, int K, double *c, double *s) {
  long long q4 = 4LL * i;
  if (q4 % K == 0) {
    int q = (int)(q4 / K) & 3;
    *c = (q == 0) ? 1.0 : (q == 2) ? -1.0 : 0.0;
    *s = (q == 1) ? 1.0 : (q == 3) ? -1.0 : 0.0;
  } else {
    double t = (double)i * K_TWO_PI / (double)K;
    *c = cos(t);
    *s = sin(t);
  }
}

static inline double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static inline double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* ---- structure ---- */
typedef struct {
  float *v;
  uint32_t n, cap;
} orc_row;

typedef struct {
  int w, h, K, S, pruned;
  double max_range, resolution;
  uint8_t *occ, *member, *clear;
  double *dcos, *dsin; /* K */
  double *yoff;        /* S */
  int *nbins;          /* S */
  size_t *row_base;    /* S+1, global row index of (s, 0) */
  orc_row *rows;
  size_t zero_points;
  uint64_t *zoff; /* CSR offsets cache, only for sector accounting */
} orc_cddt;

static inline double proj_x(const orc_cddt *c, int s, double x, double y) {
  return x * c->dcos[s] + y * c->dsin[s]; /* cddt.hpp:31 */
}
static inline double proj_y(const orc_cddt *c, int s, double x, double y) {
  return -x * c->dsin[s] + y * c->dcos[s] + c->yoff[s]; /* cddt.hpp:32 */
}

static int row_push(orc_row *r, float v) {
  if (r->n == r->cap) {
    uint32_t cap = r->cap ? r->cap * 2 : 4;
    float *nv = realloc(r->v, sizeof(float) * cap);
    if (!nv) return ORC_ENOMEM;
    r->v = nv;
    r->cap = cap;
  }
  r->v[r->n++] = v;
  return ORC_OK;
}
static int cmp_f32(const void *a, const void *b) {
  float x = *(const float *)a, y = *(const float *)b;
  return (x < y) ? -1 : (y < x) ? 1 : 0;
}
/* first index with v[i] >= q (float compare), cddt.hpp:69,75 */
static uint32_t lb_f32(const orc_row *r, float q) {
  uint32_t first = 0, len = r->n;
  while (len > 0) {
    uint32_t half = len >> 1, mid = first + half;
    if (r->v[mid] < q) {
      first = mid + 1;
      len -= half + 1;
    } else
      len = half;
  }
  return first;
}
/* ZeroPointBin::insert, cddt.hpp:67-72: insert at lower_bound */
static int row_insert(orc_row *r, float v) {
  uint32_t pos = lb_f32(r, v);
  int st = row_push(r, v);
  if (st) return st;
  memmove(r->v + pos + 1, r->v + pos, sizeof(float) * (r->n - 1 - pos));
  r->v[pos] = v;
  return ORC_OK;
}
/* ZeroPointBin::remove_one, cddt.hpp:73-79 */
static int row_remove_one(orc_row *r, float v) {
  uint32_t pos = lb_f32(r, v);
  if (pos == r->n || r->v[pos] != v) return 0;
  memmove(r->v + pos, r->v + pos + 1, sizeof(float) * (r->n - pos - 1));
  r->n--;
  return 1;
}

static inline int in_bounds(const orc_cddt *c, int x, int y) {
  return x >= 0 && x < c->w && y >= 0 && y < c->h;
}
static inline int at(const orc_cddt *c, int x, int y) { return c->occ[(size_t)y * c->w + x] != 0; }

/* is_edge_cell, proj/src/grid.cpp:110-119 */
static int is_edge(const orc_cddt *c, int x, int y) {
  if (!at(c, x, y)) return 0;
  for (int dy = -1; dy <= 1; dy++)
    for (int dx = -1; dx <= 1; dx++) {
      if (dx == 0 && dy == 0) continue;
      int nx = x + dx, ny = y + dy;
      if (!in_bounds(c, nx, ny) || !at(c, nx, ny)) return 1;
    }
  return 0;
}

/* clear_around / rebuild_clear_mask, proj/src/cddt.cpp:173-190 */
static void rebuild_clear(orc_cddt *c, int x0, int y0, int x1, int y1) {
  if (x0 < 0) x0 = 0;
  if (y0 < 0) y0 = 0;
  if (x1 > c->w - 1) x1 = c->w - 1;
  if (y1 > c->h - 1) y1 = c->h - 1;
  for (int y = y0; y <= y1; y++)
    for (int x = x0; x <= x1; x++) {
      int clr = 1;
      for (int dy = -1; dy <= 1 && clr; dy++)
        for (int dx = -1; dx <= 1; dx++) {
          int nx = x + dx, ny = y + dy;
          if (in_bounds(c, nx, ny) && at(c, nx, ny)) {
            clr = 0;
            break;
          }
        }
      c->clear[(size_t)y * c->w + x] = (uint8_t)clr;
    }
}

/* for_each_bin_of_pixel, proj/src/cddt.cpp:118-134: rows [r0, r1] and the
 * stored value of pixel (px, py) in slice s */
static void pixel_rows(const orc_cddt *c, int s, int px, int py, int *r0o, int *r1o, float *vo) {
  double c0 = proj_y(c, s, px, py);
  double c1 = proj_y(c, s, px + 1, py);
  double c2 = proj_y(c, s, px, py + 1);
  double c3 = proj_y(c, s, px + 1, py + 1);
  double lo = dmin(dmin(c0, c1), dmin(c2, c3));
  double hi = dmax(dmax(c0, c1), dmax(c2, c3));
  int r0 = (int)floor(lo);
  int r1 = (int)ceil(hi) - 1;
  if (r0 < 0) r0 = 0;
  if (r1 >= c->nbins[s]) r1 = c->nbins[s] - 1;
  *r0o = r0;
  *r1o = r1;
  *vo = (float)proj_x(c, s, px + 0.5, py + 0.5);
}

static int add_pixel_points(orc_cddt *c, int px, int py, int sorted_insert) {
  for (int s = 0; s < c->S; s++) {
    int r0, r1;
    float v;
    pixel_rows(c, s, px, py, &r0, &r1, &v);
    for (int r = r0; r <= r1; r++) {
      orc_row *row = &c->rows[c->row_base[s] + r];
      int st = sorted_insert ? row_insert(row, v) : row_push(row, v);
      if (st) return st;
      c->zero_points++;
    }
  }
  return ORC_OK;
}
static void remove_pixel_points(orc_cddt *c, int px, int py) {
  for (int s = 0; s < c->S; s++) {
    int r0, r1;
    float v;
    pixel_rows(c, s, px, py, &r0, &r1, &v);
    for (int r = r0; r <= r1; r++)
      if (row_remove_one(&c->rows[c->row_base[s] + r], v)) c->zero_points--;
  }
}

void orc_cddt_destroy(orc_cddt *c) {
  if (!c) return;
  if (c->rows)
    for (size_t i = 0; i < c->row_base[c->S]; i++) free(c->rows[i].v);
  free(c->rows);
  free(c->zoff);
  free(c->occ);
  free(c->member);
  free(c->clear);
  free(c->dcos);
  free(c->dsin);
  free(c->yoff);
  free(c->nbins);
  free(c->row_base);
  free(c);
}

/* geometry + empty rows (Cddt::Cddt prologue, proj/src/cddt.cpp:136-153;
 * RangeMethodConfig::validate / resolved_max_range, raycast.hpp:55-63;
 * SliceProjection::make, cddt.cpp:44-60) */
static int cddt_alloc(const uint8_t *grid, int w, int h, double resolution, int K,
                      double max_range, orc_cddt **out) {
  *out = NULL;
  if (w <= 0 || h <= 0 || !(resolution > 0.0)) return ORC_EINVAL;
  if (max_range < 0.0) return ORC_EINVAL;
  if (K < 4 || K % 2 != 0) return ORC_EINVAL;
  orc_cddt *c = calloc(1, sizeof(orc_cddt));
  if (!c) return ORC_ENOMEM;
  c->w = w;
  c->h = h;
  c->K = K;
  c->S = K / 2;
  c->resolution = resolution;
  c->max_range = max_range > 0.0 ? max_range : sqrt((double)w * w + (double)h * h);
  size_t wh = (size_t)w * h;
  c->occ = malloc(wh);
  c->member = calloc(wh, 1);
  c->clear = calloc(wh, 1);
  c->dcos = malloc(sizeof(double) * K);
  c->dsin = malloc(sizeof(double) * K);
  c->yoff = malloc(sizeof(double) * c->S);
  c->nbins = malloc(sizeof(int) * c->S);
  c->row_base = malloc(sizeof(size_t) * (c->S + 1));
  if (!c->occ || !c->member || !c->clear || !c->dcos || !c->dsin || !c->yoff || !c->nbins ||
      !c->row_base) {
    orc_cddt_destroy(c);
    return ORC_ENOMEM;
  }
  for (size_t i = 0; i < wh; i++) c->occ[i] = grid[i] ? 1 : 0;
  for (int a = 0; a < K; a++) orc_direction_components(a, K, &c->dcos[a], &c->dsin[a]);
  size_t base = 0;
  for (int s = 0; s < c->S; s++) {
    double sn = c->dsin[s], cs = c->dcos[s];
    double A = 0.0, B = -(double)w * sn, C = (double)h * cs, D = B + C;
    double lo = dmin(dmin(A, B), dmin(C, D)), hi = dmax(dmax(A, B), dmax(C, D));
    c->yoff[s] = -lo;
    c->nbins[s] = (int)ceil(hi - lo) + 1;
    c->row_base[s] = base;
    base += (size_t)c->nbins[s];
  }
  c->row_base[c->S] = base;
  c->rows = calloc(base ? base : 1, sizeof(orc_row));
  if (!c->rows) {
    orc_cddt_destroy(c);
    return ORC_ENOMEM;
  }
  *out = c;
  return ORC_OK;
}

/* Cddt::Cddt, proj/src/cddt.cpp:136-171 */
int orc_cddt_create(const uint8_t *grid, int w, int h, double resolution, int K, double max_range,
                    orc_cddt **out) {
  orc_cddt *c;
  int st = cddt_alloc(grid, w, h, resolution, K, max_range, &c);
  if (st) return st;
  size_t base = c->row_base[c->S];
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++)
      if (is_edge(c, x, y)) {
        c->member[(size_t)y * w + x] = 1;
        if (add_pixel_points(c, x, y, 0)) {
          orc_cddt_destroy(c);
          return ORC_ENOMEM;
        }
      }
  for (size_t r = 0; r < base; r++)
    if (c->rows[r].n > 1) qsort(c->rows[r].v, c->rows[r].n, sizeof(float), cmp_f32);
  rebuild_clear(c, 0, 0, w - 1, h - 1);
  *out = c;
  return ORC_OK;
}

/* Load bins from a CSR export (as deserialize_cddt loads bins from a
 * snapshot, cddt.cpp:502-579): used to run the restatement on a structure
 * produced elsewhere, e.g. a GPU-pruned PCDDT. */
int orc_cddt_load(const uint8_t *grid, int w, int h, double resolution, int K, double max_range,
                  const uint64_t *row_off, const float *zp, const uint8_t *member, int pruned,
                  orc_cddt **out) {
  orc_cddt *c;
  int st = cddt_alloc(grid, w, h, resolution, K, max_range, &c);
  if (st) return st;
  size_t nrows = c->row_base[c->S];
  for (size_t r = 0; r < nrows; r++) {
    uint64_t a = row_off[r], b = row_off[r + 1];
    orc_row *row = &c->rows[r];
    row->n = row->cap = (uint32_t)(b - a);
    if (row->n) {
      row->v = malloc(sizeof(float) * row->n);
      if (!row->v) {
        orc_cddt_destroy(c);
        return ORC_ENOMEM;
      }
      memcpy(row->v, zp + a, sizeof(float) * row->n);
    }
    c->zero_points += row->n;
  }
  memcpy(c->member, member, (size_t)w * h);
  c->pruned = pruned;
  rebuild_clear(c, 0, 0, w - 1, h - 1);
  *out = c;
  return ORC_OK;
}

/* ---- sector accounting for the roofline (device layout: 1 flag byte per
 * cell, u32 row offsets, f32 zero points) ---- */
typedef struct {
  uint64_t s[512];
  int n;
} sector_set;
static inline void touch(sector_set *ss, int space, uint64_t byte) {
  if (!ss) return;
  uint64_t key = ((uint64_t)space << 60) | (byte >> 5);
  for (int i = 0; i < ss->n; i++)
    if (ss->s[i] == key) return;
  if (ss->n < 512) ss->s[ss->n++] = key;
}

/* ---- optional work counters (single-threaded profiling of the algorithm) ---- */
static long g_stats[8];
void orc_stats_reset(void) { memset(g_stats, 0, sizeof g_stats); }
void orc_stats_get(long *out) { memcpy(out, g_stats, sizeof g_stats); }
enum { ST_QUERIES, ST_NEAR, ST_WALK_STEPS, ST_CANDS, ST_LAND_HIT, ST_WINDOWS, ST_PLACES, ST_SEARCH };

/* ---- RayWalker, proj/include/rangelib/detail/ray_walker.hpp:21-104 ---- */
typedef struct {
  const orc_cddt *c;
  double ox, oy, dx, dy, t, tnx, tny;
  int cx, cy;
  sector_set *ss;
} walker;

static inline double boundary_t(double d, double o, int c) {
  if (d > 0) return ((double)c + 1.0 - o) / d;
  if (d < 0) return ((double)c - o) / d;
  return INFINITY;
}
static void w_place(walker *w, double t) {
  g_stats[ST_PLACES]++;
  w->t = t;
  double px = w->ox + t * w->dx, py = w->oy + t * w->dy;
  w->cx = (int)floor(px);
  w->cy = (int)floor(py);
  if (w->dx < 0 && px == (double)w->cx) w->cx--;
  if (w->dy < 0 && py == (double)w->cy) w->cy--;
  w->tnx = boundary_t(w->dx, w->ox, w->cx);
  w->tny = boundary_t(w->dy, w->oy, w->cy);
}
static void w_init(walker *w, const orc_cddt *c, double ox, double oy, double dx, double dy,
                   sector_set *ss) {
  w->c = c;
  w->ox = ox;
  w->oy = oy;
  w->dx = dx;
  w->dy = dy;
  w->ss = ss;
  w_place(w, 0.0);
}
static inline void w_seek(walker *w, double t) {
  if (t > w->t) w_place(w, t);
}
static void w_advance(walker *w) {
  if (w->tnx == w->tny) {
    w->t = w->tnx;
    w->cx += w->dx > 0 ? 1 : -1;
    w->cy += w->dy > 0 ? 1 : -1;
    w->tnx = boundary_t(w->dx, w->ox, w->cx);
    w->tny = boundary_t(w->dy, w->oy, w->cy);
  } else if (w->tnx < w->tny) {
    w->t = w->tnx;
    w->cx += w->dx > 0 ? 1 : -1;
    w->tnx = boundary_t(w->dx, w->ox, w->cx);
  } else {
    w->t = w->tny;
    w->cy += w->dy > 0 ? 1 : -1;
    w->tny = boundary_t(w->dy, w->oy, w->cy);
  }
}
static double w_scan_to(walker *w, double lim) {
  for (;;) {
    if (!in_bounds(w->c, w->cx, w->cy)) return W_EXIT;
    touch(w->ss, 0, (uint64_t)w->cy * w->c->w + w->cx);
    if (at(w->c, w->cx, w->cy)) return w->t;
    double tn = w->tnx < w->tny ? w->tnx : w->tny;
    if (tn > lim) return W_NONE;
    g_stats[ST_WALK_STEPS]++;
    w_advance(w);
  }
}

/* Cddt::directional_cast, proj/src/cddt.cpp:207-269 (visit_above/visit_below
 * cddt.hpp:106-131). Outputs beyond the reference:
 *   hit       : occupied cell index (y*w+x) that settled the answer, or -1
 *   res_row   : global row index of the resolving zero point, or -1
 *   res_idx   : its sorted position within the row, or -1
 *   sectors   : distinct 32-byte sectors touched (device layout), or NULL */
double orc_directional_cast(const orc_cddt *c, double x, double y, int a, int32_t *hit,
                            int64_t *res_row, int32_t *res_idx, int *sectors) {
  sector_set ssv, *ss = sectors ? &ssv : NULL;
  if (ss) ss->n = 0;
  g_stats[ST_QUERIES]++;
  int32_t h_ = -1;
  int64_t rr = -1;
  int32_t ri = -1;
  double result;
  const int cxi = (int)floor(x), cyi = (int)floor(y);
  if (!in_bounds(c, cxi, cyi)) {
    result = c->max_range;
    goto done;
  }
  touch(ss, 0, (uint64_t)cyi * c->w + cxi);
  if (at(c, cxi, cyi)) {
    result = 0.0;
    h_ = cyi * c->w + cxi;
    goto done;
  }
  {
    const int S = c->S;
    const int forward = a < S;
    const int s = forward ? a : a - S;
    const double xq = proj_x(c, s, x, y);
    const double yq = proj_y(c, s, x, y);
    int row = (int)yq;
    if (row < 0) row = 0;
    if (row >= c->nbins[s]) row = c->nbins[s] - 1;
    const double dx = c->dcos[a], dy = c->dsin[a];
    walker wk;
    int have_walker = 0;
    if (!c->clear[(size_t)cyi * c->w + cxi]) {
      g_stats[ST_NEAR]++;
      w_init(&wk, c, x, y, dx, dy, ss);
      have_walker = 1;
      double r = w_scan_to(&wk, K_NEAR_FIELD);
      if (r >= 0.0) {
        result = dmin(r, c->max_range);
        h_ = wk.cy * c->w + wk.cx;
        goto done;
      }
      if (r == W_EXIT) {
        result = c->max_range;
        goto done;
      }
    }
    result = c->max_range;
    const double gw = (double)c->w, gh = (double)c->h;
    const size_t grow = c->row_base[s] + (size_t)row;
    const orc_row *bin = &c->rows[grow];
    touch(ss, 1, grow * 4);
    touch(ss, 1, grow * 4 + 4);
    /* CSR position of this row's first point, for zp sector accounting */
    uint64_t zbase = (ss && c->zoff) ? c->zoff[grow] : 0;
    /* upper_bound (forward) / lower_bound (backward) over double(v) vs xq */
    uint32_t first = 0, len = bin->n;
    while (len > 0) {
      uint32_t half = len >> 1, mid = first + half;
      touch(ss, 2, (zbase + mid) * 4);
      int go_right = forward ? !(xq < (double)bin->v[mid]) : ((double)bin->v[mid] < xq);
      if (go_right) {
        first = mid + 1;
        len -= half + 1;
      } else
        len = half;
    }
    long idx = forward ? (long)first : (long)first - 1;
    long step = forward ? 1 : -1;
    g_stats[ST_SEARCH] += bin->n;
    for (; idx >= 0 && idx < (long)bin->n; idx += step) {
      g_stats[ST_CANDS]++;
      touch(ss, 2, (zbase + (uint64_t)idx) * 4);
      double v = (double)bin->v[idx];
      double d = forward ? v - xq : xq - v;
      if (d >= c->max_range) break;
      const double px = x + d * dx, py = y + d * dy;
      if (px >= 0.0 && py >= 0.0 && px < gw && py < gh) {
        const int hx = (int)px, hy = (int)py;
        const double fx = px - (double)hx, fy = py - (double)hy;
        if (fx > K_LATTICE_EPS && fx < 1.0 - K_LATTICE_EPS && fy > K_LATTICE_EPS &&
            fy < 1.0 - K_LATTICE_EPS) {
          touch(ss, 0, (uint64_t)hy * c->w + hx);
          if (at(c, hx, hy)) {
            g_stats[ST_LAND_HIT]++;
            rr = (int64_t)grow;
            ri = (int32_t)idx;
            result = d;
            h_ = hy * c->w + hx;
            break;
          }
        }
      }
      if (!have_walker) {
        w_init(&wk, c, x, y, dx, dy, ss);
        have_walker = 1;
      }
      g_stats[ST_WINDOWS]++;
      w_seek(&wk, d - K_VERIFY_HALF);
      double r = w_scan_to(&wk, d + K_VERIFY_HALF);
      if (r == W_EXIT) break;
      if (r < 0.0) continue;
      rr = (int64_t)grow;
      ri = (int32_t)idx;
      result = d;
      h_ = wk.cy * c->w + wk.cx;
      break;
    }
  }
done:
  if (hit) *hit = h_;
  if (res_row) *res_row = rr;
  if (res_idx) *res_idx = ri;
  if (sectors) *sectors = ss->n;
  return result;
}

/* Cddt::cast, proj/src/cddt.cpp:271-273 (RayQuery normalises, raycast.hpp:47) */
double orc_cast(const orc_cddt *c, double x, double y, double theta) {
  return orc_directional_cast(c, x, y, orc_direction_index(orc_normalize_angle_2pi(theta), c->K),
                              NULL, NULL, NULL, NULL);
}

/* Batched f32 casts (the loop body of run_batches, proj/src/bench.cpp:86-106,
 * over a query array); optional f64 ranges, hit cells, resolving index and
 * sector counts. Parallel over queries with OpenMP when nthreads > 1. */
void orc_cast_batch(const orc_cddt *c, const float *qx, const float *qy, const float *qt,
                    size_t n, float *out32, double *out64, int32_t *hit, int64_t *res_row,
                    int32_t *res_idx, int32_t *sectors, int nthreads) {
  if (sectors) {
    orc_cddt *mc = (orc_cddt *)c;
    size_t nrows = c->row_base[c->S];
    free(mc->zoff);
    mc->zoff = malloc(sizeof(uint64_t) * (nrows + 1));
    uint64_t off = 0;
    for (size_t r = 0; r < nrows; r++) {
      mc->zoff[r] = off;
      off += c->rows[r].n;
    }
    mc->zoff[nrows] = off;
  }
#pragma omp parallel for schedule(dynamic, 1024) num_threads(nthreads > 0 ? nthreads : 1)
  for (size_t i = 0; i < n; i++) {
    double x = (double)qx[i], y = (double)qy[i];
    double th = orc_normalize_angle_2pi((double)qt[i]);
    int a = orc_direction_index(th, c->K);
    int sec = 0;
    double r = orc_directional_cast(c, x, y, a, hit ? &hit[i] : NULL,
                                    res_row ? &res_row[i] : NULL, res_idx ? &res_idx[i] : NULL,
                                    sectors ? &sec : NULL);
    if (out32) out32[i] = (float)r;
    if (out64) out64[i] = r;
    if (sectors) sectors[i] = sec;
  }
}

/* Cddt::prune, proj/src/cddt.cpp:281-330: mark the resolving index and its
 * near-side neighbour for every free cell centre x every direction, keep
 * marked points. */
int orc_prune(orc_cddt *c, int nthreads) {
  if (c->pruned) return ORC_OK;
  size_t nrows = c->row_base[c->S];
  uint8_t **marks = calloc(nrows, sizeof(uint8_t *));
  if (!marks) return ORC_ENOMEM;
  for (size_t r = 0; r < nrows; r++) {
    marks[r] = calloc(c->rows[r].n ? c->rows[r].n : 1, 1);
    if (!marks[r]) return ORC_ENOMEM;
  }
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int cy = 0; cy < c->h; cy++)
    for (int cx = 0; cx < c->w; cx++) {
      if (at(c, cx, cy)) continue;
      const double px = cx + 0.5, py = cy + 0.5;
      for (int a = 0; a < c->K; a++) {
        int64_t rr;
        int32_t ri;
        orc_directional_cast(c, px, py, a, NULL, &rr, &ri, NULL);
        if (rr < 0) continue;
        uint8_t *rb = marks[rr];
        __atomic_store_n(&rb[ri], 1, __ATOMIC_RELAXED);
        if (a < c->S) {
          if (ri > 0) __atomic_store_n(&rb[ri - 1], 1, __ATOMIC_RELAXED);
        } else {
          if ((uint32_t)ri + 1 < c->rows[rr].n) __atomic_store_n(&rb[ri + 1], 1, __ATOMIC_RELAXED);
        }
      }
    }
  c->zero_points = 0;
  for (size_t r = 0; r < nrows; r++) {
    orc_row *row = &c->rows[r];
    uint32_t k = 0;
    for (uint32_t i = 0; i < row->n; i++)
      if (marks[r][i]) row->v[k++] = row->v[i];
    row->n = k;
    c->zero_points += k;
    free(marks[r]);
  }
  free(marks);
  c->pruned = 1;
  return ORC_OK;
}

/* Cddt::set_occupancy, proj/src/cddt.cpp:332-377 */
int orc_set_occupancy(orc_cddt *c, int x, int y, int occupied) {
  if (c->pruned) return ORC_ELOGIC;
  if (!in_bounds(c, x, y)) return ORC_ERANGE;
  occupied = occupied != 0;
  if (at(c, x, y) == occupied) return ORC_OK;
  const int w = c->w;
  const size_t idx = (size_t)y * w + x;
  c->occ[idx] = (uint8_t)occupied;
  if (occupied) {
    if (is_edge(c, x, y)) {
      c->member[idx] = 1;
      if (add_pixel_points(c, x, y, 1)) return ORC_ENOMEM;
    }
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        if (dx == 0 && dy == 0) continue;
        int nx = x + dx, ny = y + dy;
        if (!in_bounds(c, nx, ny)) continue;
        size_t n = (size_t)ny * w + nx;
        if (c->member[n] && !is_edge(c, nx, ny)) {
          c->member[n] = 0;
          remove_pixel_points(c, nx, ny);
        }
      }
  } else {
    if (c->member[idx]) {
      c->member[idx] = 0;
      remove_pixel_points(c, x, y);
    }
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        if (dx == 0 && dy == 0) continue;
        int nx = x + dx, ny = y + dy;
        if (!in_bounds(c, nx, ny)) continue;
        size_t n = (size_t)ny * w + nx;
        if (at(c, nx, ny) && !c->member[n]) {
          c->member[n] = 1;
          if (add_pixel_points(c, nx, ny, 1)) return ORC_ENOMEM;
        }
      }
  }
  rebuild_clear(c, x - 1, y - 1, x + 1, y + 1);
  return ORC_OK;
}

/* ---- structure export (concatenation of Cddt::bin(s,r).values() in
 * (slice,row) order) ---- */
void orc_cddt_info(const orc_cddt *c, int64_t *out) {
  out[0] = c->w;
  out[1] = c->h;
  out[2] = c->K;
  out[3] = c->S;
  out[4] = (int64_t)c->row_base[c->S];
  out[5] = (int64_t)c->zero_points;
  out[6] = c->pruned;
  /* Cddt::memory_bytes, cddt.hpp:200-203 */
  out[7] = (int64_t)(4 * c->zero_points + ((size_t)c->w * c->h + 7) / 8 + (size_t)c->S * 48);
}
double orc_cddt_max_range(const orc_cddt *c) { return c->max_range; }

void orc_cddt_export(const orc_cddt *c, uint32_t *slice_row_base, uint64_t *row_off, float *zp,
                     uint8_t *member, uint8_t *clear, double *yoff, int32_t *nbins) {
  if (slice_row_base)
    for (int s = 0; s <= c->S; s++) slice_row_base[s] = (uint32_t)c->row_base[s];
  size_t nrows = c->row_base[c->S];
  uint64_t off = 0;
  for (size_t r = 0; r < nrows; r++) {
    if (row_off) row_off[r] = off;
    if (zp) memcpy(zp + off, c->rows[r].v, sizeof(float) * c->rows[r].n);
    off += c->rows[r].n;
  }
  if (row_off) row_off[nrows] = off;
  size_t wh = (size_t)c->w * c->h;
  if (member) memcpy(member, c->member, wh);
  if (clear) memcpy(clear, c->clear, wh);
  if (yoff) memcpy(yoff, c->yoff, sizeof(double) * c->S);
  if (nbins) memcpy(nbins, c->nbins, sizeof(int32_t) * c->S);
}
void orc_cddt_dirs(const orc_cddt *c, double *dcos, double *dsin) {
  memcpy(dcos, c->dcos, sizeof(double) * c->K);
  memcpy(dsin, c->dsin, sizeof(double) * c->K);
}
void orc_cddt_grid(const orc_cddt *c, uint8_t *grid) { memcpy(grid, c->occ, (size_t)c->w * c->h); }

/* ---- beam sensor model ---- */

/* beam_likelihood, proj/src/mcl.cpp:11-40. p = {w_hit, w_short, w_max,
 * w_rand, sigma_hit, lambda_short, z_max} */
double orc_beam_likelihood(const double *p, double expected, double measured) {
  const double zm = p[6];
  if (!(zm > 0.0)) return NAN;
  const double e = expected < 0.0 ? 0.0 : (zm < expected ? zm : expected);
  const double m = measured < 0.0 ? 0.0 : (zm < measured ? zm : measured);
  double hit = 0.0;
  if (p[0] > 0.0) {
    const double s = p[4];
    const double inv_sqrt2 = 0.7071067811865476;
    double eta = 0.5 * (erf((zm - e) / s * inv_sqrt2) - erf((0.0 - e) / s * inv_sqrt2));
    if (eta > 1e-12) {
      double z = (m - e) / s;
      hit = exp(-0.5 * z * z) / (s * 2.5066282746310002) / eta;
    }
  }
  double shrt = 0.0;
  if (p[1] > 0.0 && e > 0.0 && m <= e) {
    double denom = 1.0 - exp(-p[5] * e);
    if (denom > 1e-12) shrt = p[5] * exp(-p[5] * m) / denom;
  }
  double mx = (m >= zm - 1.0) ? 1.0 : 0.0;
  double rnd = 1.0 / zm;
  return p[0] * hit + p[1] * shrt + p[2] * mx + p[3] * rnd;
}

/* discretised likelihood table T[m][e] = float(beam_likelihood(e, m)) at
 * e, m = i / inv_res for i in [0, zdim) */
void orc_beam_table(const double *p, int zdim, double inv_res, float *table) {
  for (int m = 0; m < zdim; m++)
    for (int e = 0; e < zdim; e++)
      table[(size_t)m * zdim + e] =
          (float)orc_beam_likelihood(p, (double)e / inv_res, (double)m / inv_res);
}

static inline double beam_offset(int i, int nb, double fov) {
  if (nb <= 1) return 0.0; /* ScanSpec::beam_offset, mcl.hpp:42-51 */
  return -fov / 2.0 + fov * (double)i / (double)(nb - 1);
}
static inline int table_index(double r, double inv_res, int zdim) {
  long i = orc_iround(r * inv_res);
  if (i < 0) i = 0;
  if (i > zdim - 1) i = zdim - 1;
  return (int)i;
}

/* sensor_update, proj/src/mcl.cpp:58-120 on the unpaired path (UnpairedView,
 * proj/tests/test_mcl.cpp:21-31). table == NULL selects the analytic
 * beam_likelihood with params p; otherwise logs of the table entries are
 * summed. Writes log-weights and normalised weights; returns 1 when the
 * weights were degenerate and reset to uniform (the reference's false). */
int orc_sensor_update(const orc_cddt *c, const double *px, const double *py, const double *pt,
                      long n, const double *scan, int nb, double fov, const double *p,
                      const float *table, int zdim, double inv_res, double *logw, double *weight,
                      int nthreads) {
  if (n == 0) return 0;
  double max_lw = -INFINITY;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
  for (long i = 0; i < n; i++) {
    double lw = 0.0;
    for (int b = 0; b < nb; b++) {
      double th = orc_normalize_angle_2pi(pt[i] + beam_offset(b, nb, fov));
      double e = orc_directional_cast(c, px[i], py[i], orc_direction_index(th, c->K), NULL, NULL,
                                      NULL, NULL);
      double like;
      if (table)
        like = (double)table[(size_t)table_index(scan[b], inv_res, zdim) * zdim +
                             table_index(e, inv_res, zdim)];
      else
        like = orc_beam_likelihood(p, e, scan[b]);
      lw += log(like);
    }
    logw[i] = lw;
  }
  for (long i = 0; i < n; i++)
    if (logw[i] > max_lw) max_lw = logw[i];
  double sum = 0.0;
  for (long i = 0; i < n; i++) {
    double w = exp(logw[i] - max_lw);
    weight[i] = w;
    sum += w;
  }
  if (!(sum > 0.0) || !isfinite(sum)) {
    for (long i = 0; i < n; i++) weight[i] = 1.0 / (double)n;
    return 1;
  }
  for (long i = 0; i < n; i++) weight[i] /= sum;
  return 0;
}

/* ---- particle filter (Mcl::step, proj/src/mcl.cpp:42-56, 108-142, 176-201)
 * with the counter-based noise of the GPU path: Philox4x32-10 keyed by the
 * seed, counter (particle index, draw, iteration), Box-Muller normals. ---- */
static void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
static void philox_u2(uint64_t seed, uint32_t i, uint32_t draw, uint64_t iter, double *u0,
                      double *u1) {
  uint32_t c[4] = {i, draw, (uint32_t)iter, (uint32_t)(iter >> 32)};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t a = ((uint64_t)c[1] << 32) | c[0], b = ((uint64_t)c[3] << 32) | c[2];
  *u0 = (double)(a >> 11) * 0x1.0p-53;
  *u1 = (double)(b >> 11) * 0x1.0p-53;
}
void orc_philox(uint32_t *c4, uint32_t k0, uint32_t k1) { philox(c4, k0, k1); }

/* motion_update (mcl.cpp:42-56); noise = {a, b, c, d} of MotionNoise */
void orc_motion_update(double *x, double *y, double *t, long n, uint64_t off, double dx,
                       double dy, double dth, const double *noise, uint64_t seed, uint64_t iter) {
  const double trans = hypot(dx, dy);
  double st = noise[0] * trans + noise[1] * fabs(dth);
  double sr = noise[2] * fabs(dth) + noise[3] * trans;
  if (st < 1e-12) st = 1e-12;
  if (sr < 1e-12) sr = 1e-12;
  for (long i = 0; i < n; i++) {
    uint32_t gi = (uint32_t)(off + (uint64_t)i);
    double a0, a1, b0, b1;
    philox_u2(seed, gi, 0, iter, &a0, &a1);
    philox_u2(seed, gi, 1, iter, &b0, &b1);
    double ra = sqrt(-2.0 * log(1.0 - a0)), rb = sqrt(-2.0 * log(1.0 - b0));
    double n0 = ra * cos(K_TWO_PI * a1), n1 = ra * sin(K_TWO_PI * a1), n2 = rb * cos(K_TWO_PI * b1);
    double rdx = dx + st * n0, rdy = dy + st * n1, rdt = dth + sr * n2;
    double c = cos(t[i]), s = sin(t[i]);
    x[i] += rdx * c - rdy * s;
    y[i] += rdx * s + rdy * c;
    t[i] = orc_normalize_angle_2pi(t[i] + rdt);
  }
}

/* resample_low_variance (mcl.cpp:122-142), sequential comb; r from Philox */
void orc_resample(const double *x, const double *y, const double *t, const double *w, long n,
                  double *ox, double *oy, double *ot, double *ow, int64_t *src, uint64_t seed,
                  uint64_t iter) {
  if (n <= 0) return;
  double u, unused;
  philox_u2(seed, 0xFFFFFFFFu, 0xFFFFFFFFu, iter, &u, &unused);
  const double r = (1.0 / (double)n) * u;
  double c = w[0];
  long i = 0;
  for (long m = 0; m < n; m++) {
    double target = r + (double)m / (double)n;
    while (c < target && i + 1 < n) {
      i++;
      c += w[i];
    }
    ox[m] = x[i];
    oy[m] = y[i];
    ot[m] = t[i];
    ow[m] = 1.0 / (double)n;
    if (src) src[m] = i;
  }
}

/* Mcl::estimate (mcl.cpp:176-187) */
void orc_estimate(const double *x, const double *y, const double *t, const double *w, long n,
                  double *est) {
  double sx = 0, sy = 0, sc = 0, ss = 0, sw = 0;
  for (long i = 0; i < n; i++) {
    sx += w[i] * x[i];
    sy += w[i] * y[i];
    sc += w[i] * cos(t[i]);
    ss += w[i] * sin(t[i]);
    sw += w[i];
  }
  if (!(sw > 0.0)) sw = 1.0;
  est[0] = sx / sw;
  est[1] = sy / sw;
  est[2] = orc_normalize_angle_2pi(atan2(ss, sc));
}
