/*
 * Seeded synthetic inputs for the BASELINE.json workloads (harness side, not
 * the product path): occupancy maps of the three named families, free-space
 * query streams, edit rounds, particle clouds and simulated scans.
 *
 * The paper's maps (Stata basement, Photoshop "Synthetic") are not available,
 * so these generators stand in for them with the shapes and densities that
 * BASELINE.json names. Every stream is SplitMix64
 * (the reference's portable RNG, proj/include/rangelib/rng.hpp:9-27) so the
 * same seed yields the same bytes on every machine. Compiled with
 * -ffp-contract=off so FP64 geometry is bit-reproducible.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TWO_PI 6.283185307179586476925286766559

static inline uint64_t sm_next(uint64_t *s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline double sm_uniform(uint64_t *s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }
/* independent per-item stream: state = mix(seed, item) */
static inline uint64_t sm_stream(uint64_t seed, uint64_t item) {
  uint64_t s = seed ^ 0x5851f42d4c957f2dull;
  uint64_t a = sm_next(&s);
  s = a + item * 0xd1b54a32d192ed03ull;
  (void)sm_next(&s);
  return s;
}
/* standard normal by Box-Muller on (0,1] x [0,1) */
static double sm_normal(uint64_t *s) {
  double u1 = 1.0 - sm_uniform(s);
  double u2 = sm_uniform(s);
  return sqrt(-2.0 * log(u1)) * cos(TWO_PI * u2);
}

static void fill_rect(uint8_t *g, int w, int h, int x0, int y0, int x1, int y1, uint8_t v,
                      long *occ) {
  if (x0 < 0) x0 = 0;
  if (y0 < 0) y0 = 0;
  if (x1 > w - 1) x1 = w - 1;
  if (y1 > h - 1) y1 = h - 1;
  for (int y = y0; y <= y1; y++)
    for (int x = x0; x <= x1; x++) {
      uint8_t *c = &g[(size_t)y * w + x];
      if (occ) *occ += (long)(v != 0) - (long)(*c != 0);
      *c = v;
    }
}

/* Config 1: 1-px border walls + nrect axis-aligned filled rectangles with
 * sides 5 + floor(56u) px placed uniformly inside the map. */
int synth_rect_map(uint8_t *g, int w, int h, int nrect, uint64_t seed) {
  if (w < 8 || h < 8 || nrect < 0) return 1;
  memset(g, 0, (size_t)w * h);
  uint64_t s = seed;
  fill_rect(g, w, h, 0, 0, w - 1, 0, 1, NULL);
  fill_rect(g, w, h, 0, h - 1, w - 1, h - 1, 1, NULL);
  fill_rect(g, w, h, 0, 0, 0, h - 1, 1, NULL);
  fill_rect(g, w, h, w - 1, 0, w - 1, h - 1, 1, NULL);
  for (int i = 0; i < nrect; i++) {
    int rw = 5 + (int)floor(56.0 * sm_uniform(&s));
    int rh = 5 + (int)floor(56.0 * sm_uniform(&s));
    if (rw > w) rw = w;
    if (rh > h) rh = h;
    int x0 = (int)floor(sm_uniform(&s) * (double)(w + 1 - rw));
    int y0 = (int)floor(sm_uniform(&s) * (double)(h + 1 - rh));
    fill_rect(g, w, h, x0, y0, x0 + rw - 1, y0 + rh - 1, 1, NULL);
  }
  return 0;
}

/* wall lattice along one axis: positions and thicknesses, first at 0, last
 * flush with the far border, pitch 40..120, thickness 2..4 */
static int wall_lattice(int extent, uint64_t *s, int *pos, int *thick, int cap) {
  int n = 0;
  int p = 0;
  for (;;) {
    int t = 2 + (int)floor(3.0 * sm_uniform(s));
    if (n >= cap - 1) break;
    pos[n] = p;
    thick[n] = t;
    n++;
    int pitch = 40 + (int)floor(81.0 * sm_uniform(s));
    p += pitch;
    if (p + 4 + 20 >= extent) break;
  }
  int t = 2 + (int)floor(3.0 * sm_uniform(s));
  pos[n] = extent - t;
  thick[n] = t;
  n++;
  return n;
}

/* Config 2/4/5: corridor maze. Rooms on a 40-120 px lattice, walls 2-4 px
 * thick, one door gap of 10-20 px carved in every interior wall segment,
 * then 3-12 px furniture blocks until target occupancy is reached. */
int synth_maze_map(uint8_t *g, int w, int h, double target_occ, uint64_t seed) {
  if (w < 64 || h < 64) return 1;
  memset(g, 0, (size_t)w * h);
  uint64_t s = seed;
  int cap = 4096;
  int *vx = malloc(sizeof(int) * cap), *vt = malloc(sizeof(int) * cap);
  int *hy = malloc(sizeof(int) * cap), *ht = malloc(sizeof(int) * cap);
  int nv = wall_lattice(w, &s, vx, vt, cap);
  int nh = wall_lattice(h, &s, hy, ht, cap);
  long occ = 0;
  for (int i = 0; i < nv; i++) fill_rect(g, w, h, vx[i], 0, vx[i] + vt[i] - 1, h - 1, 1, &occ);
  for (int j = 0; j < nh; j++) fill_rect(g, w, h, 0, hy[j], w - 1, hy[j] + ht[j] - 1, 1, &occ);
  /* doors in interior vertical walls: one per segment between horizontal walls */
  for (int i = 1; i + 1 < nv; i++)
    for (int j = 0; j + 1 < nh; j++) {
      int a = hy[j] + ht[j], b = hy[j + 1] - 1; /* free span [a, b] */
      int len = 10 + (int)floor(11.0 * sm_uniform(&s));
      int span = b - a + 1;
      double u = sm_uniform(&s);
      if (span < len + 4) continue;
      int y0 = a + 2 + (int)floor(u * (double)(span - len - 3));
      fill_rect(g, w, h, vx[i], y0, vx[i] + vt[i] - 1, y0 + len - 1, 0, &occ);
    }
  for (int j = 1; j + 1 < nh; j++)
    for (int i = 0; i + 1 < nv; i++) {
      int a = vx[i] + vt[i], b = vx[i + 1] - 1;
      int len = 10 + (int)floor(11.0 * sm_uniform(&s));
      int span = b - a + 1;
      double u = sm_uniform(&s);
      if (span < len + 4) continue;
      int x0 = a + 2 + (int)floor(u * (double)(span - len - 3));
      fill_rect(g, w, h, x0, hy[j], x0 + len - 1, hy[j] + ht[j] - 1, 0, &occ);
    }
  const long target = (long)ceil(target_occ * (double)w * (double)h);
  long guard = 0;
  while (occ < target && guard++ < 100000000L) {
    int bw = 3 + (int)floor(10.0 * sm_uniform(&s));
    int bh = 3 + (int)floor(10.0 * sm_uniform(&s));
    int x0 = (int)floor(sm_uniform(&s) * (double)(w - bw));
    int y0 = (int)floor(sm_uniform(&s) * (double)(h - bh));
    fill_rect(g, w, h, x0, y0, x0 + bw - 1, y0 + bh - 1, 1, &occ);
  }
  free(vx);
  free(vt);
  free(hy);
  free(ht);
  return 0;
}

static double cross3(const double *o, const double *a, const double *b) {
  return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0]);
}
static int cmp_pt(const void *pa, const void *pb) {
  const double *a = pa, *b = pb;
  if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
  if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
  return 0;
}

/* Config 3: 1-px border plus filled convex polygons (hull of 3-8 random points
 * in a disc of radius 5-60 px); a pixel is occupied iff its centre lies inside
 * the hull (FP64). Polygons are added until target occupancy is reached. */
int synth_polygon_map(uint8_t *g, int w, int h, double target_occ, uint64_t seed) {
  if (w < 16 || h < 16) return 1;
  memset(g, 0, (size_t)w * h);
  uint64_t s = seed;
  long occ = 0;
  fill_rect(g, w, h, 0, 0, w - 1, 0, 1, &occ);
  fill_rect(g, w, h, 0, h - 1, w - 1, h - 1, 1, &occ);
  fill_rect(g, w, h, 0, 0, 0, h - 1, 1, &occ);
  fill_rect(g, w, h, w - 1, 0, w - 1, h - 1, 1, &occ);
  const long target = (long)ceil(target_occ * (double)w * (double)h);
  double pts[8][2], hull[18][2];
  long guard = 0;
  while (occ < target && guard++ < 100000000L) {
    double cx = sm_uniform(&s) * w, cy = sm_uniform(&s) * h;
    double R = 5.0 + 55.0 * sm_uniform(&s);
    int n = 3 + (int)floor(6.0 * sm_uniform(&s));
    for (int i = 0; i < n; i++) {
      double a = TWO_PI * sm_uniform(&s), r = R * sqrt(sm_uniform(&s));
      pts[i][0] = cx + r * cos(a);
      pts[i][1] = cy + r * sin(a);
    }
    qsort(pts, n, sizeof(pts[0]), cmp_pt);
    int k = 0; /* Andrew monotone chain, counter-clockwise, collinear dropped */
    for (int i = 0; i < n; i++) {
      while (k >= 2 && cross3(hull[k - 2], hull[k - 1], pts[i]) <= 0) k--;
      hull[k][0] = pts[i][0];
      hull[k][1] = pts[i][1];
      k++;
    }
    for (int i = n - 2, t = k + 1; i >= 0; i--) {
      while (k >= t && cross3(hull[k - 2], hull[k - 1], pts[i]) <= 0) k--;
      hull[k][0] = pts[i][0];
      hull[k][1] = pts[i][1];
      k++;
    }
    k--; /* last equals first */
    if (k < 3) continue;
    double lo_x = hull[0][0], hi_x = lo_x, lo_y = hull[0][1], hi_y = lo_y;
    for (int i = 1; i < k; i++) {
      if (hull[i][0] < lo_x) lo_x = hull[i][0];
      if (hull[i][0] > hi_x) hi_x = hull[i][0];
      if (hull[i][1] < lo_y) lo_y = hull[i][1];
      if (hull[i][1] > hi_y) hi_y = hull[i][1];
    }
    int x0 = (int)floor(lo_x), x1 = (int)ceil(hi_x), y0 = (int)floor(lo_y), y1 = (int)ceil(hi_y);
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > w - 1) x1 = w - 1;
    if (y1 > h - 1) y1 = h - 1;
    for (int y = y0; y <= y1; y++)
      for (int x = x0; x <= x1; x++) {
        double p[2] = {x + 0.5, y + 0.5};
        int inside = 1;
        for (int i = 0; i < k && inside; i++)
          if (cross3(hull[i], hull[(i + 1) % k], p) < 0) inside = 0;
        if (inside) {
          uint8_t *c = &g[(size_t)y * w + x];
          if (!*c) {
            *c = 1;
            occ++;
          }
        }
      }
  }
  return 0;
}

static inline int cell_occ(const uint8_t *g, int w, int h, double x, double y) {
  int cx = (int)floor(x), cy = (int)floor(y);
  return cx >= 0 && cy >= 0 && cx < w && cy < h && g[(size_t)cy * w + cx];
}

/* n free-space queries: f32 x,y uniform over the map rectangle, rejected when
 * the widened point lies in an occupied cell; theta uniform in [0, 2pi).
 * Query i has its own stream so any slice [i0, i0+n) is reproducible and the
 * work splits across threads. */
int synth_free_queries(const uint8_t *g, int w, int h, uint64_t seed, size_t i0, size_t n,
                       float *qx, float *qy, float *qt) {
  const float fw = (float)w, fh = (float)h;
#pragma omp parallel for schedule(static)
  for (size_t k = 0; k < n; k++) {
    uint64_t s = sm_stream(seed, (uint64_t)(i0 + k));
    float x, y;
    int tries = 0;
    do {
      x = (float)(sm_uniform(&s) * w);
      y = (float)(sm_uniform(&s) * h);
      if (x >= fw) x = nextafterf(fw, 0.0f);
      if (y >= fh) y = nextafterf(fh, 0.0f);
    } while (cell_occ(g, w, h, (double)x, (double)y) && ++tries < 1000000);
    float t = (float)(sm_uniform(&s) * TWO_PI);
    if ((double)t >= TWO_PI) t = nextafterf(t, 0.0f);
    qx[k] = x;
    qy[k] = y;
    qt[k] = t;
  }
  return 0;
}

/* One edit round for config 5: nblocks 3x3 blocks, centre uniform, insert or
 * remove with p = 0.5, clipped to the map. Writes up to 9*nblocks (x, y, occ)
 * edits in sequential order and returns their count. */
long synth_block_edits(int w, int h, int nblocks, uint64_t seed, int32_t *xy, uint8_t *occ) {
  uint64_t s = seed;
  long n = 0;
  for (int b = 0; b < nblocks; b++) {
    int cx = (int)floor(sm_uniform(&s) * w), cy = (int)floor(sm_uniform(&s) * h);
    uint8_t op = sm_uniform(&s) < 0.5 ? 1 : 0;
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++) {
        int x = cx + dx, y = cy + dy;
        if (x < 0 || y < 0 || x >= w || y >= h) continue;
        xy[2 * n] = x;
        xy[2 * n + 1] = y;
        occ[n] = op;
        n++;
      }
  }
  return n;
}

/* Exact continuous ray cast (cell-walk to the first occupied cell's entry
 * point) used only to synthesise observed scans; the library's own oracle
 * lives under oracle/. */
double synth_exact_cast(const uint8_t *g, int w, int h, double ox, double oy, double theta,
                        double max_range) {
  int cx = (int)floor(ox), cy = (int)floor(oy);
  if (cx < 0 || cy < 0 || cx >= w || cy >= h) return max_range;
  if (g[(size_t)cy * w + cx]) return 0.0;
  double dx = cos(theta), dy = sin(theta);
  int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1;
  double tx = dx > 0 ? (cx + 1.0 - ox) / dx : dx < 0 ? (cx - ox) / dx : INFINITY;
  double ty = dy > 0 ? (cy + 1.0 - oy) / dy : dy < 0 ? (cy - oy) / dy : INFINITY;
  double t = 0.0;
  for (;;) {
    if (tx == ty) {
      t = tx;
      cx += sx;
      cy += sy;
    } else if (tx < ty) {
      t = tx;
      cx += sx;
    } else {
      t = ty;
      cy += sy;
    }
    if (t > max_range) return max_range;
    if (cx < 0 || cy < 0 || cx >= w || cy >= h) return max_range;
    if (g[(size_t)cy * w + cx]) return t;
    tx = dx > 0 ? (cx + 1.0 - ox) / dx : dx < 0 ? (cx - ox) / dx : INFINITY;
    ty = dy > 0 ? (cy + 1.0 - oy) / dy : dy < 0 ? (cy - oy) / dy : INFINITY;
  }
}

/* A pose in free space with every cell within `clearance` px free. */
int synth_free_pose(const uint8_t *g, int w, int h, int clearance, uint64_t seed, double *x,
                    double *y, double *theta) {
  uint64_t s = seed;
  for (long tries = 0; tries < 10000000L; tries++) {
    double px = sm_uniform(&s) * w, py = sm_uniform(&s) * h, pt = sm_uniform(&s) * TWO_PI;
    int cx = (int)floor(px), cy = (int)floor(py), ok = 1;
    for (int dy = -clearance; dy <= clearance && ok; dy++)
      for (int dx = -clearance; dx <= clearance && ok; dx++) {
        int nx = cx + dx, ny = cy + dy;
        if (nx < 0 || ny < 0 || nx >= w || ny >= h || g[(size_t)ny * w + nx]) ok = 0;
      }
    if (ok) {
      *x = px;
      *y = py;
      *theta = pt;
      return 0;
    }
  }
  return 1;
}

/* Gaussian particle cloud around a pose (particles inside obstacles are kept,
 * as in Mcl::init_gaussian, proj/src/mcl.cpp:165-174). theta in [0, 2pi). */
void synth_particles(double x, double y, double theta, double sxy, double sth, uint64_t seed,
                     long n, double *px, double *py, double *pt) {
  uint64_t s = seed;
  for (long i = 0; i < n; i++) {
    px[i] = x + sxy * sm_normal(&s);
    py[i] = y + sxy * sm_normal(&s);
    double t = fmod(theta + sth * sm_normal(&s), TWO_PI);
    if (t < 0) t += TWO_PI;
    if (t >= TWO_PI) t = 0.0;
    pt[i] = t;
  }
}

/* Observed scan: exact cast + N(0, sigma), with probability p_out replaced by
 * U[0, max_range], clamped to [0, max_range]. Beam bearings follow
 * ScanSpec::beam_offset (proj/include/rangelib/mcl.hpp:42-51). */
void synth_scan(const uint8_t *g, int w, int h, double x, double y, double theta, int nbeams,
                double fov, double max_range, double sigma, double p_out, uint64_t seed,
                double *scan) {
  uint64_t s = seed;
  for (int b = 0; b < nbeams; b++) {
    double off = nbeams <= 1 ? 0.0 : -fov / 2.0 + fov * (double)b / (double)(nbeams - 1);
    double d = synth_exact_cast(g, w, h, x, y, theta + off, max_range);
    double r = d + sigma * sm_normal(&s);
    if (sm_uniform(&s) < p_out) r = sm_uniform(&s) * max_range;
    if (r < 0.0) r = 0.0;
    if (r > max_range) r = max_range;
    scan[b] = r;
  }
}

/* A free-space trajectory at `step` px per iteration: straight ahead while the
 * way is clear, turning by a seeded angle when a wall is within `lookahead`.
 * Writes n+1 true poses and n robot-frame odometry increments (dx, 0, dtheta). */
int synth_trajectory(const uint8_t *g, int w, int h, double x, double y, double theta, long n,
                     double step, double lookahead, uint64_t seed, double *pose, double *odo) {
  uint64_t s = seed;
  pose[0] = x;
  pose[1] = y;
  pose[2] = theta;
  for (long i = 0; i < n; i++) {
    double dth = 0.0;
    for (int tries = 0; tries < 64; tries++) {
      double ahead = synth_exact_cast(g, w, h, x, y, theta + dth, lookahead + 1.0);
      if (ahead > lookahead) break;
      dth = (sm_uniform(&s) - 0.5) * 3.0;
    }
    /* robot-frame increment as motion_update applies it (translation in the
     * pre-step heading frame, then rotation): turn-then-move becomes
     * (step cos dth, step sin dth, dth) */
    theta = fmod(theta + dth, TWO_PI);
    if (theta < 0) theta += TWO_PI;
    x += step * cos(theta);
    y += step * sin(theta);
    odo[3 * i] = step * cos(dth);
    odo[3 * i + 1] = step * sin(dth);
    odo[3 * i + 2] = dth;
    pose[3 * (i + 1)] = x;
    pose[3 * (i + 1) + 1] = y;
    pose[3 * (i + 1) + 2] = theta;
  }
  return 0;
}

/* FNV-1a 64 over the width, height (little-endian bytes) and 0/1 cell
 * stream: the reference's map_content_id (proj/src/bench.cpp:22-34). */
uint64_t synth_map_fnv1a(const uint8_t *g, int w, int h) {
  uint64_t x = 1469598103934665603ull;
  for (int shift = 0; shift < 32; shift += 8) x = (x ^ ((uint32_t)w >> shift & 0xff)) * 1099511628211ull;
  for (int shift = 0; shift < 32; shift += 8) x = (x ^ ((uint32_t)h >> shift & 0xff)) * 1099511628211ull;
  size_t n = (size_t)w * h;
  for (size_t i = 0; i < n; i++) x = (x ^ (uint64_t)(g[i] ? 1 : 0)) * 1099511628211ull;
  return x;
}
