/* Checks the walker's division (cddt_device.cuh div_rn):
 *   q0 = RN(a * r), q1 = fma(fma(-d, q0, a), r, q0), q = fma(fma(-d, q1, a), r, q1),
 *   r = RN(1/d)
 * against IEEE a / d, bit for bit, over the operands the walker produces:
 * d = every non-axis direction cosine/sine of the theta_disc lattices
 * (direction_components, proj/src/cddt.cpp:30-42) and a = cell boundary -
 * origin, the origin a float-widened coordinate (batched casts), an arbitrary
 * f64 coordinate (sensor-model and particle-filter poses), a cell centre
 * (prune) or a float one ulp off a lattice line. The two-step form is correct
 * by Markstein's theorem (see div_rn); this is the empirical cross-check. It
 * also counts how often the ONE-step form RN(q0 + RN(a - d q0) r) would have
 * differed ("one_step_mismatches", informational: it is not used).
 * Usage: fast_div_check <samples per direction>
 *   -> prints "checked N mismatches M one_step_mismatches M1" */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define TWO_PI 6.283185307179586476925286766559

static uint64_t s = 0x243F6A8885A308D3ull;
static inline uint64_t nxt(void) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline double u01(void) { return (double)(nxt() >> 11) * 0x1.0p-53; }

static long checked = 0, bad = 0, bad1 = 0;
static void check(double a, double d) {
  double r = 1.0 / d;
  double q0 = a * r;
  double q1 = fma(fma(-d, q0, a), r, q0);
  double q = fma(fma(-d, q1, a), r, q1);
  double ref = a / d;
  checked++;
  if (q != ref || signbit(q) != signbit(ref)) {
    if (bad < 10) printf("mismatch a=%a d=%a q=%a ref=%a\n", a, d, q, ref);
    bad++;
  }
  if (q1 != ref) bad1++;
}

int main(int argc, char **argv) {
  long per = argc > 1 ? atol(argv[1]) : 2000;
  int ks[] = {4, 6, 8, 12, 16, 18, 22, 24, 32, 36, 64, 72, 100, 108, 120, 128, 200, 216, 256,
              360, 432, 512, 720, 1000, 1024, 2048, 4096};
  for (unsigned ki = 0; ki < sizeof ks / sizeof ks[0]; ki++) {
    int K = ks[ki];
    for (int i = 0; i < K; i++) {
      long long q4 = 4LL * i;
      if (q4 % K == 0) continue; /* axis-snapped: d is 0 or +-1 */
      double t = (double)i * TWO_PI / (double)K;
      double dd[2] = {cos(t), sin(t)};
      for (int k = 0; k < 2; k++) {
        double d = dd[k];
        for (long j = 0; j < per; j++) {
          int c = (int)(u01() * 8192.0) - 2;
          float of = (float)(u01() * 8192.0);
          double o = (double)of;
          check((double)c + 1.0 - o, d);
          check((double)c - o, d);
          double od = u01() * 8192.0; /* f64 origins: particle poses */
          check((double)c + 1.0 - od, d);
          check((double)c - od, d);
          double oc = (double)(int)(u01() * 8192.0) + 0.5; /* prune: cell centres */
          check((double)c + 1.0 - oc, d);
          check((double)c - oc, d);
          /* origins a hair off a lattice line */
          float near = nextafterf((float)c, (j & 1) ? 1e9f : -1e9f);
          check((double)c + 1.0 - (double)near, d);
          check((double)c - (double)near, d);
        }
      }
    }
  }
  /* direction_index: RN(theta * K / 2pi) with theta a float-widened angle in [0, 2pi) */
  for (unsigned ki = 0; ki < sizeof ks / sizeof ks[0]; ki++) {
    int K = ks[ki];
    for (long j = 0; j < per * 64; j++) {
      float th = (float)(u01() * TWO_PI);
      if ((double)th >= TWO_PI) continue;
      check((double)th * (double)K, TWO_PI);
      double thd = u01() * TWO_PI; /* f64 angles (sensor model beams) */
      check(thd * (double)K, TWO_PI);
    }
    for (int i = 0; i <= K; i++) check((double)i * TWO_PI / (double)K * (double)K, TWO_PI);
  }
  printf("checked %ld mismatches %ld one_step_mismatches %ld\n", checked, bad, bad1);
  return bad != 0;
}
