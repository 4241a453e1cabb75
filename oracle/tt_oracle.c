/* TEST INFRASTRUCTURE ONLY — CPU oracle (see tt_oracle.h for the contract).
 *
 * Every function below restates one reference routine in plain C with the
 * same per-element operation order, so on the CPU its output is bitwise equal
 * to the reference's (checked in tests/test_oracle.py against
 * oracle/_ref/libtiletuner_ref.so and the golden vectors).  Compile with
 * -ffp-contract=off: the reference's Release build contains no FMA.
 */
#include "tt_oracle.h"

#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define IDX(i, j, cols) ((size_t)(i) * (size_t)(cols) + (size_t)(j))

/* ---- mt19937_64, as specified by the C++ standard ([rand.eng.mers]) ---- */
enum { MT_N = 312, MT_M = 156 };
static const uint64_t MT_A = 0xB5026F5AA96619E9ULL;
static const uint64_t MT_UPPER = 0xFFFFFFFF80000000ULL;
static const uint64_t MT_LOWER = 0x7FFFFFFFULL;

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->idx = MT_N;
}

static void mt_twist(orc_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:17-19: (u64 >> 11) * 2^-53 */
double orc_rng_next_double(orc_rng* r) {
  return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* rng.hpp:22-25: 128-bit multiply-shift */
uint64_t orc_rng_next_index(orc_rng* r, uint64_t n) {
  return (uint64_t)(((unsigned __int128)orc_rng_next_u64(r) * n) >> 64);
}

/* ---- generators ---- */

/* kernels.cpp:38-55: B ~ U[0,1) row-major, A = B*B^T + n*I (lower computed,
 * mirrored), ascending-k sum starting from 0.0. */
int orc_gen_spd(int n, uint64_t seed, double* a) {
  if (n < 1) return 1;
  orc_rng r;
  orc_rng_seed(&r, seed);
  double* b = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  if (!b) return 9;
  for (size_t i = 0; i < (size_t)n * (size_t)n; ++i) b[i] = orc_rng_next_double(&r);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j <= i; ++j) {
      double s = 0.0;
      const double* bi = b + IDX(i, 0, n);
      const double* bj = b + IDX(j, 0, n);
      for (int k = 0; k < n; ++k) s += bi[k] * bj[k];
      a[IDX(i, j, n)] = s;
      a[IDX(j, i, n)] = s;
    }
    a[IDX(i, i, n)] += (double)n;
  }
  free(b);
  return 0;
}

/* kernels.cpp:57-69: one stream fills A (n x l), B (l x m), C (m x o), D (o x p). */
int orc_gen_3mm(int n, int l, int m, int o, int p, uint64_t seed, double* a,
                double* b, double* c, double* d) {
  if (n < 1 || l < 1 || m < 1 || o < 1 || p < 1) return 1;
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (size_t i = 0; i < (size_t)n * l; ++i) a[i] = orc_rng_next_double(&r);
  for (size_t i = 0; i < (size_t)l * m; ++i) b[i] = orc_rng_next_double(&r);
  for (size_t i = 0; i < (size_t)m * o; ++i) c[i] = orc_rng_next_double(&r);
  for (size_t i = 0; i < (size_t)o * p; ++i) d[i] = orc_rng_next_double(&r);
  return 0;
}

/* ---- 3mm ---- */

/* kernels.cpp:73-86 matmul_naive: acc = 0; acc += x(i,k)*y(k,j), ascending k. */
static void matmul_naive(const double* x, const double* y, int r, int kk, int c,
                         double* out) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) {
      double acc = 0.0;
      for (int k = 0; k < kk; ++k) acc += x[IDX(i, k, kk)] * y[IDX(k, j, c)];
      out[IDX(i, j, c)] = acc;
    }
}

/* kernels.cpp:27-34 require_tile */
static int tile_ok(int f, int extent) { return f >= 1 && f <= extent && extent % f == 0; }

/* kernels.cpp:91-111 matmul_tiled: (yo, xo, k, yi, xi) nest on a zeroed out. */
static int matmul_tiled(const double* x, const double* y, int r, int kk, int c,
                        int fy, int fx, double* out) {
  if (!tile_ok(fy, r) || !tile_ok(fx, c)) return 1;
  memset(out, 0, sizeof(double) * (size_t)r * (size_t)c);
  for (int yo = 0; yo < r; yo += fy)
    for (int xo = 0; xo < c; xo += fx)
      for (int k = 0; k < kk; ++k)
        for (int yi = 0; yi < fy; ++yi) {
          const double xv = x[IDX(yo + yi, k, kk)];
          double* orow = out + IDX(yo + yi, xo, c);
          const double* yrow = y + IDX(k, xo, c);
          for (int xi = 0; xi < fx; ++xi) orow[xi] += xv * yrow[xi];
        }
  return 0;
}

/* kernels.cpp:115-120 */
int orc_mm3_reference(const double* a, const double* b, const double* c,
                      const double* d, int n, int l, int m, int o, int p,
                      double* g) {
  double* e = (double*)malloc(sizeof(double) * (size_t)n * m);
  double* f = (double*)malloc(sizeof(double) * (size_t)m * p);
  if (!e || !f) return 9;
  matmul_naive(a, b, n, l, m, e);
  matmul_naive(c, d, m, o, p, f);
  matmul_naive(e, f, n, m, p, g);
  free(e);
  free(f);
  return 0;
}

/* kernels.cpp:122-131: arity first, then each product's factors as it runs. */
int orc_mm3_tiled(const double* a, const double* b, const double* c,
                  const double* d, int n, int l, int m, int o, int p,
                  const int* cfg, int ncfg, double* g) {
  if (ncfg != 6) return 1;
  double* e = (double*)malloc(sizeof(double) * (size_t)n * m);
  double* f = (double*)malloc(sizeof(double) * (size_t)m * p);
  if (!e || !f) return 9;
  int rc = matmul_tiled(a, b, n, l, m, cfg[0], cfg[1], e);
  if (!rc) rc = matmul_tiled(c, d, m, o, p, cfg[2], cfg[3], f);
  if (!rc) rc = matmul_tiled(e, f, n, m, p, cfg[4], cfg[5], g);
  free(e);
  free(f);
  return rc;
}

/* ---- LU without pivoting ---- */

static const double kPivotFloor = 1e-300; /* kernels.cpp:15 */

/* kernels.cpp:178-218: right-looking blocked LU, panel width bx, trailing
 * rows tiled by `by`, columns by `bx`. */
int orc_lu_factor_inplace(double* a, int n, int by, int bx, int* fail_index) {
  if (n < 1) return 1;
  if (!tile_ok(by, n) || !tile_ok(bx, n)) return 1;
  for (int p = 0; p < n; p += bx) {
    const int pe = p + bx;
    for (int k = p; k < pe; ++k) { /* panel, :186-196 */
      const double pivot = a[IDX(k, k, n)];
      if (fabs(pivot) < kPivotFloor) {
        if (fail_index) *fail_index = k;
        return 2;
      }
      for (int i = k + 1; i < n; ++i) a[IDX(i, k, n)] /= pivot;
      for (int i = k + 1; i < n; ++i) {
        const double lik = a[IDX(i, k, n)];
        for (int j = k + 1; j < pe; ++j) a[IDX(i, j, n)] -= lik * a[IDX(k, j, n)];
      }
    }
    for (int k = p; k < pe; ++k) /* U12, :198-203 */
      for (int i = k + 1; i < pe; ++i) {
        const double lik = a[IDX(i, k, n)];
        for (int j = pe; j < n; ++j) a[IDX(i, j, n)] -= lik * a[IDX(k, j, n)];
      }
    for (int ib = pe; ib < n; ib += by) { /* trailing, :205-216 */
      const int ie = ib + by < n ? ib + by : n;
      for (int jb = pe; jb < n; jb += bx) {
        const int je = jb + bx < n ? jb + bx : n;
        for (int i = ib; i < ie; ++i)
          for (int k = p; k < pe; ++k) {
            const double lik = a[IDX(i, k, n)];
            for (int j = jb; j < je; ++j) a[IDX(i, j, n)] -= lik * a[IDX(k, j, n)];
          }
      }
    }
  }
  return 0;
}

/* ---- Cholesky ---- */

/* kernels.cpp:264-308: left-looking blocked Cholesky; only j <= i is written. */
int orc_cholesky_factor_inplace(double* a, int n, int by, int bx, int* fail_index) {
  if (n < 1) return 1;
  if (!tile_ok(by, n) || !tile_ok(bx, n)) return 1;
  for (int p = 0; p < n; p += bx) {
    const int pe = p + bx;
    for (int ib = p; ib < n; ib += by) { /* left update, :273-286 */
      const int ie = ib + by < n ? ib + by : n;
      for (int kb = 0; kb < p; kb += bx) {
        const int ke = kb + bx;
        for (int i = ib; i < ie; ++i) {
          const int jmax = pe - 1 < i ? pe - 1 : i;
          for (int j = p; j <= jmax; ++j) {
            double s = a[IDX(i, j, n)];
            for (int k = kb; k < ke; ++k) s -= a[IDX(i, k, n)] * a[IDX(j, k, n)];
            a[IDX(i, j, n)] = s;
          }
        }
      }
    }
    for (int i = p; i < n; ++i) { /* panel, :289-306 */
      const int jmax = pe - 1 < i ? pe - 1 : i;
      for (int j = p; j <= jmax; ++j) {
        if (j < i) {
          double s = a[IDX(i, j, n)];
          for (int k = p; k < j; ++k) s -= a[IDX(i, k, n)] * a[IDX(j, k, n)];
          a[IDX(i, j, n)] = s / a[IDX(j, j, n)];
        } else {
          double diag = a[IDX(i, i, n)];
          for (int k = p; k < i; ++k) diag -= a[IDX(i, k, n)] * a[IDX(i, k, n)];
          if (diag <= 0.0) {
            if (fail_index) *fail_index = i;
            return 2;
          }
          a[IDX(i, i, n)] = sqrt(diag);
        }
      }
    }
  }
  return 0;
}

/* ---- residuals (kernels.cpp:318-364) ---- */

static double max_abs(const double* m, size_t count) {
  double v = 0.0;
  for (size_t i = 0; i < count; ++i) {
    const double x = fabs(m[i]);
    v = v > x ? v : x; /* std::max(v, |x|) keeps v on ties and NaN-x */
  }
  return v;
}

/* kernels.cpp:326-338, with L/U read from the packed factor (unit diag). */
double orc_lu_residual_packed(const double* a, const double* packed, int n) {
  double num = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      const int kmax = i < j ? i : j;
      for (int k = 0; k <= kmax; ++k) {
        const double lik = k == i ? 1.0 : packed[IDX(i, k, n)];
        s += lik * packed[IDX(k, j, n)];
      }
      const double d = fabs(s - a[IDX(i, j, n)]);
      num = num > d ? num : d;
    }
  const double denom = max_abs(a, (size_t)n * n);
  return denom > 0.0 ? num / denom : num;
}

/* kernels.cpp:340-352 on the lower triangle of `fac`. */
double orc_cholesky_residual(const double* a, const double* fac, int n) {
  double num = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      const int kmax = i < j ? i : j;
      for (int k = 0; k <= kmax; ++k) s += fac[IDX(i, k, n)] * fac[IDX(j, k, n)];
      const double d = fabs(s - a[IDX(i, j, n)]);
      num = num > d ? num : d;
    }
  const double denom = max_abs(a, (size_t)n * n);
  return denom > 0.0 ? num / denom : num;
}

/* kernels.cpp:354-364 */
double orc_mm3_residual(const double* ref, const double* out, int64_t count) {
  double num = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double d = fabs(out[i] - ref[i]);
    num = num > d ? num : d;
  }
  const double denom = max_abs(ref, (size_t)count);
  return denom > 0.0 ? num / denom : num;
}
