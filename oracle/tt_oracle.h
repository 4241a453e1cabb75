/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the hot path.
 *
 * Plain-C restatement of the reference's fp64 kernels
 * (/root/reference/proj/core/src/kernels.cpp) and of its input generators
 * (kernels.cpp:38-69 over rng.hpp:11-32).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.  The
 * product library (paper_2309_07235_b200/csrc) never links or calls it.
 *
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   - against the reference's own golden vectors (kernels_test.cpp:89-92,
 *     :99-121, :166-181, :232-243) committed under tests/golden/;
 *   - bitwise against the unmodified reference compiled by oracle/Makefile
 *     (oracle/_ref/libtiletuner_ref.so) on seeded inputs, whenever that
 *     library is present.
 *
 * Matrices are dense row-major doubles, index i*cols+j (matrix.hpp:18-23).
 * Status codes: 0 ok, 1 invalid argument, 2 numerical failure.
 */
#ifndef TT_ORACLE_H
#define TT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* mt19937_64 stream + the reference's conversions (rng.hpp:17-25). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_next_double(orc_rng* r);
uint64_t orc_rng_next_index(orc_rng* r, uint64_t n);

int orc_gen_spd(int n, uint64_t seed, double* out);
int orc_gen_3mm(int n, int l, int m, int o, int p, uint64_t seed, double* a,
                double* b, double* c, double* d);

int orc_mm3_reference(const double* a, const double* b, const double* c,
                      const double* d, int n, int l, int m, int o, int p,
                      double* g);
int orc_mm3_tiled(const double* a, const double* b, const double* c,
                  const double* d, int n, int l, int m, int o, int p,
                  const int* cfg, int ncfg, double* g);

/* fail_index (may be NULL) receives the failing column / row on status 2. */
int orc_lu_factor_inplace(double* a, int n, int by, int bx, int* fail_index);
int orc_cholesky_factor_inplace(double* a, int n, int by, int bx, int* fail_index);

double orc_lu_residual_packed(const double* a, const double* packed, int n);
double orc_cholesky_residual(const double* a, const double* fac, int n);
double orc_mm3_residual(const double* ref, const double* out, int64_t count);

#ifdef __cplusplus
}
#endif
#endif
