// Panel / triangular-solve / generator / residual kernels (declarations).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tt {

// Widest panel one fused panel kernel factors: a reference panel of width
// bx <= 64 is ONE launch; wider panels are factored as ceil(bx/64)
// sub-panels, each a fused panel + U-row solve + DMMA update (same
// per-element operation set).
constexpr int kIB = 64;

// Status word value meaning "no numerical failure" (memset byte 0x7F).
constexpr int kNoFailure = 0x7F7F7F7F;

// LU sub-panel [q, q+w) x rows [q, n): diag getrf + L21 row solves
// (kernels.cpp:186-196 restricted to the sub-panel's columns).
// `ws` is a w*w scratch block receiving the factored diag block.
void launch_lu_panel(double* a, long long ld, int n, int q, int w, double* ws, int* info,
                     cudaStream_t s);
// U rows [q, q+w) x cols [c0, c0+ncols): forward substitution with the unit
// lower L of the sub-panel's diag block (kernels.cpp:198-203), read from
// `lsrc` (leading dim `lld`: the scratch `ws` with lld = w, or `a` itself).
// With `writeback` CTA 0 also copies the diag block from `lsrc` into `a`.
void launch_lu_trsm_u(double* a, long long ld, int q, int w, int c0, int ncols,
                      const double* lsrc, long long lld, int writeback, const int* info,
                      cudaStream_t s);
// Cholesky sub-panel: diag potrf (diag <= 0 fails, kernels.cpp:297-302) +
// row solves below (kernels.cpp:292-295); lower triangle only.  The factored
// diag block goes to `ws`; launch_diag_writeback copies it into `a`.
void launch_chol_panel(double* a, long long ld, int n, int q, int w, double* ws, int* info,
                       cudaStream_t s);
void launch_diag_writeback(double* a, long long ld, int q, int w, const double* ws,
                           int lower_only, cudaStream_t s);

// gen_spd on the device, bitwise equal to kernels.cpp:38-55: a = b*b^T + n*I
// with unfused, ascending-k products (b row-major n x n, ld_b).
void launch_spd_product(const double* b, long long ldb, int n, double* a, long long lda,
                        cudaStream_t s);

// Counter-based U[0,1) fill of rows [row0, row0+rows) of a global matrix
// (`stream` separates matrices): shard-invariant device inputs for the
// scaled 3mm, where no CPU oracle exists.
void launch_fill_uniform(double* a, long long ld, int rows, int cols, long long row0,
                         unsigned long long seed, int stream, cudaStream_t s);

// Residual helpers.
void launch_unpack_lu(const double* f, long long ldf, int n, double* l, double* u, long long ld,
                      cudaStream_t s);
void launch_lower_of(const double* f, long long ldf, int n, double* l, long long ld,
                     cudaStream_t s);
// out[0] = max(out[0], max |x - y|), out[1] = max(out[1], max |y|) over an
// rows x cols view (out are doubles reinterpreted as ordered uint64).
void launch_maxdiff(const double* x, long long ldx, const double* y, long long ldy, int rows,
                    int cols, unsigned long long* out, cudaStream_t s);

}  // namespace tt
