// Stream-ordered schedules of the three tuned kernels, parameterised by the
// reference's knobs.  These are what the instantiation cache captures into
// one CUDA graph per (kernel, buffer, shape, knob setting).
#pragma once
#include <cuda_runtime.h>

#include "factor_kernels.cuh"
#include "gemm.hpp"

namespace tt {

struct ScheduleStats {
  long long launches = 0;  // kernel launches enqueued
};

// The critical stream s, the side stream s2 for the look-ahead trailing
// update, and two events reused for the s <-> s2 edges (valid under graph
// capture: a wait binds to the most recent record).
struct Streams {
  cudaStream_t s, s2;
  cudaEvent_t ev_panel, ev_g2;
};

// Right-looking blocked LU without pivoting (kernels.cpp:178-218), in place
// on the n x n row-major matrix `a` (leading dim ld).  Knobs: bx = panel
// width and trailing column tile, by = trailing row tile; the trailing
// update A22 -= L21*U12 runs with CTA region (by, bx) and K = bx.
// `ws` is a kIB*kIB scratch block, `info` the device status word.
cudaError_t enqueue_lu(TmapCache& tc, double* a, int n, long long ld, int by, int bx, double* ws,
                       int* info, const Streams& ss, ScheduleStats* st);

// Blocked Cholesky (kernels.cpp:264-308) in its right-looking form: per
// panel p of width bx: sub-panel potrf + row solves, the in-panel SYRK, then
// the trailing SYRK A22 -= L21*L21^T (lower only) with CTA region (by, bx).
// Per element the updates arrive in the same ascending-k order as the
// reference's left-looking loop; the upper triangle is never written.
cudaError_t enqueue_cholesky(TmapCache& tc, double* a, int n, long long ld, int by, int bx,
                             double* ws, int* info, const Streams& ss, ScheduleStats* st);

// 3mm (kernels.cpp:122-131): E = A*B (P0,P1), F = C*D (P2,P3) on two
// streams (they are independent), then G = E*F (P4,P5).  Dims positional
// (problem.cpp:35-36): A n x l, B l x m, C m x o, D o x p.
struct Mm3Bufs {
  const double *a, *b, *c, *d;
  long long lda, ldb, ldc, ldd;
  double *e, *f, *g;
  long long lde, ldf, ldg;
};
cudaError_t enqueue_mm3(TmapCache& tc, const Mm3Bufs& m, int n, int l, int mm, int o, int p,
                        const int* cfg, const Streams& ss, ScheduleStats* st);

}  // namespace tt
