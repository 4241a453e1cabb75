// Knob-parameterised schedules (see schedules.cuh).
#include <algorithm>

#include "schedules.cuh"

namespace tt {

namespace {

// Region of the internal (non-knob) sub-panel updates: 64 x 64 CTA tiles.
constexpr int kInnerRegion = 64;

#define TT_TRY(x)                          \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) return e_;      \
  } while (0)

}  // namespace

cudaError_t enqueue_lu(TmapCache& tc, double* a, int n, long long ld, int by, int bx, double* ws,
                       int* info, cudaStream_t s, ScheduleStats* st) {
  const Operand whole{a, n, n, ld, 0, 0};
  for (int p = 0; p < n; p += bx) {
    const int pe = p + bx;
    // Panel [p, pe): factored as sub-panels of width <= kIB.  Sub-panel q:
    // diag getrf + L rows (kernels.cpp:186-196), its U rows for every column
    // right of it (:198-203 and the in-panel part of :192-195), then the
    // rank-w update of the rest of the panel and of the panel's U12 rows.
    for (int q = p; q < pe; q += kIB) {
      const int w = std::min(kIB, pe - q);
      const int qe = q + w;
      launch_lu_panel(a, ld, n, q, w, ws, info, s);
      launch_lu_trsm_u(a, ld, q, w, qe, n - qe, ws, info, s);
      st->launches += 2;
      if (qe < pe) {
        Operand A = whole, B = whole;
        A.r0 = qe; A.c0 = q;  // L rows below the sub-panel
        B.r0 = q;  B.c0 = qe;  // U of the sub-panel, in-panel columns
        TT_TRY(gemm(tc, A, B, false, a + qe * ld + qe, ld, n - qe, pe - qe, w, kInnerRegion,
                    kInnerRegion, 1, 1, 0, 0, s));
        st->launches += 1;
        if (pe < n) {
          Operand A2 = whole, B2 = whole;
          A2.r0 = qe; A2.c0 = q;  // L of the later sub-panel rows of this panel
          B2.r0 = q;  B2.c0 = pe;  // U12 rows of this sub-panel
          TT_TRY(gemm(tc, A2, B2, false, a + qe * ld + pe, ld, pe - qe, n - pe, w, kInnerRegion,
                      kInnerRegion, 1, 1, 0, 0, s));
          st->launches += 1;
        }
      }
    }
    if (pe < n) {  // trailing update, kernels.cpp:205-216: region (by, bx), K = bx
      Operand A = whole, B = whole;
      A.r0 = pe; A.c0 = p;
      B.r0 = p;  B.c0 = pe;
      TT_TRY(gemm(tc, A, B, false, a + pe * ld + pe, ld, n - pe, n - pe, bx, by, bx, 1, 1, 0, 0, s));
      st->launches += 1;
    }
  }
  return cudaGetLastError();
}

cudaError_t enqueue_cholesky(TmapCache& tc, double* a, int n, long long ld, int by, int bx,
                             double* ws, int* info, cudaStream_t s, ScheduleStats* st) {
  const Operand whole{a, n, n, ld, 0, 0};
  for (int p = 0; p < n; p += bx) {
    const int pe = p + bx;
    for (int q = p; q < pe; q += kIB) {
      const int w = std::min(kIB, pe - q);
      const int qe = q + w;
      launch_chol_panel(a, ld, n, q, w, ws, info, s);
      st->launches += 2;
      if (qe < pe) {  // in-panel SYRK: A[qe:n, qe:pe] -= L[qe:n, q:qe] * L[qe:pe, q:qe]^T
        Operand A = whole, B = whole;
        A.r0 = qe; A.c0 = q;
        B.r0 = qe; B.c0 = q;
        TT_TRY(gemm(tc, A, B, true, a + qe * ld + qe, ld, n - qe, pe - qe, w, kInnerRegion,
                    kInnerRegion, 1, 1, 1, 0, s));
        st->launches += 1;
      }
    }
    if (pe < n) {  // trailing SYRK, lower only, region (by, bx), K = bx
      Operand A = whole, B = whole;
      A.r0 = pe; A.c0 = p;
      B.r0 = pe; B.c0 = p;
      TT_TRY(gemm(tc, A, B, true, a + pe * ld + pe, ld, n - pe, n - pe, bx, by, bx, 1, 1, 1, 0, s));
      st->launches += 1;
    }
  }
  return cudaGetLastError();
}

cudaError_t enqueue_mm3(TmapCache& tc, const Mm3Bufs& m, int n, int l, int mm, int o, int p,
                        const int* cfg, cudaStream_t s, cudaStream_t s2, cudaEvent_t fork,
                        cudaEvent_t join, ScheduleStats* st) {
  // F = C*D runs on s2 concurrently with E = A*B on s.
  TT_TRY(cudaEventRecord(fork, s));
  TT_TRY(cudaStreamWaitEvent(s2, fork, 0));
  const Operand C{m.c, mm, o, m.ldc, 0, 0}, D{m.d, o, p, m.ldd, 0, 0};
  TT_TRY(gemm(tc, C, D, false, m.f, m.ldf, mm, p, o, cfg[2], cfg[3], 0, 0, 0, 0, s2));
  TT_TRY(cudaEventRecord(join, s2));
  const Operand A{m.a, n, l, m.lda, 0, 0}, B{m.b, l, mm, m.ldb, 0, 0};
  TT_TRY(gemm(tc, A, B, false, m.e, m.lde, n, mm, l, cfg[0], cfg[1], 0, 0, 0, 0, s));
  TT_TRY(cudaStreamWaitEvent(s, join, 0));
  const Operand E{m.e, n, mm, m.lde, 0, 0}, F{m.f, mm, p, m.ldf, 0, 0};
  TT_TRY(gemm(tc, E, F, false, m.g, m.ldg, n, p, mm, cfg[4], cfg[5], 0, 0, 0, 0, s));
  st->launches += 3;
  return cudaGetLastError();
}

}  // namespace tt
