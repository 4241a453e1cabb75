// Knob-parameterised schedules (see schedules.cuh).
//
// LU and Cholesky run as a two-stream DAG with look-ahead of one panel: the
// trailing update of step k is split into G1 (the next panel's column block,
// on the critical stream s) and G2 (all later columns, on the side stream
// s2), so the panel factorisation of step k+1 overlaps G2 of step k.  Both
// G1 and G2 keep the reference's trailing tiling: CTA regions of (by x bx)
// anchored at the trailing origin (kernels.cpp:205-216, 273-286).
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
                       int* info, const Streams& ss, ScheduleStats* st) {
  const Operand whole{a, n, n, ld, 0, 0};
  cudaStream_t s = ss.s, s2 = ss.s2;
  const int nq = (bx + kIB - 1) / kIB;
  bool g2_pending = false;
  for (int p = 0; p < n; p += bx) {
    const int pe = p + bx;
    // -- panel phase: needs only column block k (updated by G1 of step k-1).
    // Sub-panel q: fused panel factorisation (kernels.cpp:186-196); for wide
    // panels also its U rows inside the panel and the in-panel update.
    for (int q = p; q < pe; q += kIB) {
      const int w = std::min(kIB, pe - q);
      const int qe = q + w;
      launch_lu_panel(a, ld, n, q, w, ws, info, s);
      st->launches += 1;
      if (nq > 1) {
        launch_lu_trsm_u(a, ld, q, w, qe, pe - qe, ws, w, 1, info, s);
        st->launches += 1;
        if (qe < pe) {
          Operand A = whole, B = whole;
          A.r0 = qe; A.c0 = q;
          B.r0 = q;  B.c0 = qe;
          TT_TRY(gemm(tc, A, B, false, a + qe * ld + qe, ld, n - qe, pe - qe, w, kInnerRegion,
                      kInnerRegion, 1, 1, 0, 0, s));
          st->launches += 1;
        }
      }
    }
    // -- U12 phase (kernels.cpp:198-203): block row k, columns [pe, n), needs
    // G2 of step k-1.
    if (g2_pending) TT_TRY(cudaStreamWaitEvent(s, ss.ev_g2, 0));
    if (nq == 1) {
      launch_lu_trsm_u(a, ld, p, bx, pe, n - pe, ws, bx, 1, info, s);  // + diag write-back
      st->launches += 1;
    } else if (pe < n) {
      for (int q = p; q < pe; q += kIB) {
        const int w = std::min(kIB, pe - q);
        const int qe = q + w;
        launch_lu_trsm_u(a, ld, q, w, pe, n - pe, a + q * ld + q, ld, 0, info, s);
        st->launches += 1;
        if (qe < pe) {
          Operand A = whole, B = whole;
          A.r0 = qe; A.c0 = q;
          B.r0 = q;  B.c0 = pe;
          TT_TRY(gemm(tc, A, B, false, a + qe * ld + pe, ld, pe - qe, n - pe, w, kInnerRegion,
                      kInnerRegion, 1, 1, 0, 0, s));
          st->launches += 1;
        }
      }
    }
    if (pe >= n) break;
    // -- trailing update A22 -= L21 * U12, K = bx, regions (by, bx).
    Operand A = whole, B = whole;
    A.r0 = pe; A.c0 = p;
    B.r0 = p;
    TT_TRY(cudaEventRecord(ss.ev_panel, s));
    const int c1 = std::min(n, pe + bx);
    B.c0 = pe;  // G1: the next panel's column block, on the critical stream
    TT_TRY(gemm(tc, A, B, false, a + pe * ld + pe, ld, n - pe, c1 - pe, bx, by, bx, 1, 1, 0, 0, s));
    st->launches += 1;
    if (c1 < n) {  // G2: the rest, on the side stream
      TT_TRY(cudaStreamWaitEvent(s2, ss.ev_panel, 0));
      B.c0 = c1;
      TT_TRY(gemm(tc, A, B, false, a + pe * ld + c1, ld, n - pe, n - c1, bx, by, bx, 1, 1, 0, 0,
                  s2));
      TT_TRY(cudaEventRecord(ss.ev_g2, s2));
      st->launches += 1;
      g2_pending = true;
    } else {
      g2_pending = false;
    }
  }
  if (g2_pending) TT_TRY(cudaStreamWaitEvent(s, ss.ev_g2, 0));  // join the side stream
  return cudaGetLastError();
}

cudaError_t enqueue_cholesky(TmapCache& tc, double* a, int n, long long ld, int by, int bx,
                             double* ws, int* info, const Streams& ss, ScheduleStats* st) {
  const Operand whole{a, n, n, ld, 0, 0};
  cudaStream_t s = ss.s, s2 = ss.s2;
  bool g2_pending = false;
  for (int p = 0; p < n; p += bx) {
    const int pe = p + bx;
    // -- panel phase (kernels.cpp:289-306): needs only column block k
    for (int q = p; q < pe; q += kIB) {
      const int w = std::min(kIB, pe - q);
      const int qe = q + w;
      launch_chol_panel(a, ld, n, q, w, ws, info, s);
      launch_diag_writeback(a, ld, q, w, ws, 1, s);
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
    if (pe >= n) break;
    // -- trailing SYRK (kernels.cpp:273-286 applied right-looking), lower only
    TT_TRY(cudaEventRecord(ss.ev_panel, s));
    if (g2_pending) TT_TRY(cudaStreamWaitEvent(s, ss.ev_g2, 0));  // block k+1 got step k-1
    Operand A = whole, B = whole;
    A.r0 = pe; A.c0 = p;
    B.c0 = p;
    const int c1 = std::min(n, pe + bx);
    B.r0 = pe;  // G1: rows [pe, n) x the next column block
    TT_TRY(gemm(tc, A, B, true, a + pe * ld + pe, ld, n - pe, c1 - pe, bx, by, bx, 1, 1, 1, 0, s));
    st->launches += 1;
    if (c1 < n) {  // G2: rows [c1, n) x columns [c1, n) ... and its lower part only
      TT_TRY(cudaStreamWaitEvent(s2, ss.ev_panel, 0));
      B.r0 = c1;
      TT_TRY(gemm(tc, A, B, true, a + pe * ld + c1, ld, n - pe, n - c1, bx, by, bx, 1, 1, 1,
                  pe - c1, s2));
      TT_TRY(cudaEventRecord(ss.ev_g2, s2));
      st->launches += 1;
      g2_pending = true;
    } else {
      g2_pending = false;
    }
  }
  if (g2_pending) TT_TRY(cudaStreamWaitEvent(s, ss.ev_g2, 0));  // join the side stream
  return cudaGetLastError();
}

cudaError_t enqueue_mm3(TmapCache& tc, const Mm3Bufs& m, int n, int l, int mm, int o, int p,
                        const int* cfg, const Streams& ss, ScheduleStats* st) {
  // F = C*D runs on s2 concurrently with E = A*B on s.
  cudaStream_t s = ss.s, s2 = ss.s2;
  TT_TRY(cudaEventRecord(ss.ev_panel, s));
  TT_TRY(cudaStreamWaitEvent(s2, ss.ev_panel, 0));
  const Operand C{m.c, mm, o, m.ldc, 0, 0}, D{m.d, o, p, m.ldd, 0, 0};
  TT_TRY(gemm(tc, C, D, false, m.f, m.ldf, mm, p, o, cfg[2], cfg[3], 0, 0, 0, 0, s2));
  TT_TRY(cudaEventRecord(ss.ev_g2, s2));
  const Operand A{m.a, n, l, m.lda, 0, 0}, B{m.b, l, mm, m.ldb, 0, 0};
  TT_TRY(gemm(tc, A, B, false, m.e, m.lde, n, mm, l, cfg[0], cfg[1], 0, 0, 0, 0, s));
  TT_TRY(cudaStreamWaitEvent(s, ss.ev_g2, 0));
  const Operand E{m.e, n, mm, m.lde, 0, 0}, F{m.f, mm, p, m.ldf, 0, 0};
  TT_TRY(gemm(tc, E, F, false, m.g, m.ldg, n, p, mm, cfg[4], cfg[5], 0, 0, 0, 0, s));
  st->launches += 3;
  return cudaGetLastError();
}

}  // namespace tt
