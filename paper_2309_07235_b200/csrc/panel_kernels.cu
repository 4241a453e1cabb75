// Fused tall-panel factorisation and U-row solve kernels (sm_100a).
//
// One launch factors a whole panel of width w <= 64 (kernels.cpp:186-196 for
// LU, :289-306 for Cholesky) over all its rows [q, n):
//   * every CTA loads the (w x w) diag block and factors it REDUNDANTLY in
//     shared memory — warp-shuffle register factorisation of 32x32
//     sub-blocks plus a 2-level blocked update for w > 32 — so no CTA ever
//     waits for another (identical arithmetic gives identical bits);
//   * CTA 0 stores the factored diag block to the scratch `ws` (writing it to
//     `a` here would race with other CTAs still loading it; the U-row solve
//     or launch_diag_writeback copies it back);
//   * each thread then owns one row below the diag block, held in 64
//     registers, and solves it against U11 (LU) / L11 (Cholesky).
// Per element the updates arrive in the reference's ascending-k order.  The
// diag block divides exactly like the reference; the tall rows multiply by
// the correctly rounded reciprocal of the pivot (<= 1 ulp per multiplier,
// inside the stated tolerance), which keeps the w-step dependency chain short.
#include <climits>
#include <cmath>

#include "diag_factor.cuh"

namespace tt {

namespace {

using namespace diag;

// ---- fused panel kernels ----
// Rows below the diag block are solved with the lanes of a warp spread over
// the panel's columns (lane j owns x_j and x_{j+32}) and four rows carried
// at once for ILP: per step k the finished x_k is broadcast by a shuffle and
// every lane j > k applies x_j -= x_k * u_kj.  That keeps 8 warps per CTA
// busy instead of one serial 64-step chain per thread.

constexpr int kThreads = 256;          // 8 warps
constexpr int kGroup = 4;              // rows (or columns) per warp in flight
constexpr int kPerWarp = 2 * kGroup;   // rows (columns) per warp
constexpr int kPerCta = 8 * kPerWarp;  // 64

template <int W, bool CHOL>
__global__ void __launch_bounds__(kThreads) panel_kernel(double* __restrict__ a, long long ld, int n,
                                                         int q, int w, double* __restrict__ ws,
                                                         int* info) {
  // D: the diag block.  After factorisation row k of D holds what step k of the
  // row solve needs: u_kj for LU; for Cholesky l_jk is mirrored into the
  // (otherwise unused) upper triangle so the lanes read contiguous words.
  __shared__ double D[kIB][kLd];
  __shared__ double rinv[kIB];
  __shared__ __align__(16) double buf[64];
  if (failed(info)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = q + w + blockIdx.x * kPerCta + warp * kPerWarp;
  for (int e = tid; e < w * w; e += kThreads) {
    const int i = e / w, j = e - (e / w) * w;
    D[i][j] = (!CHOL || j <= i) ? a[static_cast<long long>(q + i) * ld + q + j] : 0.0;
  }
  __syncthreads();
  if (CHOL)
    block_potrf(D, buf, w, q, info, blockIdx.x == 0);
  else
    block_getrf(D, buf, w, q, info, blockIdx.x == 0);
  if (blockIdx.x == 0) {
    for (int e = tid; e < w * w; e += kThreads) ws[e] = D[e / w][e - (e / w) * w];
  }
  if (tid < w) rinv[tid] = 1.0 / D[tid][tid];
  if (CHOL) {
    __syncthreads();
    for (int e = tid; e < w * w; e += kThreads) {
      const int k = e / w, j = e - (e / w) * w;
      if (j > k) D[k][j] = D[j][k];
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int grp = 0; grp < 2; ++grp) {
    const int rb = row0 + grp * kGroup;
    if (rb >= n) break;
    double xl[kGroup], xh[kGroup];
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int r = rb + g;
      const double* rp = a + static_cast<long long>(r < n ? r : q) * ld + q;
      xl[g] = (r < n && lane < w) ? rp[lane] : 0.0;
      xh[g] = (W > 32 && r < n && lane + 32 < w) ? rp[lane + 32] : 0.0;
    }
    for (int k = 0; k < w; ++k) {
      const double ul = D[k][lane];
      const double uh = W > 32 ? D[k][lane + 32] : 0.0;
      const double rk = rinv[k];
      const bool lo = k < 32;
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        const double xk = __shfl_sync(0xffffffffu, lo ? xl[g] : xh[g], k & 31) * rk;
        if (lo) {
          if (lane == k) xl[g] = xk;
          if (lane > k) xl[g] -= xk * ul;
        } else if (lane == k - 32) {
          xh[g] = xk;
        }
        if (W > 32 && lane + 32 > k) xh[g] -= xk * uh;
      }
    }
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int r = rb + g;
      if (r < n) {
        double* rp = a + static_cast<long long>(r) * ld + q;
        if (lane < w) rp[lane] = xl[g];
        if (W > 32 && lane + 32 < w) rp[lane + 32] = xh[g];
      }
    }
  }
}

// ---- LU U-row solve: rows [q, q+w) x cols [c0, c0+ncols) ----
// Forward substitution with the unit lower L of the factored diag block
// (`lsrc`, leading dim `lld`): for k: for i > k: x_i -= l_ik * x_k
// (kernels.cpp:198-203).  Lanes span the rows (lane i owns x_i, x_{i+32}),
// four columns per warp in flight.  With `writeback`, CTA 0 also copies the
// factored diag block from `lsrc` (the scratch) into `a`.
template <int W>
__global__ void __launch_bounds__(kThreads) trsm_u_kernel(double* __restrict__ a, long long ld,
                                                          int q, int w, int c0, int ncols,
                                                          const double* __restrict__ lsrc,
                                                          long long lld, int writeback,
                                                          const int* info) {
  __shared__ double Lt[kIB][kIB];  // Lt[k][i] = l_ik
  if (failed(info)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < w * w; e += kThreads) {
    const int i = e / w, j = e - (e / w) * w;
    const double v = lsrc[i * lld + j];
    Lt[j][i] = v;
    if (writeback && blockIdx.x == 0) a[static_cast<long long>(q + i) * ld + q + j] = v;
  }
  __syncthreads();
  const int cend = c0 + ncols;
#pragma unroll 1
  for (int grp = 0; grp < 2; ++grp) {
    const int cb = c0 + blockIdx.x * kPerCta + warp * kPerWarp + grp * kGroup;
    if (cb >= cend) break;
    double xl[kGroup], xh[kGroup];
    const double* rl = a + static_cast<long long>(q + lane) * ld;
    const double* rh = a + static_cast<long long>(q + lane + 32) * ld;
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int c = cb + g;
      xl[g] = (c < cend && lane < w) ? rl[c] : 0.0;
      xh[g] = (W > 32 && c < cend && lane + 32 < w) ? rh[c] : 0.0;
    }
    for (int k = 0; k + 1 < w; ++k) {
      const double ll = Lt[k][lane];
      const double lh = W > 32 ? Lt[k][lane + 32] : 0.0;
      const bool lo = k < 32;
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        const double xk = __shfl_sync(0xffffffffu, lo ? xl[g] : xh[g], k & 31);
        if (lane > k) xl[g] -= ll * xk;
        if (W > 32 && lane + 32 > k) xh[g] -= lh * xk;
      }
    }
#pragma unroll
    for (int g = 0; g < kGroup; ++g) {
      const int c = cb + g;
      if (c < cend) {
        if (lane >= 1 && lane < w) const_cast<double*>(rl)[c] = xl[g];
        if (W > 32 && lane + 32 < w) const_cast<double*>(rh)[c] = xh[g];
      }
    }
  }
}

unsigned blocks_for(long long work, int per) {
  const long long b = (work + per - 1) / per;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace

void launch_lu_panel(double* a, long long ld, int n, int q, int w, double* ws, int* info,
                     cudaStream_t s) {
  const unsigned g = blocks_for(n - q - w, kPerCta);
  if (w <= 32)
    panel_kernel<32, false><<<g, kThreads, 0, s>>>(a, ld, n, q, w, ws, info);
  else
    panel_kernel<64, false><<<g, kThreads, 0, s>>>(a, ld, n, q, w, ws, info);
}

void launch_chol_panel(double* a, long long ld, int n, int q, int w, double* ws, int* info,
                       cudaStream_t s) {
  const unsigned g = blocks_for(n - q - w, kPerCta);
  if (w <= 32)
    panel_kernel<32, true><<<g, kThreads, 0, s>>>(a, ld, n, q, w, ws, info);
  else
    panel_kernel<64, true><<<g, kThreads, 0, s>>>(a, ld, n, q, w, ws, info);
}

void launch_lu_trsm_u(double* a, long long ld, int q, int w, int c0, int ncols,
                      const double* lsrc, long long lld, int writeback, const int* info,
                      cudaStream_t s) {
  if (ncols < 0) ncols = 0;
  const unsigned g = blocks_for(ncols, kPerCta);
  if (w <= 32)
    trsm_u_kernel<32><<<g, kThreads, 0, s>>>(a, ld, q, w, c0, ncols, lsrc, lld, writeback, info);
  else
    trsm_u_kernel<64><<<g, kThreads, 0, s>>>(a, ld, q, w, c0, ncols, lsrc, lld, writeback, info);
}

}  // namespace tt
