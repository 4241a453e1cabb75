// Diagonal-block factorisations shared by the panel kernels and the
// persistent tile-DAG kernel: warp-register getrf/potrf of 32x32 blocks and
// their 2-level blocked composition for blocks up to 64 x 64 held in shared
// memory (kernels.cpp:186-196 restricted to the block, :289-306).
#pragma once
#include <cmath>

#include "factor_kernels.cuh"

namespace tt {
namespace diag {

constexpr int kLd = kIB + 1;

__device__ __forceinline__ bool failed(const int* info) {
  return *reinterpret_cast<const volatile int*>(info) != kNoFailure;
}

// ---- warp-level 32x32 factorisations in registers (lane i owns row i) ----
// The step-k operand every lane needs (LU: pivot row k; Cholesky: column k
// of L) goes through a small shared buffer and is read back with 128-bit
// broadcast loads — half the instructions of 64-bit shuffles.  Lanes that
// must not change use a zero multiplier instead of predication (x - 0*u = x
// for the finite u of a factorisation in progress).  `buf` is 2 x 32 doubles.

__device__ __forceinline__ void warp_getrf32(double (*D)[kLd], double* buf, int o, int w32,
                                             int gcol, int* info, bool report) {
  const int i = threadIdx.x & 31;
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (i < w32 && j < w32) ? D[o + i][o + j] : 0.0;
  if (i == 0) {
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[j] = x[j];
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k < w32) {
      const double* u = buf + (k & 1) * 32;  // pivot row k (final)
      const double piv = u[k];
      if (report && i == 0 && fabs(piv) < 1e-300) atomicMin(info, gcol + o + k);  // :187-190
      const bool act = i > k;
      const double l = act ? x[k] / piv : 0.0;  // :191, true division
      if (act) x[k] = l;
#pragma unroll
      for (int j = k + 1; j < 32; ++j) x[j] = fma(-l, u[j], x[j]);  // :192-195
      if (i == k + 1) {  // row k+1 is final now: publish it for step k+1
        double* nb = buf + ((k + 1) & 1) * 32;
#pragma unroll
        for (int j = 0; j < 32; ++j) nb[j] = x[j];
      }
      __syncwarp();
    }
  }
  if (i < w32) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < w32) D[o + i][o + j] = x[j];
  }
  __syncwarp();
}

__device__ __forceinline__ void warp_potrf32(double (*D)[kLd], double* buf, int o, int w32,
                                             int gcol, int* info, bool report) {
  const int i = threadIdx.x & 31;
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (i < w32 && j <= i) ? D[o + i][o + j] : 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k < w32) {
      double* col = buf + (k & 1) * 32;
      if (i == k) {
        const double d = x[k];
        if (report && d <= 0.0) atomicMin(info, gcol + o + k);  // :297-302 (NaN passes)
        x[k] = sqrt(d);
        col[k] = x[k];
      }
      __syncwarp();
      const double lkk = col[k];
      const bool act = i > k;
      const double l = act ? x[k] / lkk : 0.0;  // :295, true division
      if (act) x[k] = l;
      if (i != k) col[i] = l;  // column k of L (0 above the diagonal); col[k] keeps l_kk
      __syncwarp();
#pragma unroll
      for (int j = k + 1; j < 32; ++j) x[j] = fma(-l, col[j], x[j]);  // :293-294 (j > i unused)
    }
  }
  if (i < w32) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j <= i) D[o + i][o + j] = x[j];
  }
  __syncwarp();
}

// ---- the (w x w) diag block, w <= 64, 128 threads ----

__device__ inline void block_getrf(double (*D)[kLd], double* buf, int w, int gcol, int* info,
                            bool report) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = min(w, 32);
  if (warp == 0) warp_getrf32(D, buf, 0, w0, gcol, info, report);
  __syncthreads();
  if (w <= 32) return;
  const int w1 = w - 32;
  if (warp == 1 && lane < w1) {  // L rows 32.. against U(0:32)
    const int r = 32 + lane;
    double x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = D[r][j];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      x[k] = x[k] / D[k][k];
#pragma unroll
      for (int j = k + 1; j < 32; ++j) x[j] = fma(-x[k], D[k][j], x[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) D[r][j] = x[j];
  } else if (warp == 2 && lane < w1) {  // U columns 32.. with unit L(0:32)
    const int c = 32 + lane;
    double y[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) y[i] = D[i][c];
#pragma unroll
    for (int k = 0; k < 32; ++k)
#pragma unroll
      for (int i = k + 1; i < 32; ++i) y[i] -= D[i][k] * y[k];
#pragma unroll
    for (int i = 1; i < 32; ++i) D[i][c] = y[i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < w1 * w1; e += blockDim.x) {  // rank-32 update, ascending k
    const int i = 32 + e / w1, j = 32 + e - (e / w1) * w1;
    double s = D[i][j];
#pragma unroll 8
    for (int k = 0; k < 32; ++k) s -= D[i][k] * D[k][j];
    D[i][j] = s;
  }
  __syncthreads();
  if (warp == 0) warp_getrf32(D, buf, 32, w1, gcol, info, report);
  __syncthreads();
}

__device__ inline void block_potrf(double (*D)[kLd], double* buf, int w, int gcol, int* info,
                            bool report) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = min(w, 32);
  if (warp == 0) warp_potrf32(D, buf, 0, w0, gcol, info, report);
  __syncthreads();
  if (w <= 32) return;
  const int w1 = w - 32;
  if (warp == 1 && lane < w1) {  // L rows 32.. against L(0:32)
    const int r = 32 + lane;
    double x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = D[r][j];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      x[k] = x[k] / D[k][k];
#pragma unroll
      for (int j = k + 1; j < 32; ++j) x[j] = fma(-x[k], D[j][k], x[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) D[r][j] = x[j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < w1 * w1; e += blockDim.x) {  // lower rank-32 update
    const int i = 32 + e / w1, j = 32 + e - (e / w1) * w1;
    if (j > i) continue;
    double s = D[i][j];
#pragma unroll 8
    for (int k = 0; k < 32; ++k) s -= D[i][k] * D[j][k];
    D[i][j] = s;
  }
  __syncthreads();
  if (warp == 0) warp_potrf32(D, buf, 32, w1, gcol, info, report);
  __syncthreads();
}


}  // namespace diag
}  // namespace tt
