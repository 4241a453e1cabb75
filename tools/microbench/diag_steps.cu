// Per-step clock stamps of the DIAG loop (owner warp of the next pivot row).
#include <cstdio>
#include <vector>
#include "../../paper_2309_07235_b200/csrc/dag_factor.cu"
using namespace tt::dag;
namespace tt { namespace dag { namespace {
template <bool CHOL>
__device__ __forceinline__ void tile_factor_stamped(double* __restrict__ dk, long long ld, int T, int gcol,
                                            int* info, double* pbuf, double* rk,
                                            unsigned long long* ph, long long* st) {
  // pbuf parity block: [0,64) pivot row (LU), [64,128) column k, [128] 1/pivot, [129] l_kk
  // rk[c]: 1/pivot of column c (LU) or 1/l_cc (Cholesky); rk[64 + c]: l_cc
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = 8 * w;
  const bool wide = T > 32;
  double x[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      x[q][h] = (i < T && c < T && (!CHOL || c <= i))
                    ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
    }
  }
  // publish step 0: column 0 (+ row 0 for LU) and the pivot's reciprocal
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) pbuf[64 + i0 + q] = x[q][0];
  }
  if (w == 0) {
    if (!CHOL) {
      pbuf[lane] = x[0][0];
      pbuf[lane + 32] = x[0][1];
    }
    if (lane == 0) {
      const double d = x[0][0];
      if (!CHOL) {
        if (fabs(d) < 1e-300) atomicMin(info, gcol);  // kernels.cpp:187-190
        rk[0] = pbuf[128] = rcp_nr(d);
      } else {
        if (d <= 0.0) atomicMin(info, gcol);  // kernels.cpp:297-302 (NaN passes)
        const double l0 = sqrt(d);
        rk[64] = pbuf[129] = l0;
        rk[0] = pbuf[128] = rcp_nr(l0);
      }
    }
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * kPB;
    double* nb = pbuf + ((k + 1) & 1) * kPB;
    const int k1 = k + 1;
    const bool own = ((k1 >> 3) == w) && lane == 0 && st;
    if (own) st[k * 5 + 0] = clock64();
    if (i0 + 7 > k) {  // warp-uniform: this warp still has rows > k
      const double r = cb[128];
      double m[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        m[q] = v.x * r;
        m[q + 1] = v.y * r;
      }
      if (i0 <= k) {  // the warp holding row k: rows <= k are final
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (i0 + q <= k) m[q] = 0.0;
      }
      // operand row: LU pivot row k, Cholesky l_ck = a_ck / l_kk; 0 for columns <= k
      const double* src = CHOL ? cb + 64 : cb;
      const double sc = CHOL ? r : 1.0;
      const double u0 = lane > k ? src[lane] * sc : 0.0;
      if (wide) {
        const double u1 = lane + 32 > k ? src[lane + 32] * sc : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q][0] = fma(-m[q], u0, x[q][0]);
          x[q][1] = fma(-m[q], u1, x[q][1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-m[q], u0, x[q][0]);
      }
      if (own) st[k * 5 + 1] = clock64() + (long long)(x[0][0] * 0);
      if (k1 < T) {
        // publish column k+1 of my rows (the lane holding it)
        if (lane == (k1 & 31)) {
          if (k1 >= 32) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][1], x[q + 1][1]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
          }
        }
        // publish row k+1 (LU) and the next pivot's reciprocal (its owner warp)
        if ((k1 >> 3) == w) {
          const int q1 = k1 & 7;
          double v0 = x[0][0], v1 = x[0][1];
#pragma unroll
          for (int q = 1; q < 8; ++q)
            if (q == q1) {
              v0 = x[q][0];
              v1 = x[q][1];
            }
          if (!CHOL) {
            nb[lane] = v0;
            nb[lane + 32] = v1;
          }
          if (own) st[k * 5 + 2] = clock64();
          if (lane == (k1 & 31)) {
            const double d = k1 >= 32 ? v1 : v0;
            if (!CHOL) {
              if (fabs(d) < 1e-300) atomicMin(info, gcol + k1);  // kernels.cpp:187-190
              rk[k1] = nb[128] = rcp_nr(d);
            } else {
              if (d <= 0.0) atomicMin(info, gcol + k1);  // kernels.cpp:297-302
              const double l1 = sqrt(d);
              rk[64 + k1] = nb[129] = l1;
              rk[k1] = nb[128] = rcp_nr(l1);
            }
          }
        }
      }
    }
    if (own) st[k * 5 + 3] = clock64();
    __syncthreads();
    if (own) st[k * 5 + 4] = clock64();
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();
  // multipliers below the diagonal (and l_cc on it for Cholesky), then store
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (i < T && c < T && (!CHOL || c <= i)) {
        double v = x[q][h];
        if (c < i) v *= rk[c];
        if (CHOL && c == i) v = rk[64 + c];
        dk[static_cast<long long>(i) * ld + c] = v;
      }
    }
  }
}


} } }
__global__ void __launch_bounds__(256, 1) bench(double* a, long long ld, int T, int* info, long long* st) {
  __shared__ __align__(16) double pbuf[2 * 132];
  __shared__ double rk[128];
  tt::dag::tile_factor_stamped<false>(a, ld, T, 0, info, pbuf, rk, nullptr, st);
}
int main() {
  const int n = 64;
  std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double* d; int* info; long long* st;
  cudaMalloc(&d, n * n * 8); cudaMalloc(&info, 4); cudaMallocManaged(&st, 64 * 5 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaMemset(info, 0x7f, 4);
    cudaMemset(st, 0, 64 * 5 * 8);
    bench<<<1, 256>>>(d, n, 50, info, st);
    cudaDeviceSynchronize();
  }
  for (int k = 10; k < 20; ++k)
    printf("k=%d start->upd %lld upd->rowpub %lld rowpub->rcp+pub %lld bar %lld | next start %lld\n", k,
           st[k*5+1]-st[k*5+0], st[k*5+2]-st[k*5+1], st[k*5+3]-st[k*5+2], st[k*5+4]-st[k*5+3],
           st[(k+1)*5+0]-st[k*5+4]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
