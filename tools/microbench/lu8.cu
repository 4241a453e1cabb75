// The 8x8 diagonal-block factorisation of the blocked DIAG, in isolation.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
template <int MODE>
__global__ void lu8(double* D, int* info, double* rk, long long* cyc) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (MODE & 4) {
    __syncthreads();
    if (threadIdx.x >= 32) { __syncthreads(); return; }
  }
  double v0 = D[g * 8 + 2 * t], v1 = D[g * 8 + 2 * t + 1];
  __syncwarp();
  long long t0 = clock64();
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const double sel = (kk & 1) ? v1 : v0;
    const double piv = __shfl_sync(0xffffffffu, sel, kk * 4 + (kk >> 1));
    const double agk = __shfl_sync(0xffffffffu, sel, g * 4 + (kk >> 1));
    const double u0 = __shfl_sync(0xffffffffu, v0, kk * 4 + t);
    const double u1 = __shfl_sync(0xffffffffu, v1, kk * 4 + t);
    const double r = (MODE & 1) ? rcp_nr(piv) : piv * 0.5;
    const double m = g > kk ? agk * r : 0.0;
    if (2 * t > kk) v0 = fma(-m, u0, v0);
    if (2 * t + 1 > kk) v1 = fma(-m, u1, v1);
    if (g > kk && 2 * t == kk) v0 = m;
    if (g > kk && 2 * t + 1 == kk) v1 = m;
    if (MODE & 2) {
      if (lane == 0) {
        rk[kk] = r;
        if (fabs(piv) < 1e-300) atomicMin(info, kk);
      }
    }
  }
  long long t1 = clock64() + (long long)(v0 * 0.0 + v1 * 0.0);
  if (lane == 0) cyc[0] = t1 - t0;
  D[64 + g * 8 + 2 * t] = v0;
  D[64 + g * 8 + 2 * t + 1] = v1;
  if (MODE & 4) __syncthreads();
}
template <int MODE>
void run(double* D, int* info, double* rk, long long* cyc, const char* name) {
  for (int r = 0; r < 3; ++r) lu8<MODE><<<1, (MODE & 4) ? 256 : 32>>>(D, info, rk, cyc);
  cudaDeviceSynchronize();
  printf("%-28s %lld cycles\n", name, cyc[0]);
}
int main() {
  double h[128];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) h[i * 8 + j] = (i == j ? 10.0 : 0.0) + 1.0 / (1 + i + j);
  double *D, *rk; int* info; long long* cyc;
  cudaMalloc(&D, 128 * 8); cudaMalloc(&rk, 64 * 8); cudaMalloc(&info, 4); cudaMallocManaged(&cyc, 8);
  cudaMemcpy(D, h, 64 * 8, cudaMemcpyHostToDevice);
  run<0>(D, info, rk, cyc, "shfl+fma only");
  run<1>(D, info, rk, cyc, "+ rcp_nr");
  run<3>(D, info, rk, cyc, "+ lane0 rk store + atomic");
  run<2>(D, info, rk, cyc, "no rcp, + lane0 block");
  run<5>(D, info, rk, cyc, "rcp, 7 warps at barrier");
  run<7>(D, info, rk, cyc, "rcp+lane0, 7 warps at barrier");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
