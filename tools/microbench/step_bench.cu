// What does one pivot step of the DIAG loop cost?  Variants strip pieces off.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256, 1) step(double* out, int T, long long* cyc) {
  __shared__ double pbuf[2 * 66];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double x[8][2];
  for (int q = 0; q < 8; ++q) { x[q][0] = 1.0 + w + q + lane; x[q][1] = 2.0 + lane; }
  if (threadIdx.x < 132) pbuf[threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * 66;
    double* nb = pbuf + ((k + 1) & 1) * 66;
    const int lk = k & 31;
    const double r = cb[64];
    double l[8];
    if (MODE & 1) {
#pragma unroll
      for (int q = 0; q < 8; ++q) l[q] = __shfl_sync(0xffffffffu, x[q][0], lk);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) l[q] = x[q][1];
    }
    const double u0 = cb[lane], u1 = cb[lane + 32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const bool act = w + 8 * q > k;
      const double m = act ? l[q] * r : 0.0;
      x[q][0] = fma(-m, u0, x[q][0]);
      x[q][1] = fma(-m, u1, x[q][1]);
    }
    if (MODE & 2) {
      if (((k + 1) & 7) == w) {
        nb[lane] = x[0][0];
        nb[lane + 32] = x[0][1];
        if (lane == ((k + 1) & 31)) nb[64] = (MODE & 4) ? 1.0 / x[0][0] : x[0][0] * 0.5;
      }
    }
    if (MODE & 8) __syncthreads(); else __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double acc = 0;
  for (int q = 0; q < 8; ++q) acc += x[q][0] + x[q][1];
  out[threadIdx.x] = acc;
}

template <int MODE>
void run(double* out, long long* cyc, const char* name) {
  step<MODE><<<1, 256>>>(out, 50, cyc);
  step<MODE><<<1, 256>>>(out, 50, cyc);
  cudaDeviceSynchronize();
  printf("%-40s %7.1f cycles/step\n", name, cyc[0] / 50.0);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * 8);
  cudaMallocManaged(&cyc, 8);
  run<0>(out, cyc, "fma only, syncwarp");
  run<8>(out, cyc, "fma + syncthreads");
  run<9>(out, cyc, "shfl + fma + syncthreads");
  run<11>(out, cyc, "shfl + fma + publish + syncthreads");
  run<15>(out, cyc, "... + 1/x");
  run<7>(out, cyc, "shfl + fma + publish + 1/x, syncwarp");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
