// Incremental cost of the pieces of one DIAG pivot step (T=16: two warps active).
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
__global__ void __launch_bounds__(256, 1) step(double* out, int T, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, i0 = 8 * w;
  double x[8][2];
  for (int q = 0; q < 8; ++q) { x[q][0] = 1.0 + w + q + lane; x[q][1] = 2.0 + lane; }
  if (threadIdx.x < 264) pbuf[threadIdx.x] = 1.0 + threadIdx.x * 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * 132;
    double* nb = pbuf + ((k + 1) & 1) * 132;
    const int k1 = k + 1;
    if ((MODE & 1) && i0 + 7 > k && i0 < T) {
      const double r = cb[128];
      double a[8];
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        a[q] = v.x; a[q + 1] = v.y;
      }
      const double u0 = lane > k ? cb[lane] * r : 0.0;
      if (MODE & 2) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-a[q], u0, x[q][0]);
      }
      if (MODE & 4) {
        if (lane == (k1 & 31)) {
#pragma unroll
          for (int q = 0; q < 8; q += 2)
            *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
        }
      }
      if (MODE & 8) {
        if ((k1 >> 3) == w) {
          double v0 = x[0][0];
          switch (k1 & 7) {
            case 1: v0 = x[1][0]; break; case 2: v0 = x[2][0]; break; case 3: v0 = x[3][0]; break;
            case 4: v0 = x[4][0]; break; case 5: v0 = x[5][0]; break; case 6: v0 = x[6][0]; break;
            case 7: v0 = x[7][0]; break; default: break;
          }
          if (lane == (k1 & 31)) nb[128] = (MODE & 16) ? rcp_nr(v0) : v0;
          nb[lane] = v0;
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double acc = 0;
  for (int q = 0; q < 8; ++q) acc += x[q][0] + x[q][1];
  out[threadIdx.x] = acc;
}
template <int MODE>
void run(double* out, long long* cyc, const char* name) {
  for (int r = 0; r < 2; ++r) step<MODE><<<1, 256>>>(out, 16, cyc);
  cudaDeviceSynchronize();
  printf("%-44s %7.1f cycles/step\n", name, cyc[0] / 16.0);
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 256 * 8); cudaMallocManaged(&cyc, 8);
  run<0>(out, cyc, "barrier only");
  run<1>(out, cyc, "+ LDS (r, column, row)");
  run<3>(out, cyc, "+ 8 DFMA");
  run<7>(out, cyc, "+ column publish");
  run<15>(out, cyc, "+ row publish (switch)");
  run<31>(out, cyc, "+ rcp_nr");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
