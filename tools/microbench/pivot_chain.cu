// Cycles per pivot of the 8x8 fragment-layout elimination (factor_block8's
// loop) and of stripped variants, one warp, registers only:
//   0 full (6 double shuffles, reciprocal chain, v and W updates)
//   1 no W tracking            2 no pivot-row shuffles (u from registers)
//   3 chain only: pivot shuffle -> reciprocal chain -> one update
//   4 full, 1/pivot by rcp.rn (IEEE) instead of seed + series
//   5 no W, pivot row through shared memory instead of shuffles
//   6 no W (the kernel's current loop)
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ double prow[8];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double v0 = 1.0 + 0.01 * lane + (g == 2 * t ? 8.0 : 0.0), v1 = 0.5 + 0.02 * lane + (g == 2 * t + 1 ? 8.0 : 0.0);
  double w0 = g == 2 * t ? 1.0 : 0.0, w1 = g == 2 * t + 1 ? 1.0 : 0.0;
  double acc = 0.0;
  __syncwarp();
  long long c0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const double sel = (kk & 1) ? v1 : v0;
      const double piv = __shfl_sync(0xffffffffu, sel, kk * 4 + (kk >> 1));
      const double agk_all = V == 3 ? sel : __shfl_sync(0xffffffffu, sel, g * 4 + (kk >> 1));
      const double agk = g > kk ? -agk_all : 0.0;
      double u0 = 0.3, u1 = 0.2, x0 = 0.1, x1 = 0.05;
      if (V == 5) {
        __syncwarp();
        if (g == kk) {
          prow[2 * t] = v0;
          prow[2 * t + 1] = v1;
        }
        __syncwarp();
        u0 = prow[2 * t];
        u1 = prow[2 * t + 1];
      } else if (V != 2 && V != 3) {
        u0 = __shfl_sync(0xffffffffu, v0, kk * 4 + t);
        u1 = __shfl_sync(0xffffffffu, v1, kk * 4 + t);
      }
      if (V != 1 && V != 3 && V != 5 && V != 6) {
        x0 = __shfl_sync(0xffffffffu, w0, kk * 4 + t);
        x1 = __shfl_sync(0xffffffffu, w1, kk * 4 + t);
      }
      double nm;
      if (V == 4) {
        double r;
        asm("rcp.rn.f64 %0, %1;" : "=d"(r) : "d"(piv));
        nm = agk * r;
      } else {
        double r0;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(piv));
        const double e = fma(-piv, r0, 1.0);
        const double tq = fma(e, e, e);
        const double nm0 = agk * r0;
        nm = fma(nm0, tq, nm0);
      }
      if (2 * t > kk) v0 = fma(nm, u0, v0);
      if (V != 3 && 2 * t + 1 > kk) v1 = fma(nm, u1, v1);
      if (g > kk && 2 * t == kk) v0 = -nm;
      if (g > kk && 2 * t + 1 == kk) v1 = -nm;
      if (V != 1 && V != 3 && V != 5 && V != 6) {
        w0 = fma(nm, x0, w0);
        w1 = fma(nm, x1, w1);
      }
    }
    // keep values bounded: restore the diagonal dominance each rep
    v0 = (g == 2 * t ? 8.0 : 0.0) + v0 * 1e-3;
    v1 = (g == 2 * t + 1 ? 8.0 : 0.0) + v1 * 1e-3;
  }
  long long c1 = clock64() + static_cast<long long>((v0 + v1 + w0 + w1) * 0.0);
  acc = v0 + v1 + w0 + w1;
  out[lane] = acc;
  if (lane == 0) *cyc = c1 - c0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8);
  const int reps = 2000;
  const char* names[] = {"full", "no W", "no pivot-row shuffles", "chain only", "full, rcp.rn",
                         "no W, pivot row via smem", "no W (kernel loop)"};
  for (int v = 0; v < 7; ++v) {
    long long h = 0;
    for (int it = 0; it < 2; ++it) {
      if (v == 0) k<0><<<1, 32>>>(out, cyc, reps);
      if (v == 1) k<1><<<1, 32>>>(out, cyc, reps);
      if (v == 2) k<2><<<1, 32>>>(out, cyc, reps);
      if (v == 3) k<3><<<1, 32>>>(out, cyc, reps);
      if (v == 4) k<4><<<1, 32>>>(out, cyc, reps);
      if (v == 5) k<5><<<1, 32>>>(out, cyc, reps);
      if (v == 6) k<6><<<1, 32>>>(out, cyc, reps);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-24s %.1f cycles/pivot\n", names[v], double(h) / (reps * 8.0));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
