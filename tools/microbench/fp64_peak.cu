// fp64 peak probe for the roofline denominator (MEASURED_PEAKS.json has no fp64 entry).
// (1) DMMA: mma.sync.m8n8k4 f64 issue-rate loop, 8 independent accumulators per warp.
// (2) DFMA: scalar fma.rn.f64 chains, 8 independent per thread.
// Each reports TFLOP/s over a CUDA-event-timed launch at several warps/SM.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    for (int kind = 0; kind < 2; ++kind) {
      dim3 grid(sms), block(32 * warps);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) dmma_loop<<<grid, block>>>(out, iters);
        else dfma_loop<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = kind == 0
            ? 2.0 * 256.0 * 8 * iters * (double)warps * sms  // 8x8x4 per mma per warp
            : 2.0 * 8 * iters * (double)warps * 32 * sms;
        if (rep == 1)
          printf("{\"kind\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
                 kind == 0 ? "dmma_m8n8k4" : "dfma", warps, ms, flops / ms / 1e9);
      }
    }
  }
  return 0;
}
