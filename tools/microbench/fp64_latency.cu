// Dependent-chain latencies (cycles per op, 64-op unrolled chains, no loop
// overhead) of the ops on the factorisation critical path.
#include <cstdio>
#include <cuda_runtime.h>

#define R64(x) x x x x x x x x x x x x x x x x x x x x x x x x x x x x x x x x \
               x x x x x x x x x x x x x x x x x x x x x x x x x x x x x x x x

__global__ void lat(double* out, long long* cyc, double seed, int idx0) {
  __shared__ double sh[64];
  __shared__ int shi[64];
  if (threadIdx.x < 64) { sh[threadIdx.x] = seed + threadIdx.x; shi[threadIdx.x] = (threadIdx.x + 1) & 63; }
  __syncthreads();
  double x = seed, y = seed + 1.0, r = 1.5 + seed, q = 3.0 + seed, s = 2.0 + seed;
  float f = (float)seed;
  int id = idx0;
  double v = seed;
  long long t0, t1;
#define TIME(slot, body) t0 = clock64(); R64(body) t1 = clock64(); if (threadIdx.x == 0) cyc[slot] = (t1 - t0);
  const double c1 = 0.999999, c2 = 1e-9, c3 = 1.7;
  TIME(0, asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(c1), "d"(c2));)
  TIME(1, asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(y) : "d"(c1));)
  TIME(2, asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(c2));)
  TIME(3, asm volatile("rcp.rn.f64 %0, %0;" : "+d"(r));)
  TIME(4, asm volatile("div.rn.f64 %0, %0, %1;" : "+d"(q) : "d"(c3));)
  TIME(5, asm volatile("sqrt.rn.f64 %0, %0;" : "+d"(s));)
  TIME(6, asm volatile("ld.shared.s32 %0, [%1];" : "=r"(id) : "r"((unsigned)__cvta_generic_to_shared(&shi[id & 63])));)
  TIME(7, asm volatile("shfl.sync.idx.b32 %0, %0, %1, 31, -1;" : "+r"(id) : "r"((int)(threadIdx.x + 1) & 31));)
  TIME(8, asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f) : "f"(0.999f));)
  TIME(9, __syncthreads();)
  double d0 = seed, d1 = seed;
  TIME(10, asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(x), "d"(y));)
  double rc = 1.3 + seed;
  TIME(11, asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(rc));)
  out[threadIdx.x] = x + y + r + q + s + id + v + f + d0 + d1 + rc;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"DFMA", "DMUL", "DADD", "1.0/x (full)", "x/1.7 (full)", "sqrt", "LDS (int chase)",
                         "SHFL", "FFMA fp32", "__syncthreads", "DMMA m8n8k4 (acc chain)", "rcp.approx.f64 (MUFU)"};
  for (int threads : {32, 256}) {
    for (int rep = 0; rep < 2; ++rep) lat<<<1, threads>>>(out, cyc, 0.5, 0);
    cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 12; ++i) printf("  %-26s %6.1f cycles\n", names[i], cyc[i] / 64.0);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
