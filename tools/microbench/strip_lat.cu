// Latency of one GEMM strip's operand loads (16 rows x 50 doubles of A by
// cp.async.cg into shared memory + the C strip by ld.global.cg into
// registers) as issued by gemm_strips, per warp, with 1..148 CTAs x 8 warps
// loading concurrently from a 32 MB L2-resident matrix.  Variants: plain,
// preceded by an acquire load, and with an acquire poll issued while the
// loads are in flight (as the next-strip dependency check does).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const double* a, long long ld, int* flag, long long* out,
                                            int reps) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* buf = sm + warp * 16 * 68;
  long long tot = 0;
  double sink = 0;
  for (int r = 0; r < reps; ++r) {
    const int row0 = ((blockIdx.x * 8 + warp) * 16 + r * 4096) % 1968;
    const double* A = a + row0 * ld;
    const double* C = a + row0 * ld + 1000;
    __syncwarp();
    long long t0 = clock64();
    if (MODE == 1) sink += ld_acq(flag);
    if (MODE != 3 && MODE != 5)
    for (int e = lane; e < 16 * 25; e += 32) {
      const int rr = e / 25, v = e - rr * 25;
      cp16(buf + rr * 68 + 2 * v, A + rr * ld + 2 * v);
    }
    asm volatile("cp.async.commit_group;");
    double c[2][7][2];
    if (MODE == 6) {
#pragma unroll
      for (int mf = 0; mf < 2; ++mf)
#pragma unroll
        for (int nf = 0; nf < 7; ++nf) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(C + (mf * 8 + g) * ld + nf * 8 + 2 * t));
          c[mf][nf][0] = v.x;
          c[mf][nf][1] = v.y;
        }
    } else if (MODE == 7) {  // C strip by cp.async into smem, then fragments from smem
      double* cb = sm + 8 * 16 * 68 + warp * 16 * 68;
      for (int e = lane; e < 16 * 25; e += 32) {
        const int rr = e / 25, v = e - rr * 25;
        cp16(cb + rr * 68 + 2 * v, C + rr * ld + 2 * v);
      }
      asm volatile("cp.async.commit_group;");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int mf = 0; mf < 2; ++mf)
#pragma unroll
        for (int nf = 0; nf < 7; ++nf) {
          c[mf][nf][0] = cb[(mf * 8 + g) * 68 + nf * 8 + 2 * t];
          c[mf][nf][1] = cb[(mf * 8 + g) * 68 + nf * 8 + 2 * t + 1];
        }
    } else
#pragma unroll
    for (int mf = 0; mf < 2; ++mf)
#pragma unroll
      for (int nf = 0; nf < 7; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          c[mf][nf][h] = (MODE == 4 || (MODE == 3 && (mf | nf | h))) ? 0.0
                                                                   : __ldcg(C + (mf * 8 + g) * ld + nf * 8 + 2 * t + h);
    if (MODE == 2) sink += ld_acq(flag);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    double s = 0;
#pragma unroll
    for (int mf = 0; mf < 2; ++mf)
#pragma unroll
      for (int nf = 0; nf < 7; ++nf) s += c[mf][nf][0] + c[mf][nf][1];
    s += buf[g * 68 + t];
    long long t1 = clock64() + static_cast<long long>(s * 0.0);
    tot += t1 - t0;
    sink += s;
  }
  if (lane == 0) out[blockIdx.x * 8 + warp] = tot / reps;
  if (sink == 12345.678) out[0] = 0;
}

int main() {
  const long long ld = 2000;
  double* a;
  int* flag;
  long long* out;
  cudaMalloc(&a, 4000 * ld * 8);
  cudaMemset(a, 0, 4000 * ld * 8);
  cudaMalloc(&flag, 4);
  cudaMemset(flag, 0, 4);
  cudaMalloc(&out, 148 * 8 * 8);
  const int smem = 2 * 8 * 16 * 68 * 8;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[148 * 8];
  const char* names[] = {"plain", "acquire before", "acquire in flight", "one ldcg", "cp.async only",
                         "C ldcg only", "A cp.async + C ldcg.v2", "A + C both cp.async"};
  for (int mode = 0; mode < 8; ++mode)
    for (int grid : {1, 148}) {
      for (int it = 0; it < 2; ++it) {
        if (mode == 0) k<0><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 1) k<1><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 2) k<2><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 3) k<3><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 4) k<4><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 5) k<5><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 6) k<6><<<grid, 256, smem>>>(a, ld, flag, out, 64);
        if (mode == 7) k<7><<<grid, 256, smem>>>(a, ld, flag, out, 64);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, grid * 8 * 8, cudaMemcpyDeviceToHost);
      double s = 0;
      long long mx = 0;
      for (int i = 0; i < grid * 8; ++i) { s += h[i]; mx = h[i] > mx ? h[i] : mx; }
      printf("mode %d (%s) grid %3d: mean %.0f cycles, max %lld\n", mode, names[mode], grid,
             s / (grid * 8), mx);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
