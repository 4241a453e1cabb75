// Standalone timing of the persistent kernel's DIAG tile factorisation
// (tile_factor in dag_factor.cu) on one CTA, to separate its cost from the
// scheduling environment.
#include <cstdio>
#include <vector>
#include "../../paper_2309_07235_b200/csrc/dag_factor.cu"

using namespace tt::dag;

template <bool CHOL>
__global__ void __launch_bounds__(256, 1) bench(double* a, long long ld, int T, int* info, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132];
  __shared__ double rk[128];
  __shared__ double slv[64];
  __syncthreads();
  long long t0 = clock64();
  tile_factor<CHOL>(a, ld, T, 0, info, pbuf, rk, nullptr, slv);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  const int n = 64;
  std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double* d;
  int* info;
  long long* cyc;
  cudaMalloc(&d, n * n * 8);
  cudaMalloc(&info, 4);
  cudaMallocManaged(&cyc, 8);
  for (int T : {16, 32, 50, 64}) {
    for (int chol = 0; chol < 2; ++chol) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
        cudaMemset(info, 0x7f, 4);
        if (chol) bench<true><<<1, 256>>>(d, n, T, info, cyc);
        else bench<false><<<1, 256>>>(d, n, T, info, cyc);
        cudaDeviceSynchronize();
      }
      printf("T=%d %s: %lld cycles (%.1f per pivot)\n", T, chol ? "potrf" : "getrf", cyc[0],
             (double)cyc[0] / T);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
