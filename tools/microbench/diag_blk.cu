#include <cstdio>
#include <vector>
#include "../../paper_2309_07235_b200/csrc/dag_factor.cu"
namespace tt { namespace dag { namespace {
template <bool CHOL>
__device__ __forceinline__ void tfb_stamped(double* __restrict__ dk, long long ld, int T,
                                                    int gcol, int* info, double* D, double* inv,
                                                    double* rk, unsigned long long* ph,
                                                    double* solve, long long* st) {
  // inv: [0,64) inv(U_bb) row-major, [64,128) inv(L_bb); rk: 64 reciprocals of u_jj
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int NB = (T + 7) >> 3, Tp = NB * 8;
  {  // load (Cholesky: mirror the lower triangle), identity padding
    constexpr int kPer = 64 * 64 / kThreads;
    double v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kThreads, i = e >> 6, c = e & 63;
      const int si = (CHOL && c > i) ? c : i, sc = (CHOL && c > i) ? i : c;
      v[u] = (i < T && c < T) ? __ldcg(dk + static_cast<long long>(si) * ld + sc)
                              : (i == c ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kThreads;
      D[(e >> 6) * kNP + (e & 63)] = v[u];
    }
  }
  __syncthreads();
  if (ph && tid == 0) ph[0] = globaltimer();
  for (int b = 0; b < NB; ++b) {
    const int p = 8 * b;
    if (tid == 0) st[b * 6 + 0] = clock64();
    if (warp == 0) {
      __syncwarp();  // converged warp: keeps the shuffles on the fast (non-divergent) path
      // ---- 8x8 diagonal block, lane (g,t) holds (g, 2t), (g, 2t+1)
      double v0 = D[(p + g) * kNP + p + 2 * t], v1 = D[(p + g) * kNP + p + 2 * t + 1];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const double sel = (kk & 1) ? v1 : v0;
        const double piv = __shfl_sync(0xffffffffu, sel, kk * 4 + (kk >> 1));
        const double agk = __shfl_sync(0xffffffffu, sel, g * 4 + (kk >> 1));
        const double u0 = __shfl_sync(0xffffffffu, v0, kk * 4 + t);
        const double u1 = __shfl_sync(0xffffffffu, v1, kk * 4 + t);
        const double r = rcp_nr(piv);
        const double m = g > kk ? agk * r : 0.0;
        if (2 * t > kk) v0 = fma(-m, u0, v0);
        if (2 * t + 1 > kk) v1 = fma(-m, u1, v1);
        if (g > kk && 2 * t == kk) v0 = m;
        if (g > kk && 2 * t + 1 == kk) v1 = m;
        if (lane == 0 && p + kk < T) {
          rk[p + kk] = r;
          if (CHOL ? !(piv > 0.0) && piv == piv : fabs(piv) < 1e-300)
            atomicMin(info, gcol + p + kk);  // kernels.cpp:187-190 / :297-302
        }
      }
      D[(p + g) * kNP + p + 2 * t] = v0;
      D[(p + g) * kNP + p + 2 * t + 1] = v1;
      if (tid == 0) st[b * 6 + 1] = clock64() + (long long)(v0 * 0.0);
      __syncwarp();
      // inv(U_bb): lanes 0..7 (column c); inv(L_bb) (unit lower): lanes 8..15.
      // The block is preloaded into registers (independent loads), then the
      // column is solved in axpy form: one dependent FMA per step.
      if (lane < 16) {
        const int c = lane & 7;
        const bool up = lane < 8;
        double m8[8][8];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii)
#pragma unroll
          for (int mm = 0; mm < 8; ++mm) m8[ii][mm] = D[(p + ii) * kNP + p + mm];
        double rr[8];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) rr[ii] = p + ii < T ? rk[p + ii] : 1.0;
        double x[8];
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) x[ii] = ii == c ? 1.0 : 0.0;
        if (up) {  // U X = I, columns: x_kk final -> subtract from rows above
#pragma unroll
          for (int kk = 7; kk >= 0; --kk) {
            x[kk] *= rr[kk];
#pragma unroll
            for (int ii = 0; ii < kk; ++ii) x[ii] = fma(-m8[ii][kk], x[kk], x[ii]);
          }
        } else {  // L X = I (unit): x_kk final -> subtract from rows below
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
#pragma unroll
            for (int ii = kk + 1; ii < 8; ++ii) x[ii] = fma(-m8[ii][kk], x[kk], x[ii]);
        }
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) inv[(up ? 0 : 64) + ii * 8 + c] = x[ii];
      }
    }
    if (tid == 0) st[b * 6 + 2] = clock64();
    __syncthreads();
    if (tid == 0) st[b * 6 + 3] = clock64();
    const int nr = NB - b - 1;  // blocks beyond the diagonal one
    if (nr == 0) break;
    // ---- panels: job < nr: L block (b+1+job, b) = A * inv(U_bb);
    //               job >= nr: U block (b, b+1+job-nr) = inv(L_bb) * A
    for (int job = warp; job < 2 * nr; job += kWarps) {
      double c0 = 0.0, c1 = 0.0;
      if (job < nr) {
        const int rb = 8 * (b + 1 + job);
        const double a0 = D[(rb + g) * kNP + p + t], a1 = D[(rb + g) * kNP + p + 4 + t];
        const double b0 = inv[t * 8 + g], b1 = inv[(4 + t) * 8 + g];
        dmma_8x8x4(c0, c1, a0, b0);
        dmma_8x8x4(c0, c1, a1, b1);
        __syncwarp();
        D[(rb + g) * kNP + p + 2 * t] = c0;
        D[(rb + g) * kNP + p + 2 * t + 1] = c1;
      } else {
        const int cb = 8 * (b + 1 + job - nr);
        const double a0 = inv[64 + g * 8 + t], a1 = inv[64 + g * 8 + 4 + t];
        const double b0 = D[(p + t) * kNP + cb + g], b1 = D[(p + 4 + t) * kNP + cb + g];
        dmma_8x8x4(c0, c1, a0, b0);
        dmma_8x8x4(c0, c1, a1, b1);
        __syncwarp();
        D[(p + g) * kNP + cb + 2 * t] = c0;
        D[(p + g) * kNP + cb + 2 * t + 1] = c1;
      }
    }
    __syncthreads();
    if (tid == 0) st[b * 6 + 4] = clock64();
    // ---- trailing update: block (ib, jb) -= L(ib, b) * U(b, jb)
    for (int job = warp; job < nr * nr; job += kWarps) {
      const int ib = 8 * (b + 1 + job / nr), jb = 8 * (b + 1 + job % nr);
      double c0 = D[(ib + g) * kNP + jb + 2 * t], c1 = D[(ib + g) * kNP + jb + 2 * t + 1];
      const double a0 = -D[(ib + g) * kNP + p + t], a1 = -D[(ib + g) * kNP + p + 4 + t];
      const double b0 = D[(p + t) * kNP + jb + g], b1 = D[(p + 4 + t) * kNP + jb + g];
      dmma_8x8x4(c0, c1, a0, b0);
      dmma_8x8x4(c0, c1, a1, b1);
      D[(ib + g) * kNP + jb + 2 * t] = c0;
      D[(ib + g) * kNP + jb + 2 * t + 1] = c1;
    }
    __syncthreads();
    if (tid == 0) st[b * 6 + 5] = clock64();
  }
  if (ph && tid == 0) ph[1] = globaltimer();
  // Cholesky: l_jj = sqrt(u_jj), 1/l_jj for the solves
  if (CHOL && tid < T) {
    const double l = sqrt(D[tid * kNP + tid]);
    rk[64 + tid] = l;
    rk[tid] = rcp_nr(l);
  }
  if (CHOL) __syncthreads();
  {  // store the factored tile (Cholesky: lower only, scaled)
    constexpr int kPer = 64 * 64 / kThreads;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kThreads, i = e >> 6, c = e & 63;
      if (i < T && c < T && (!CHOL || c <= i)) {
        double v = D[i * kNP + c];
        if (CHOL) v = c == i ? rk[64 + c] : v * rk[64 + c];
        dk[static_cast<long long>(i) * ld + c] = v;
      }
    }
  }
  if (tid < 64) solve[tid] = rk[tid];
  (void)Tp;
}


} } }
__global__ void __launch_bounds__(256, 1) bench(double* a, long long ld, int T, int* info, long long* st) {
  __shared__ __align__(16) double D[64 * 68]; __shared__ double inv[264]; __shared__ double rk[128]; __shared__ double slv[64];
  tt::dag::tfb_stamped<false>(a, ld, T, 0, info, D, inv, rk, nullptr, slv, st);
}
int main() {
  const int n = 64; std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double* d; int* info; long long* st; cudaMalloc(&d, n*n*8); cudaMalloc(&info, 4); cudaMallocManaged(&st, 64*8);
  for (int r = 0; r < 2; ++r) { cudaMemcpy(d, h.data(), n*n*8, cudaMemcpyHostToDevice); cudaMemset(info, 0x7f, 4); bench<<<1,256>>>(d, n, 50, info, st); cudaDeviceSynchronize(); }
  for (int b = 0; b < 7; ++b) printf("b=%d diag8x8 %lld inverses %lld bar %lld panels+bar %lld trailing+bar %lld | next %lld\n", b,
     st[b*6+1]-st[b*6+0], st[b*6+2]-st[b*6+1], st[b*6+3]-st[b*6+2], st[b*6+4]-st[b*6+3], st[b*6+5]-st[b*6+4], b < 6 ? st[(b+1)*6]-st[b*6+5] : 0);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
