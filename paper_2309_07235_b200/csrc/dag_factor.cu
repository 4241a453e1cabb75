// Persistent tile-DAG LU / Cholesky (see dag_factor.cuh).
//
// Execution model: 1 CTA per SM, 8 warps.  Thread 0 takes the next task
// index with one atomicAdd, spins (ld.acquire.gpu) on the tile counters the
// task depends on, then the CTA runs it and every warp publishes the rows it
// finished with red.release.gpu.add on the output tile's counter.  Tasks
// are taken in list order and only ever wait on earlier tasks, so the
// schedule cannot deadlock whatever the number of resident CTAs.
//
// Counter protocol: cnt[i][j] counts finished rows of tile (i,j) summed over
// its stages.  Stage s < min(i,j) is the step-s trailing update, stage
// min(i,j) the final DIAG / TRSM; stage s of a tile is complete exactly when
// cnt >= (s+1) * T.  Every task sees its inputs through L2 (ld.global.cg), so
// no SM reads a stale L1 line of a tile another SM rewrote.
//
// Per element the arithmetic is fixed by the task list, independent of
// which CTA runs a task or when: repeated runs are bitwise identical
// (kernels_test.cpp:284-296).
#include <climits>

#include "dag_factor.cuh"
#include "diag_factor.cuh"
#include "tt_ptx.cuh"

namespace tt {
namespace dag {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMF = 2;            // 8-row DMMA blocks per warp strip
constexpr int kStrip = 8 * kMF;   // rows per warp strip
// Shared row stride (doubles) of the B / M tiles: == 4 (mod 16) so the DMMA
// B-fragment loads (lane g,t reads row 4s+t, column 8nf+g) hit every bank
// pair exactly twice — the 2-wavefront minimum for 256 bytes.
constexpr int kNP = 68;
constexpr int kNoLower = INT_MAX / 2;

struct Params {
  double* a;
  long long ld;
  int n, T, nt;
  const int4* tasks;
  int ntasks;
  int* cnt;    // nt*nt tile counters
  int* next;   // task counter
  int* abort;  // 1: numerical failure, 2: watchdog
  int* info;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread 0 only.  False when the schedule was aborted.
__device__ bool wait_ge(const Params& p, const int* addr, int need) {
  if (ld_acquire(addr) >= need) return true;
  const unsigned long long t0 = globaltimer();
  for (;;) {
    if (ld_acquire(addr) >= need) return true;
    if (*reinterpret_cast<volatile int*>(p.abort)) return false;
    if (globaltimer() - t0 > static_cast<unsigned long long>(kWatchdogNs)) {
      atomicExch(p.abort, 2);
      atomicMin(p.info, kTimeout);
      return false;
    }
  }
}

template <bool CHOL>
__device__ bool wait_deps(const Params& p, int4 tk) {
  const int kind = tk.x & 3, j = tk.x >> 2, k = tk.y, r0 = tk.z, r1 = tk.w;
  const int T = p.T, nt = p.nt, kT = k * T;
  const int* cnt = p.cnt;
  switch (kind) {
    case kDiag:  // stage k-1 of tile (k,k)
      return wait_ge(p, &cnt[k * nt + k], kT);
    case kTrsmL:  // stage k-1 of the row tiles, then DIAG(k)
      for (int i = r0 / T; i * T < r1; ++i)
        if (!wait_ge(p, &cnt[i * nt + k], kT)) return false;
      return wait_ge(p, &cnt[k * nt + k], kT + T);
    case kTrsmU:
      if (!wait_ge(p, &cnt[k * nt + j], kT)) return false;
      return wait_ge(p, &cnt[k * nt + k], kT + T);
    default:  // kGemm: stage k-1 of the output tiles, L(rows, k) and U(k, j) / L(j, k) final
      for (int i = r0 / T; i * T < r1; ++i) {
        if (!wait_ge(p, &cnt[i * nt + j], kT)) return false;
        if (!wait_ge(p, &cnt[i * nt + k], kT + T)) return false;
      }
      return wait_ge(p, CHOL ? &cnt[j * nt + k] : &cnt[k * nt + j], kT + T);
  }
}

// All lanes of a warp, after storing rows [ra, rb) of tile column j.
__device__ __forceinline__ void warp_signal(const Params& p, int ra, int rb, int j) {
  __threadfence();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    for (int i = ra / p.T; i * p.T < rb; ++i) {
      const int lo = max(ra, i * p.T), hi = min(rb, (i + 1) * p.T);
      red_release_add(&p.cnt[i * p.nt + j], hi - lo);
    }
  }
}

// ---------------------------------------------------------------- GEMM
// C[r, c] (r < nrows, c < T) -= sum_k A[r, k] * B[k, c]  with B (Kp x Tp,
// zero-padded) in shared memory; one warp, 16 rows, DMMA 8x8x4 atoms.
// Stores only where r + lower_off >= c (Cholesky diagonal tiles).
template <int NF>
__device__ __forceinline__ void warp_gemm(const double* __restrict__ A, long long lda,
                                          double* __restrict__ C, long long ldc, int nrows, int T,
                                          const double* __restrict__ Bs, int lower_off) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[kMF][NF][2];
  double af[kMF][2 * NF];
#pragma unroll
  for (int mf = 0; mf < kMF; ++mf) {
    const int r = mf * 8 + g;
    const bool rv = r < nrows;
    const double* crow = C + static_cast<long long>(rv ? r : 0) * ldc;
    const double* arow = A + static_cast<long long>(rv ? r : 0) * lda;
#pragma unroll
    for (int nf = 0; nf < NF; ++nf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = nf * 8 + 2 * t + h;
        acc[mf][nf][h] = (rv && c < T) ? __ldcg(crow + c) : 0.0;
      }
#pragma unroll
    for (int s = 0; s < 2 * NF; ++s) {
      const int kk = 4 * s + t;
      af[mf][s] = (rv && kk < T) ? -__ldcg(arow + kk) : 0.0;
    }
  }
#pragma unroll
  for (int s = 0; s < 2 * NF; ++s) {
    if (4 * s < T) {
      double b[NF];
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) b[nf] = Bs[(4 * s + t) * kNP + nf * 8 + g];
#pragma unroll
      for (int mf = 0; mf < kMF; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], af[mf][s], b[nf]);
    }
  }
#pragma unroll
  for (int mf = 0; mf < kMF; ++mf) {
    const int r = mf * 8 + g;
    if (r < nrows) {
      double* crow = C + static_cast<long long>(r) * ldc;
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = nf * 8 + 2 * t + h;
          if (c < T && r + lower_off >= c) crow[c] = acc[mf][nf][h];
        }
    }
  }
}

// ---------------------------------------------------------------- TRSM
// In place X * M = S for one 16-row strip: element (r, c) of S/X lives at
// base + r*rs + c*cs (rs = ld, cs = 1 for row strips; rs = 1, cs = ld for the
// transposed U12 solve).  M (Tp x Tp upper triangular, identity-padded) and
// the inverses of its 8x8 diagonal blocks are in shared memory.  Blocked by
// 8 columns: R_b = S_b - X_<b * M_<b,b (DMMA), X_b = R_b * inv(M_bb) (DMMA).
template <int NF>
__device__ __forceinline__ void warp_trsm(double* __restrict__ base, long long rs, long long cs,
                                          int nrows, int T, const double* __restrict__ Ms,
                                          const double* __restrict__ Minv) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double ra[NF][kMF][2];
#pragma unroll
  for (int mf = 0; mf < kMF; ++mf) {
    const int r = mf * 8 + g;
    const bool rv = r < nrows;
    const double* row = base + static_cast<long long>(rv ? r : 0) * rs;
#pragma unroll
    for (int b = 0; b < NF; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = b * 8 + 2 * t + h;
        ra[b][mf][h] = (rv && c < T) ? __ldcg(row + static_cast<long long>(c) * cs) : 0.0;
      }
  }
  // source lanes of the accumulator -> A-fragment relayout inside a quad:
  // A-layout k-step s needs column 4s + t, held by lane (g, 2s + t/2), half t&1.
  const int src0 = (lane & ~3) | (t >> 1), src1 = (lane & ~3) | (2 + (t >> 1));
  const bool odd = t & 1;
  double xa[NF][kMF][2];  // -X in A-fragment layout
#pragma unroll
  for (int b = 0; b < NF; ++b) {
    double acc[kMF][2];
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      acc[mf][0] = ra[b][mf][0];
      acc[mf][1] = ra[b][mf][1];
    }
#pragma unroll
    for (int bb = 0; bb < b; ++bb)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double m = Ms[(bb * 8 + 4 * s + t) * kNP + b * 8 + g];
#pragma unroll
        for (int mf = 0; mf < kMF; ++mf) dmma_8x8x4(acc[mf][0], acc[mf][1], xa[bb][mf][s], m);
      }
    double rf[kMF][2];
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const double v0 = __shfl_sync(0xffffffffu, acc[mf][0], src0);
      const double v1 = __shfl_sync(0xffffffffu, acc[mf][1], src0);
      const double w0 = __shfl_sync(0xffffffffu, acc[mf][0], src1);
      const double w1 = __shfl_sync(0xffffffffu, acc[mf][1], src1);
      rf[mf][0] = odd ? v1 : v0;
      rf[mf][1] = odd ? w1 : w0;
    }
    double xo[kMF][2] = {};
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double m = Minv[b * 64 + (4 * s + t) * 8 + g];
#pragma unroll
      for (int mf = 0; mf < kMF; ++mf) dmma_8x8x4(xo[mf][0], xo[mf][1], rf[mf][s], m);
    }
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const int r = mf * 8 + g;
      if (r < nrows) {
        double* row = base + static_cast<long long>(r) * rs;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = b * 8 + 2 * t + h;
          if (c < T) row[static_cast<long long>(c) * cs] = xo[mf][h];
        }
      }
    }
    if (b + 1 < NF) {
#pragma unroll
      for (int mf = 0; mf < kMF; ++mf) {
        const double v0 = __shfl_sync(0xffffffffu, xo[mf][0], src0);
        const double v1 = __shfl_sync(0xffffffffu, xo[mf][1], src0);
        const double w0 = __shfl_sync(0xffffffffu, xo[mf][0], src1);
        const double w1 = __shfl_sync(0xffffffffu, xo[mf][1], src1);
        xa[b][mf][0] = -(odd ? v1 : v0);
        xa[b][mf][1] = -(odd ? w1 : w0);
      }
    }
  }
}

// Inverse of the 8x8 upper-triangular diagonal block b of Ms (warp b,
// lanes 0..7 one column each, back substitution) into Minv[b] (row-major).
__device__ __forceinline__ void block_inverse8(const double* __restrict__ Ms, double* Minv, int b) {
  const int c = threadIdx.x & 31;
  if (c < 8) {
    const double* M = Ms + (b * 8) * kNP + b * 8;
    double x[8];
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int m = i + 1; m < 8; ++m) s -= M[i * kNP + m] * x[m];
      x[i] = s / M[i * kNP + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Minv[b * 64 + i * 8 + c] = x[i];
  }
}

// M for the solves, from the factored diagonal tile at `d` (leading dim ld):
//   upper = true : M = U11 (upper, incl. diagonal)                 LU  L21 solve
//   upper = false: M = L11^T (n > k from d[n][k]; unit or d[k][k])  LU U12 / Cholesky L21
__device__ __forceinline__ void load_m(double* Ms, const double* __restrict__ d, long long ld, int T,
                                       int Tp, bool upper, bool unit) {
  for (int e = threadIdx.x; e < Tp * Tp; e += kThreads) {
    int k, c;
    if (upper) {
      k = e / Tp;
      c = e - k * Tp;
    } else {  // read d row-contiguously: d[c][k]
      c = e / Tp;
      k = e - c * Tp;
    }
    double v;
    if (k >= T || c >= T) {
      v = (k == c) ? 1.0 : 0.0;
    } else if (c < k) {
      v = 0.0;
    } else if (c == k) {
      v = unit ? 1.0 : __ldcg(d + static_cast<long long>(k) * ld + k);
    } else {
      v = upper ? __ldcg(d + static_cast<long long>(k) * ld + c)
                : __ldcg(d + static_cast<long long>(c) * ld + k);
    }
    Ms[k * kNP + c] = v;
  }
}

// ---------------------------------------------------------------- kernel

template <int NF, bool CHOL>
__global__ void __launch_bounds__(kThreads, 1) dag_kernel(Params p) {
  constexpr int Tp = NF * 8;
  __shared__ __align__(16) double sm[kIB * diag::kLd > Tp * kNP ? kIB * diag::kLd : Tp * kNP];
  __shared__ __align__(16) double minv[8 * 64];
  __shared__ __align__(16) double buf[64];
  __shared__ int4 s_task;
  __shared__ int s_go;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int T = p.T, nt = p.nt;
  const long long ld = p.ld;

  for (;;) {
    if (tid == 0) {
      const int id = atomicAdd(p.next, 1);
      int4 tk = make_int4(-1, 0, 0, 0);
      if (id < p.ntasks) tk = p.tasks[id];
      s_task = tk;
      s_go = tk.x >= 0 && wait_deps<CHOL>(p, tk);
    }
    __syncthreads();
    if (!s_go) break;
    const int4 tk = s_task;
    const int kind = tk.x & 3, j = tk.x >> 2, k = tk.y, r0 = tk.z, r1 = tk.w;
    const int kT = k * T;
    double* dk = p.a + static_cast<long long>(kT) * ld + kT;  // diagonal tile (k,k)

    if (kind == kDiag) {
      double(*D)[diag::kLd] = reinterpret_cast<double(*)[diag::kLd]>(sm);
      for (int e = tid; e < T * T; e += kThreads) {
        const int i = e / T, c = e - i * T;
        D[i][c] = (!CHOL || c <= i) ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
      }
      __syncthreads();
      if (CHOL)
        diag::block_potrf(D, buf, T, kT, p.info, true);  // diag <= 0 fails, kernels.cpp:297-302
      else
        diag::block_getrf(D, buf, T, kT, p.info, true);  // |pivot| < 1e-300, kernels.cpp:187-190
      for (int e = tid; e < T * T; e += kThreads) {
        const int i = e / T, c = e - i * T;
        if (!CHOL || c <= i) dk[static_cast<long long>(i) * ld + c] = D[i][c];
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        if (diag::failed(p.info))
          atomicExch(p.abort, 1);
        else
          red_release_add(&p.cnt[k * nt + k], T);
      }
    } else if (kind == kGemm) {
      // B = U(k, j) (LU) or L(j, k)^T (Cholesky), zero-padded to Tp x Tp
      const double* bsrc = CHOL ? p.a + static_cast<long long>(j * T) * ld + kT
                                : p.a + static_cast<long long>(kT) * ld + j * T;
      for (int e = tid; e < Tp * Tp; e += kThreads) {
        const int x = e / Tp, y = e - x * Tp;  // x: slow index in memory order
        const double v = (x < T && y < T) ? __ldcg(bsrc + static_cast<long long>(x) * ld + y) : 0.0;
        if (CHOL)
          sm[y * kNP + x] = v;  // B[k][n] = L[n][k]
        else
          sm[x * kNP + y] = v;
      }
      __syncthreads();
      const int jT = j * T;
      for (int ra = r0 + warp * kStrip; ra < r1; ra += kWarps * kStrip) {
        const int nr = min(kStrip, r1 - ra);
        double* rowp = p.a + static_cast<long long>(ra) * ld;
        warp_gemm<NF>(rowp + kT, ld, rowp + jT, ld, nr, T, sm, CHOL ? ra - jT : kNoLower);
        warp_signal(p, ra, ra + nr, j);
      }
    } else {  // TRSM
      const bool lsolve = kind == kTrsmL;
      load_m(sm, dk, ld, T, Tp, !CHOL && lsolve, !CHOL && !lsolve);
      __syncthreads();
      if (warp < NF) block_inverse8(sm, minv, warp);
      __syncthreads();
      if (lsolve) {
        for (int ra = r0 + warp * kStrip; ra < r1; ra += kWarps * kStrip) {
          const int nr = min(kStrip, r1 - ra);
          warp_trsm<NF>(p.a + static_cast<long long>(ra) * ld + kT, ld, 1, nr, T, sm, minv);
          warp_signal(p, ra, ra + nr, k);
        }
      } else {  // U12 tile (k, j): strip rows are the tile's columns
        for (int c0 = warp * kStrip; c0 < T; c0 += kWarps * kStrip) {
          const int nc = min(kStrip, T - c0);
          warp_trsm<NF>(dk + static_cast<long long>(j - k) * T + c0, 1, ld, nc, T, sm, minv);
          __threadfence();
          __syncwarp();
          if ((tid & 31) == 0) red_release_add(&p.cnt[k * nt + j], nc);
        }
      }
    }
    __syncthreads();  // shared tiles are reused by the next task
  }
}

template <int NF, bool CHOL>
cudaError_t launch(const Params& prm, int grid, cudaStream_t s) {
  dag_kernel<NF, CHOL><<<grid, kThreads, 0, s>>>(prm);
  return cudaGetLastError();
}

template <bool CHOL>
cudaError_t launch_nf(int nf, const Params& prm, int grid, cudaStream_t s) {
  switch (nf) {
    case 1: return launch<1, CHOL>(prm, grid, s);
    case 2: return launch<2, CHOL>(prm, grid, s);
    case 3: return launch<3, CHOL>(prm, grid, s);
    case 4: return launch<4, CHOL>(prm, grid, s);
    case 5: return launch<5, CHOL>(prm, grid, s);
    case 6: return launch<6, CHOL>(prm, grid, s);
    case 7: return launch<7, CHOL>(prm, grid, s);
    case 8: return launch<8, CHOL>(prm, grid, s);
  }
  return cudaErrorInvalidValue;
}

long long count_tasks(bool chol, int n, int by, int bx) {
  const int nt = n / bx;
  long long total = 1;
  for (int k = 0; k + 1 < nt; ++k) {
    const int pe = (k + 1) * bx;
    const long long regions = (n - pe + by - 1) / by;
    const long long cols = nt - k - 1;
    total += regions + 1 + (chol ? 0 : cols) + regions * cols;
  }
  return total;
}

}  // namespace

bool eligible(int n, int by, int bx) {
  if (bx < kMinTile || bx > kMaxTile || n % bx || by < 1 || n % by) return false;
  return count_tasks(false, n, by, bx) <= kMaxTasks;
}

std::vector<int4> build_tasks(bool chol, int n, int by, int bx) {
  const int T = bx, nt = n / bx;
  std::vector<int4> v;
  v.reserve(static_cast<size_t>(count_tasks(chol, n, by, bx)));
  auto task = [&](int kind, int k, int r0, int r1, int j) {
    v.push_back(make_int4(kind | (j << 2), k, r0, r1));
  };
  task(kDiag, 0, 0, T, 0);
  for (int k = 0; k + 1 < nt; ++k) {
    const int pe = (k + 1) * T;
    std::vector<std::pair<int, int>> reg;
    for (int r = pe; r < n; r += by) reg.emplace_back(r, std::min(n, r + by));
    auto gemm = [&](size_t ri, int j) {
      int r0 = reg[ri].first;
      const int r1 = reg[ri].second;
      if (chol) r0 = std::max(r0, j * T);  // lower triangle only
      if (r0 < r1) task(kGemm, k, r0, r1, j);
    };
    // critical chain of step k -> DIAG(k+1): first solves, column k+1
    task(kTrsmL, k, reg[0].first, reg[0].second, 0);
    if (!chol) task(kTrsmU, k, 0, 0, k + 1);
    for (size_t ri = 1; ri < reg.size(); ++ri) task(kTrsmL, k, reg[ri].first, reg[ri].second, 0);
    for (size_t ri = 0; ri < reg.size(); ++ri) gemm(ri, k + 1);
    task(kDiag, k + 1, 0, T, 0);  // look-ahead: overlaps the rest of step k
    if (!chol)
      for (int j = k + 2; j < nt; ++j) task(kTrsmU, k, 0, 0, j);
    for (int j = k + 2; j < nt; ++j)
      for (size_t ri = 0; ri < reg.size(); ++ri) gemm(ri, j);
  }
  return v;
}

cudaError_t create(Workspace* w, bool chol, int n, int by, int bx) {
  const std::vector<int4> tasks = build_tasks(chol, n, by, bx);
  const int nt = n / bx;
  w->ntasks = static_cast<int>(tasks.size());
  w->cnt_bytes = (static_cast<size_t>(nt) * nt + 2) * sizeof(int);
  cudaError_t e = cudaMalloc(&w->tasks, tasks.size() * sizeof(int4));
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(w->tasks, tasks.data(), tasks.size() * sizeof(int4), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&w->cnt, w->cnt_bytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  w->grid = std::max(1, std::min(sms, w->ntasks));
  return cudaSuccess;
}

void destroy(Workspace* w) {
  if (w->tasks) cudaFree(w->tasks);
  if (w->cnt) cudaFree(w->cnt);
  *w = Workspace{};
}

cudaError_t enqueue(const Workspace& w, bool chol, double* a, int n, long long ld, int bx,
                    int* info, cudaStream_t s) {
  const int nt = n / bx;
  cudaError_t e = cudaMemsetAsync(w.cnt, 0, w.cnt_bytes, s);
  if (e != cudaSuccess) return e;
  Params prm;
  prm.a = a;
  prm.ld = ld;
  prm.n = n;
  prm.T = bx;
  prm.nt = nt;
  prm.tasks = w.tasks;
  prm.ntasks = w.ntasks;
  prm.cnt = w.cnt;
  prm.next = w.cnt + static_cast<size_t>(nt) * nt;
  prm.abort = prm.next + 1;
  prm.info = info;
  const int nf = (bx + 7) / 8;
  return chol ? launch_nf<true>(nf, prm, w.grid, s) : launch_nf<false>(nf, prm, w.grid, s);
}

}  // namespace dag
}  // namespace tt
