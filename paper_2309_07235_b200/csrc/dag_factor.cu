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
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "dag_factor.cuh"
#include "devattr.hpp"
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
constexpr int kSmemB = kIB * kNP;                // one walker tile / the TRSM M tile
// single-step GEMM tasks: per-warp double-buffered A strips (16 rows x <= 66
// columns, row stride kAW == 4 mod 16: conflict-free A-fragment loads)
// staged by cp.async.cg after the B tile
constexpr int kAW = 68;
constexpr int kABuf = kStrip * kAW;              // doubles per buffer
constexpr int kSmemA = kWarps * 2 * kABuf;       // all warps' A buffers
// walker-only: DIAG block inverses (1024) + the U12-solve block inverses (512)
constexpr int kSmemW = 1536;
// walker: tiles D, L(k+1,k), U(k,k+1), the reciprocals rk (128), the inverses
// and the prefetch buffer of the next diagonal tile
constexpr int kWalkerSmem = 4 * kSmemB + 128 + kSmemW;
// Dynamic shared memory of every CTA (one CTA per SM): the walker's tiles, a
// queue CTA's TRSM tile + block inverses, or a GEMM task's q stacked B tiles.
constexpr int kSmemBytes = 224 * 1024;
constexpr int kBudget = kSmemBytes / 8;  // doubles
static_assert(kWalkerSmem <= kBudget, "walker tiles exceed shared memory");
static_assert(kSmemB + kSmemA <= kBudget, "single-step GEMM staging exceeds shared memory");
// Row strides (doubles) of the staged GEMM B tiles.  LU stages B[k][n] and
// loads fragments with 8-byte loads (lanes t and t+1 two rows apart): a stride
// == 4 (mod 8) puts them on opposite bank halves, the 2-wavefront minimum.
// Cholesky stages B^T[n][k] and loads both k-halves of a permuted fragment
// with one 16-byte load: == 8 (mod 16) keeps each 8-lane phase conflict-free.
__host__ __device__ constexpr int bstride(int tp, bool chol) {
  return chol ? (tp % 16 == 8 ? tp : tp + 8) : tp + 4;
}
constexpr int kSolveSlot = 64;  // per step: diagonal reciprocals written by DIAG

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

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
  unsigned long long* trace;  // optional: per task {fetch, ready, done ns, smid, 4 phase stamps}
  double* solve;  // per step: 64 reciprocals of the factored diagonal (DIAG -> TRSM)
  int nurgent;    // tasks[0, nurgent): urgent queue; [nurgent, ntasks): bulk queue
  int nuw;        // CTAs 1..nuw serve the urgent queue
  int d;          // chunk depth (dag_factor.cuh)
  int eager_sig;  // publish GEMM strips right after their stores: 0 no, 1 all, 2 urgent, 3 bulk
  int fence;      // TT_DAG_FENCE=1: gpu-scope fence after each task's dependency wait
  int pipe;       // GEMM tasks through gemm_pipe (TT_DAG_PIPE=0: the register path)
  int nodeps;     // TT_DAG_NODEPS=1 (measurement aid): every counter starts satisfied and
                  // no walker runs — the queues' task throughput alone, numerics void
  int wide;       // bulk GEMM tasks with T <= 40 run 32-row strips (TT_DAG_WIDE=0: off)
  int pf_mask;    // bit 0: urgent CTAs, bit 1: bulk CTAs fetch the next task before
                  // the current one's dependency wait (else when warp 0 finishes it)
};


__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Acquire load (LDG.STRONG.GPU + L1 invalidate; unlike fence.acq_rel it does
// not wait for this thread's outstanding loads and stores, so prefetches
// stay in flight across a dependency check).
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spins (acquire gpu-scope loads, with a short back-off so waiting CTAs do
// not hammer the counter's L2 slice) until *addr >= need.  False when the
// schedule was aborted.
__device__ bool wait_ge(const Params& p, const int* addr, int need) {
  if (ld_acquire(addr) < need) {
    const unsigned long long t0 = globaltimer();
    for (int it = 0;; ++it) {
      __nanosleep(100);
      if (ld_acquire(addr) >= need) break;
      if ((it & 15) == 15) {
        if (ld_relaxed(p.abort)) return false;
        // timeout = 4 s of %globaltimer AND >= 2^20 polls (each >= 100 ns of
        // sleep), so one anomalous timer reading cannot abort a healthy
        // schedule (long sweeps once reported a timeout whose record showed
        // no progress at all)
        const long long dt = static_cast<long long>(globaltimer() - t0);
        if (it >= (1 << 20) && dt > kWatchdogNs) {
          // first expiring waiter records what it waited for (diagnostics:
          // CTA, counter index, target, last value seen)
          if (atomicCAS(p.abort + 3, 0, 1) == 0) {
            p.abort[4] = blockIdx.x;
            p.abort[5] = static_cast<int>(addr - p.cnt);
            p.abort[6] = need;
            p.abort[7] = ld_relaxed(addr);
            p.abort[8] = ld_relaxed(p.next);      // urgent queue position
            p.abort[9] = ld_relaxed(p.next + 2);  // bulk queue position
            p.abort[10] = it;                         // polls
            p.abort[11] = static_cast<int>(dt / 1000000);  // ms waited
            p.abort[12] = ld_relaxed(p.abort + 2);    // CTAs of this launch that started
            p.abort[13] = gridDim.x;
          }
          atomicExch(p.abort, 2);
          atomicMin(p.info, kTimeout);
          return false;
        }
      }
    }
  }
  return true;
}

// Counter targets (finished rows) under the chunked stage numbering
// (dag_factor.cuh): tile (i, col), m = min(i, col) updates, has finished the
// stages covering the steps < s, resp. is final.
__device__ __forceinline__ int need_before(const Params& p, int m, int col, int s) {
  return stages_before(m, s, p.d, col % p.d) * p.T;
}
__device__ __forceinline__ int need_final(const Params& p, int m, int col) {
  return stages_total(m, p.d, col % p.d) * p.T;
}

// Task-level dependencies: what the whole CTA reads (the diagonal tile, the
// B operand).  Row-strip dependencies (the strip's own output tiles and its
// L rows) are waited for per strip by the warp that processes it, so a
// task's first strips start as soon as their rows are ready (dataflow along
// the rows: DIAG(k) -> first TRSM_L strips -> first GEMM strips -> DIAG(k+1)).
// A GEMM over steps [k0, kl] waits only for the operands of step kl: U(kl, j)
// final implies tile (kl, j) received the step kl-1 update, whose operand
// U(kl-1, j) was therefore final (and so on down to k0); the same holds for
// L(i, kl) / L(j, kl).  Acquire/release is transitive, so the chain makes the
// earlier tiles visible as well.
__device__ __forceinline__ int dep_count(int kind) { return kind == kTrsmU ? 2 : 1; }

template <bool CHOL>
__device__ __forceinline__ void dep_at(const Params& p, int kind, int j, int k, int d, int* idx,
                                       int* need) {
  const int nt = p.nt;
  switch (kind) {
    case kTrsmL:  // DIAG(k)
      *idx = k * nt + k;
      *need = need_final(p, k, k);
      return;
    case kTrsmU:  // every update of tile (k,j), DIAG(k)
      *idx = d == 0 ? k * nt + j : k * nt + k;
      *need = d == 0 ? need_before(p, k, j, k) : need_final(p, k, k);
      return;
    default:  // kGemm over steps [k0, k]: B operand U(k, j) / L(j, k) final
      *idx = CHOL ? j * nt + k : k * nt + j;
      *need = need_final(p, k, CHOL ? k : j);
  }
}

// Task word: {kind | j << 2, k0 | q << 16, r0, r1}.
__device__ __forceinline__ int task_k0(int4 tk) { return tk.y & 0xFFFF; }
__device__ __forceinline__ int task_q(int4 tk) { return max(1, tk.y >> 16); }

template <bool CHOL>
__device__ bool wait_deps(const Params& p, int4 tk) {
  const int kind = tk.x & 3, j = tk.x >> 2;
  const int k = kind == kGemm ? task_k0(tk) + task_q(tk) - 1 : task_k0(tk);
  const int nd = dep_count(kind);
  bool ok = true;
  const int d = threadIdx.x & 31;
  if (d < nd) {
    int idx, need;
    dep_at<CHOL>(p, kind, j, k, d, &idx, &need);
    ok = wait_ge(p, &p.cnt[idx], need);
  }
  return __all_sync(0xffffffffu, ok);
}

// Row-strip dependencies of rows [rs, re) writing tile column `col` with the
// stage that starts at step s: the output tiles' earlier stages, and (kl >= 0,
// GEMM) the L tiles (i, kl) final.  Lane d of the calling warp takes
// dependency d.  With `block` false this is a single poll (true only if
// everything is already satisfied).
__device__ __forceinline__ bool strip_deps(const Params& p, int rs, int re, int col, int s,
                                           int kl, bool block) {
  const int T = p.T, nt = p.nt;
  const int ti0 = rs / T, nti = (re - 1) / T - ti0 + 1;
  const int d = threadIdx.x & 31;
  bool ok = true;
  if (d < (kl >= 0 ? 2 * nti : nti)) {
    const int i = ti0 + (d < nti ? d : d - nti);
    const int* c = &p.cnt[i * nt + (d < nti ? col : kl)];
    const int need = d < nti ? need_before(p, min(i, col), col, s) : need_final(p, kl, kl);
    if (block) {
      ok = wait_ge(p, c, need);
    } else {
      ok = ld_acquire(c) >= need;
    }
  }
  return __all_sync(0xffffffffu, ok);
}

// All lanes of a warp, after storing rows [ra, rb) of tile column j.  The
// warp barrier orders every lane's stores before lane 0's release reduction
// (release is cumulative), so no per-lane fence.
__device__ __forceinline__ void warp_signal(const Params& p, int ra, int rb, int j) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    for (int i = ra / p.T; i * p.T < rb; ++i) {
      const int lo = max(ra, i * p.T), hi = min(rb, (i + 1) * p.T);
      red_release_add(&p.cnt[i * p.nt + j], hi - lo);
    }
  }
}


// ---------------------------------------------------------------- GEMM
// ---- single-step tasks (q = 1, K = T): the near-diagonal band.
// One warp's share: C[r, c] -= sum_k A[r, k] * B[k, c] over the 16-row strips
// ra = r0 + 16*warp, +128, ... of rows [r0, r1).  B (Tp x Tp, zero-padded) is
// in shared memory.  Software pipeline per strip: the next strip's A
// (cp.async.cg into the warp's other buffer, L2 only) and C (registers) are
// in flight while this strip's DMMAs run — with one step per strip the strip
// round trip, not the DMMA work, is what a strip costs.  Stores only where
// row + lower_off >= col (Cholesky diagonal tiles).
// Operands of a strip task: rows r of [r0, r1) (global rows: tile counters)
// read A from A0 + (r - r0)*lda (T columns) and update C at C0 + (r - r0)*ldc
// (T columns of tile column cj); beta = 0 starts from zero instead of C.
// Dependencies per strip: stage k-1 of the C tiles, plus (gemm) the L tiles
// (i, k) final.  The product accumulated is C - A*B.
struct StripOps {
  const double* A0;
  long long lda;
  double* C0;
  long long ldc;
  int cj;      // tile column of C (counters)
  bool gemm;   // also wait for L(i,k) final
  bool beta;   // load C
  bool eager;  // publish each strip right after its stores (else one strip later)
};

template <int NF>
__device__ __forceinline__ void gemm_strips(const Params& p, int r0, int r1, int k,
                                            const StripOps& op,
                                            const double* __restrict__ Bs, double* abuf,
                                            bool chol, unsigned long long* first_done) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  const int T = p.T, j = op.cj;
  const int jT = j * T;
  // 16-byte aligned copy origin (lda even: every row has the same parity)
  const int sh = static_cast<int>((reinterpret_cast<uintptr_t>(op.A0) >> 3) & 1);
  const int nvec = (T + sh + 1) >> 1;  // 16-byte vectors per row
  int ra = r0 + warp * kStrip;
  if (ra >= r1) return;

  auto issue_a = [&](int rs, double* buf) {
    const int nr = min(kStrip, r1 - rs);
    const double* src = op.A0 - sh + static_cast<long long>(rs - r0) * op.lda;
    for (int e = lane; e < nr * nvec; e += 32) {
      const int r = e / nvec, v = e - r * nvec;
      cp_async16(buf + r * kAW + 2 * v, src + static_cast<long long>(r) * op.lda + 2 * v);
    }
    cp_async_commit();
  };
  // C element pairs (2t, 2t+1) as one 16-byte load/store when every row of
  // the strip starts 16-byte aligned and T is even (half the LSU requests of
  // 8-byte accesses: the strip's operand round trip is bound by them)
  const bool cvec = ((reinterpret_cast<uintptr_t>(op.C0) & 15) == 0) && !(op.ldc & 1) && !(T & 1);
  auto load_c = [&](int rs, double (&cv)[kMF][NF][2]) {
    const int nr = min(kStrip, r1 - rs);
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const int r = mf * 8 + g;
      const bool rv = r < nr;
      const double* crow = op.C0 + static_cast<long long>(rs - r0 + (rv ? r : 0)) * op.ldc;
      if (cvec) {
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          const int c = nf * 8 + 2 * t;
          double2 v = make_double2(0.0, 0.0);
          if (op.beta && rv && c < T) v = __ldcg(reinterpret_cast<const double2*>(crow + c));
          cv[mf][nf][0] = v.x;
          cv[mf][nf][1] = v.y;
        }
      } else {
#pragma unroll
        for (int nf = 0; nf < NF; ++nf)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = nf * 8 + 2 * t + h;
            cv[mf][nf][h] = (op.beta && rv && c < T) ? __ldcg(crow + c) : 0.0;
          }
      }
    }
  };

  double acc[kMF][NF][2];
  int prev_ra = -1, prev_nr = 0;
  if (!strip_deps(p, ra, min(ra + kStrip, r1), j, k, op.gemm ? k : -1, true)) return;
  if (first_done && lane == 0) first_done[2] = globaltimer();  // first strip's inputs final
  issue_a(ra, abuf);
  load_c(ra, acc);
  int cur = 0;
  for (;;) {
    const int rn = ra + kWarps * kStrip;
    const bool more = rn < r1;
    double cn[kMF][NF][2];
    // prefetch the next strip now if its rows are already final, else after this one
    const bool pref = more && strip_deps(p, rn, min(rn + kStrip, r1), j, k, op.gemm ? k : -1, false);
    if (pref) {
      issue_a(rn, abuf + (cur ^ 1) * kABuf);
      load_c(rn, cn);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    if (first_done && lane == 0) first_done[1] = globaltimer();
    const int nr = min(kStrip, r1 - ra);
    const double* ab = abuf + cur * kABuf + sh;
#pragma unroll
    for (int s = 0; s < 2 * NF; ++s) {
      if (4 * s < T) {
        const int kk = 4 * s + t;
        double af[kMF];
#pragma unroll
        for (int mf = 0; mf < kMF; ++mf) {
          const int r = mf * 8 + g;
          af[mf] = (r < nr && kk < T) ? -ab[r * kAW + kk] : 0.0;
        }
        double bf[NF];
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) bf[nf] = Bs[kk * kNP + nf * 8 + g];
#pragma unroll
        for (int mf = 0; mf < kMF; ++mf)
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], af[mf], bf[nf]);
      }
    }
    // publish the previous strip now: its stores were issued a whole strip
    // ago, so the fence does not stall on their acknowledgement
    if (prev_ra >= 0 && !op.eager) warp_signal(p, prev_ra, prev_ra + prev_nr, j);
    const int lower_off = chol ? ra - jT : kNoLower;
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const int r = mf * 8 + g;
      if (r < nr) {
        double* crow = op.C0 + static_cast<long long>(ra - r0 + r) * op.ldc;
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          const int c = nf * 8 + 2 * t;
          const bool ok0 = c < T && r + lower_off >= c, ok1 = c + 1 < T && r + lower_off >= c + 1;
          if (cvec && ok0 && ok1) {
            *reinterpret_cast<double2*>(crow + c) = make_double2(acc[mf][nf][0], acc[mf][nf][1]);
          } else {
            if (ok0) crow[c] = acc[mf][nf][0];
            if (ok1) crow[c + 1] = acc[mf][nf][1];
          }
        }
      }
    }
    if (op.eager) {
      warp_signal(p, ra, ra + nr, j);  // publish this strip right away
      prev_ra = -1;
    } else {
      prev_ra = ra;
      prev_nr = nr;
    }
    if (first_done && lane == 0) {
      *first_done = globaltimer();
      first_done = nullptr;
    }
    if (!more) break;
    if (!pref) {
      if (!strip_deps(p, rn, min(rn + kStrip, r1), j, k, op.gemm ? k : -1, true)) return;  // aborted
      issue_a(rn, abuf + (cur ^ 1) * kABuf);
      load_c(rn, cn);
    }
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        acc[mf][nf][0] = cn[mf][nf][0];
        acc[mf][nf][1] = cn[mf][nf][1];
      }
    ra = rn;
    cur ^= 1;
  }
  if (prev_ra >= 0) warp_signal(p, prev_ra, prev_ra + prev_nr, j);
}


// ---- chunked tasks (q > 1):
// C(rows, j) -= sum_{k in [k0, k0+q)} L(rows, k) * B_k,  B_k = U(k, j) (LU) or
// L(j, k)^T (Cholesky), K = q*T.
//
// The q B tiles are staged once per task into shared memory (16-byte
// cp.async of matrix rows, zero-filled padding).  Each warp takes 16-row
// strips; a strip keeps -C in registers over all q steps and reads the L
// rows straight from L2 into DMMA A fragments with 16-byte loads, the next
// step's fragments in flight while the current step's DMMAs run.  The k index
// inside every 8-wide block is permuted so a lane's two A values are
// adjacent in memory: lane (g, t) supplies k = 8s + 2t + h for half h of the
// k-block pair — the B fragments use the same permutation, so each DMMA still
// forms a 4-term slice of the same dot product.  Accumulating into -C and
// negating once per strip keeps every DMMA in its natural D = A*B + C form;
// the values are exactly those of C + (-A)*B.
__device__ __forceinline__ double negd(double x) {  // sign flip on the integer pipe
  return __longlong_as_double(__double_as_longlong(x) ^ static_cast<long long>(0x8000000000000000ULL));
}

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}

// Stages B_k for k in [k0, k0+q) as q zero-padded Tp x Tp tiles of matrix
// rows: LU  Bs[kk][x][y] = A[(k0+kk)T + x][jT + y]  (x = k index, y = n),
//       Cholesky Bs[kk][y][x] = A[jT + y][(k0+kk)T + x]  (y = n, x = k).
template <int NF, bool CHOL>
__device__ __forceinline__ void stage_b(const Params& p, double* Bs, int j, int k0, int q) {
  constexpr int Tp = NF * 8, NPB = bstride(Tp, CHOL), HP = Tp / 2;
  const int T = p.T;
  const long long ld = p.ld;
  const int total = q * Tp * HP;  // element pairs
  for (int e = threadIdx.x; e < total; e += kThreads) {
    const int kk = e / (Tp * HP), rem = e - kk * (Tp * HP), x = rem / HP, y = 2 * (rem - x * HP);
    const int k = k0 + kk;
    const long long row = CHOL ? static_cast<long long>(j) * T + x : static_cast<long long>(k) * T + x;
    const long long col = CHOL ? static_cast<long long>(k) * T + y : static_cast<long long>(j) * T + y;
    const double* src = p.a + row * ld + col;
    double* dst = Bs + kk * Tp * NPB + x * NPB + y;
    if (!(T & 1)) {
      const bool valid = x < T && y < T;
      cp_async16_zfill(dst, valid ? src : p.a, valid);
    } else {  // odd T: rows are not 16-byte aligned
      dst[0] = (x < T && y < T) ? __ldcg(src) : 0.0;
      dst[1] = (x < T && y + 1 < T) ? __ldcg(src + 1) : 0.0;
    }
  }
  if (!(T & 1)) {
    cp_async_commit();
    cp_async_wait<0>();
  }
}

template <int NF, bool CHOL>
__device__ void gemm_task(const Params& p, int j, int k0, int q, int r0, int r1,
                          const double* __restrict__ Bs, bool eager,
                          unsigned long long* first_done) {
  constexpr int Tp = NF * 8, NPB = bstride(Tp, CHOL);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  const int T = p.T;
  const long long ld = p.ld;
  const int kl = k0 + q - 1, jT = j * T;
  const bool even = !(T & 1);  // element pairs of the L rows / C rows are 16-byte aligned

  // A fragments of step k for the strip at rows ra: a[mf][s].x / .y = L(r, 8s+2t) / (8s+2t+1)
  auto load_a = [&](double2 (&a)[kMF][NF], int ra, int nr, int k) {
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const int r = mf * 8 + g;
      const double* row = p.a + static_cast<long long>(ra + (r < nr ? r : 0)) * ld +
                          static_cast<long long>(k) * T;
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        const int c = 8 * s + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (r < nr) {
          if (even) {
            if (c < T) v = __ldcg(reinterpret_cast<const double2*>(row + c));
          } else {
            if (c < T) v.x = __ldcg(row + c);
            if (c + 1 < T) v.y = __ldcg(row + c + 1);
          }
        }
        a[mf][s] = v;
      }
    }
  };
  const bool cvec = even;  // C rows: same alignment argument (ld even, jT even)
  int prev_ra = -1, prev_nr = 0;
  for (int ra = r0 + warp * kStrip; ra < r1; ra += kWarps * kStrip) {
    const int nr = min(kStrip, r1 - ra);
    if (!strip_deps(p, ra, ra + nr, j, k0, kl, true)) return;  // aborted
    if (first_done && lane == 0) first_done[2] = globaltimer();
    double acc[kMF][NF][2];  // -C
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const int r = mf * 8 + g;
      const double* crow = p.a + static_cast<long long>(ra + (r < nr ? r : 0)) * ld + jT;
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) {
        const int c = nf * 8 + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (r < nr) {
          if (cvec) {
            if (c < T) v = __ldcg(reinterpret_cast<const double2*>(crow + c));
          } else {
            if (c < T) v.x = __ldcg(crow + c);
            if (c + 1 < T) v.y = __ldcg(crow + c + 1);
          }
        }
        acc[mf][nf][0] = negd(v.x);
        acc[mf][nf][1] = negd(v.y);
      }
    }
    double2 a[kMF][NF];
    load_a(a, ra, nr, k0);
    // Register budget: -C (4NF doubles) + A (4NF) + the next step's A in
    // flight (4NF).  For NF >= 7 that no longer fits next to the rest of the
    // kernel without spills, so wide tiles load each step's A when it starts
    // (the other warp of the SM sub-partition hides the latency).
    constexpr bool kPrefetch = NF <= 6;
    for (int kk = 0; kk < q; ++kk) {
      double2 an[kMF][NF];
      if (!kPrefetch && kk > 0) load_a(a, ra, nr, k0 + kk);
      if (kPrefetch && kk + 1 < q) load_a(an, ra, nr, k0 + kk + 1);
      if (first_done && lane == 0 && kk == 0) first_done[1] = globaltimer();
      const double* B = Bs + kk * Tp * NPB;
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        if (8 * s < T) {
          if (CHOL) {  // Bs[n][k]: both k-halves of lane t with one 16-byte load
            double2 bv[NF];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf)
              bv[nf] = *reinterpret_cast<const double2*>(B + (8 * nf + g) * NPB + 8 * s + 2 * t);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int mf = 0; mf < kMF; ++mf)
#pragma unroll
                for (int nf = 0; nf < NF; ++nf)
                  dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], h ? a[mf][s].y : a[mf][s].x,
                             h ? bv[nf].y : bv[nf].x);
          } else {  // Bs[k][n]
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double bv[NF];
#pragma unroll
              for (int nf = 0; nf < NF; ++nf) bv[nf] = B[(8 * s + 2 * t + h) * NPB + 8 * nf + g];
#pragma unroll
              for (int mf = 0; mf < kMF; ++mf)
#pragma unroll
                for (int nf = 0; nf < NF; ++nf)
                  dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], h ? a[mf][s].y : a[mf][s].x, bv[nf]);
            }
          }
        }
      }
      // publish the previous strip once this one's first DMMAs are issued:
      // its stores went out a whole strip ago, so the release does not stall
      if (kk == 0 && prev_ra >= 0) {
        warp_signal(p, prev_ra, prev_ra + prev_nr, j);
        prev_ra = -1;
      }
      if (kPrefetch && kk + 1 < q) {
#pragma unroll
        for (int mf = 0; mf < kMF; ++mf)
#pragma unroll
          for (int s = 0; s < NF; ++s) a[mf][s] = an[mf][s];
      }
    }
    const int lower_off = CHOL ? ra - jT : kNoLower;  // Cholesky: store only row >= col
#pragma unroll
    for (int mf = 0; mf < kMF; ++mf) {
      const int r = mf * 8 + g;
      if (r < nr) {
        double* crow = p.a + static_cast<long long>(ra + r) * ld + jT;
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          const int c = nf * 8 + 2 * t;
          const double v0 = negd(acc[mf][nf][0]), v1 = negd(acc[mf][nf][1]);
          const bool ok0 = c < T && r + lower_off >= c, ok1 = c + 1 < T && r + lower_off >= c + 1;
          if (cvec && ok0 && ok1) {
            *reinterpret_cast<double2*>(crow + c) = make_double2(v0, v1);
          } else {
            if (ok0) crow[c] = v0;
            if (ok1) crow[c + 1] = v1;
          }
        }
      }
    }
    if (first_done && lane == 0) {
      first_done[0] = globaltimer();
      first_done = nullptr;
    }
    if (eager) {
      warp_signal(p, ra, ra + nr, j);
    } else {
      prev_ra = ra;
      prev_nr = nr;
    }
  }
  if (prev_ra >= 0) warp_signal(p, prev_ra, prev_ra + prev_nr, j);
}

// ---- pipelined strip GEMM (every GEMM task, q >= 1):
// C(rows, j) -= sum_{k in [k0, k0+q)} L(rows, k) * B_k.
//
// Each warp walks its 16-row strips (ra = r0 + 16 warp + 128 i) as a stream
// of items — per strip the q A-step operands L(strip, k0+kk) and then the
// strip's C tile — copied by cp.async.cg (L2 only) into a per-warp ring of
// R shared-memory slots, up to R-1 items ahead of the one being consumed:
// the next steps' and the next strip's operands are in flight while the
// current step's DMMAs run, so no L2 round trip sits between two steps or two
// strips (the register path above paid one per strip).  The accumulators
// start from zero and C is read last: C - sum A_k B_k, so the C tile's own
// dependency (its earlier stages) is only waited for when its item is issued.
// An item whose inputs are not yet published is issued when it is next to be
// consumed (blocking there only); items are issued in order, so the cp.async
// groups retire in order.  The B tiles (q stacked, stage_b) are staged once
// per task, their copies in flight together with each warp's first items.
__host__ __device__ constexpr int sa_stride(int tp) { return tp % 16 == 8 ? tp : tp + 8; }
// Ring slots per warp for strips of 8*smf rows.  Bulk GEMM tasks with T <= 40
// run 32-row strips (smf = 4: twice the DMMAs per item, per poll and per
// release, B fragments shared by four row blocks) in a 2-slot ring; the rest
// 16-row strips in 3 (T <= 40) or 2 slots.
__host__ __device__ constexpr int ring_slots(int nf, int smf = kMF) {
  return smf == 4 ? 2 : (nf <= 5 ? 3 : 2);
}
__host__ __device__ constexpr bool wide_strips_ok(int nf) { return nf <= 5; }
__host__ __device__ constexpr int ring_doubles(int nf) {
  const int narrow = kWarps * ring_slots(nf, kMF) * kStrip * sa_stride(nf * 8);
  const int wide = kWarps * ring_slots(nf, 4) * 32 * sa_stride(nf * 8);
  return wide_strips_ok(nf) && wide > narrow ? wide : narrow;
}
// B tiles first (q stacked), the rings after them (16-byte aligned)
__host__ __device__ constexpr int ring_offset(int q, int tp, bool chol) {
  return (q * tp * bstride(tp, chol) + 1) & ~1;
}

__device__ __forceinline__ void cp_async_wait_n(int n) {
  switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    default: cp_async_wait<3>(); break;
  }
}

// Rows [rs, re) of tile column kl final (the L rows a GEMM over steps up to kl
// reads); one poll per lane, `block` waits.
__device__ __forceinline__ bool a_deps(const Params& p, int rs, int re, int kl, bool block) {
  const int T = p.T, nt = p.nt;
  const int ti0 = rs / T, nti = (re - 1) / T - ti0 + 1;
  const int d = threadIdx.x & 31;
  bool ok = true;
  if (d < nti) {
    const int* c = &p.cnt[(ti0 + d) * nt + kl];
    const int need = need_final(p, kl, kl);
    ok = block ? wait_ge(p, c, need) : ld_acquire(c) >= need;
  }
  return __all_sync(0xffffffffu, ok);
}

// Issues the cp.async copies of the B tiles (no wait: the caller's first
// pipeline items join them in flight; gemm_pipe waits before its barrier).
template <int NF, bool CHOL>
__device__ __forceinline__ void stage_b_async(const Params& p, double* Bs, int j, int k0, int q) {
  constexpr int Tp = NF * 8, NPB = bstride(Tp, CHOL), HP = Tp / 2;
  const int T = p.T;
  const long long ld = p.ld;
  const int total = q * Tp * HP;  // element pairs
  for (int e = threadIdx.x; e < total; e += kThreads) {
    const int kk = e / (Tp * HP), rem = e - kk * (Tp * HP), x = rem / HP, y = 2 * (rem - x * HP);
    const int k = k0 + kk;
    const long long row = CHOL ? static_cast<long long>(j) * T + x : static_cast<long long>(k) * T + x;
    const long long col = CHOL ? static_cast<long long>(k) * T + y : static_cast<long long>(j) * T + y;
    const double* src = p.a + row * ld + col;
    double* dst = Bs + kk * Tp * NPB + x * NPB + y;
    if (!(T & 1)) {
      const bool valid = x < T && y < T;
      cp_async16_zfill(dst, valid ? src : p.a, valid);
    } else {  // odd T: rows are not 16-byte aligned
      dst[0] = (x < T && y < T) ? __ldcg(src) : 0.0;
      dst[1] = (x < T && y + 1 < T) ? __ldcg(src + 1) : 0.0;
    }
  }
  cp_async_commit();
}

template <int NF, bool CHOL, int SMF>
__device__ void gemm_pipe(const Params& p, int j, int k0, int q, int r0, int r1,
                          double* __restrict__ smem, bool eager, unsigned long long* first_done) {
  constexpr int Tp = NF * 8, NPB = bstride(Tp, CHOL), SA = sa_stride(Tp), R = ring_slots(NF, SMF);
  constexpr int GS = 8 * SMF;  // rows per strip
  constexpr int HP = Tp / 2, kSlot = GS * SA;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  const int T = p.T;
  const long long ld = p.ld;
  const int kl = k0 + q - 1, jT = j * T;
  const bool vec = !(T & 1);  // rows and tile origins 16-byte aligned (ld even, base aligned)
  const double* __restrict__ Bs = smem;
  double* ring = smem + ring_offset(q, Tp, CHOL) + warp * R * kSlot;
  const int first = r0 + warp * GS, stride = kWarps * GS;
  const int ns = first < r1 ? (r1 - first + stride - 1) / stride : 0;
  const int per = q + 1;  // items per strip: q A steps, then C
  const int total = ns * per;
  int issued = 0;

  // Per-lane copy pattern of one item (16 rows x T columns in 16-byte
  // vectors), the same for every item: vector v = lane + 32 u is row r_u,
  // column pair c_u; offsets precomputed once per task (the integer work of
  // the copy loop was 2-3 IMAD per DMMA).
  constexpr int NVEC = (GS * HP + 31) / 32;
  int goff[NVEC], soff[NVEC];
  unsigned rowmask = 0;  // bit u: vector u in a valid column; row checked per strip
  int vrow[NVEC];
#pragma unroll
  for (int u = 0; u < NVEC; ++u) {
    const int e = lane + 32 * u, r = e / HP, c = 2 * (e - r * HP);
    vrow[u] = e < GS * HP ? r : GS;
    goff[u] = r * static_cast<int>(ld) + c;
    soff[u] = r * SA + c;
    if (e < GS * HP && c < T) rowmask |= 1u << u;
  }

  int is_i = 0, is_kk = 0;  // strip / item of the next item to issue
  auto issue = [&](int y) {
    const int i = is_i, kk = is_kk;
    const int ra = first + i * stride, nr = min(GS, r1 - ra);
    const double* src = p.a + static_cast<long long>(ra) * ld +
                        (kk < q ? static_cast<long long>(k0 + kk) * T : static_cast<long long>(jT));
    double* dst = ring + (y % R) * kSlot;
    if (vec) {
#pragma unroll
      for (int u = 0; u < NVEC; ++u) {
        if (vrow[u] < GS) {
          const bool valid = ((rowmask >> u) & 1) && vrow[u] < nr;
          cp_async16_zfill(dst + soff[u], valid ? src + goff[u] : p.a, valid);
        }
      }
    } else {  // odd T: synchronous copies (visible after the consumer's __syncwarp)
      for (int e = lane; e < GS * Tp; e += 32) {
        const int r = e / Tp, c = e - r * Tp;
        dst[r * SA + c] = (r < nr && c < T) ? __ldcg(src + static_cast<long long>(r) * ld + c) : 0.0;
      }
    }
    cp_async_commit();
  };
  // Task-start poll: one round trip checks the A and C dependencies of all
  // of this warp's strips (lane = one counter); strips found satisfied skip
  // their per-strip polls (in the bulk of the schedule the inputs of a task
  // are final by the time it starts).  Bit i of a_ok / c_ok: strip i ready.
  unsigned a_ok = 0, c_ok = 0;
  {
    const int ti_lo = first / T;
    const int ti_hi = ns > 0 ? (min(r1, first + (ns - 1) * stride + GS) - 1) / T : ti_lo - 1;
    const int ntile = ti_hi - ti_lo + 1;
    bool tile_ok = false;  // lane d < ntile: tile row ti_lo + d, A dep; ntile <= d < 2 ntile: C dep
    if (ntile > 0 && 2 * ntile <= 32 && ns <= 32) {
      if (lane < 2 * ntile) {
        const int i = ti_lo + (lane < ntile ? lane : lane - ntile);
        const int* c = lane < ntile ? &p.cnt[i * p.nt + kl] : &p.cnt[i * p.nt + j];
        const int need = lane < ntile ? need_final(p, kl, kl)
                                      : need_before(p, min(i, j), j, k0);
        tile_ok = ld_acquire(c) >= need;
      }
      const unsigned okm = __ballot_sync(0xffffffffu, tile_ok);
      const unsigned am = okm & ((1u << ntile) - 1), cm = (okm >> ntile) & ((1u << ntile) - 1);
      for (int i = 0; i < ns; ++i) {
        const int rs = first + i * stride, re = min(r1, rs + GS);
        const int t0 = rs / T - ti_lo, t1 = (re - 1) / T - ti_lo;
        const unsigned need = ((2u << t1) - 1) & ~((1u << t0) - 1);
        if ((am & need) == need) a_ok |= 1u << i;
        if ((cm & need) == need) c_ok |= 1u << i;
      }
    }
  }
  // issue items up to x + R - 1 in order; item x itself waits for its inputs
  // when `block_x` (false: only on abort)
  auto pump = [&](int x, bool block_x) -> bool {
    while (issued < total && issued < x + R) {
      const int y = issued, i = is_i, kk = is_kk;
      if ((kk == 0 && !((a_ok >> i) & 1)) || (kk == q && !((c_ok >> i) & 1))) {
        const int rs = first + i * stride, re = min(r1, rs + GS);
        const bool blk = block_x && y == x;
        const bool ok = kk == 0 ? a_deps(p, rs, re, kl, blk) : strip_deps(p, rs, re, j, k0, -1, blk);
        if (!ok) {
          if (blk) return false;  // aborted
          break;
        }
      }
      issue(y);
      ++issued;
      if (++is_kk == per) {
        is_kk = 0;
        ++is_i;
      }
    }
    return true;
  };

  pump(0, false);  // first items in flight with the B tiles
  cp_async_wait_n(issued);  // the oldest group: B
  __syncthreads();
  if (first_done && lane == 0) first_done[2] = globaltimer();

  double acc[SMF][NF][2];
#pragma unroll
  for (int mf = 0; mf < SMF; ++mf)
#pragma unroll
    for (int nf = 0; nf < NF; ++nf) acc[mf][nf][0] = acc[mf][nf][1] = 0.0;
  int prev_ra = -1, prev_nr = 0;
  for (int x = 0, i = 0, kk = 0; x < total; ++x) {
    if (!pump(x, true)) return;
    cp_async_wait_n(issued - x - 1);
    __syncwarp();
    const double* slot = ring + (x % R) * kSlot;
    const int ra = first + i * stride, nr = min(GS, r1 - ra);
    if (kk < q) {
      if (first_done && lane == 0 && x == 0) first_done[1] = globaltimer();
      const double* B = Bs + kk * Tp * NPB;
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        if (8 * s < T) {
          double2 af[SMF];
#pragma unroll
          for (int mf = 0; mf < SMF; ++mf)
            af[mf] = *reinterpret_cast<const double2*>(slot + (mf * 8 + g) * SA + 8 * s + 2 * t);
          if (CHOL) {  // Bs[n][k]: both k-halves of lane t with one 16-byte load
            double2 bv[NF];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf)
              bv[nf] = *reinterpret_cast<const double2*>(B + (8 * nf + g) * NPB + 8 * s + 2 * t);
            // k-half outer: consecutive DMMAs on one accumulator are SMF*NF
            // apart (back to back, the compiler pads the DMMA latency with NOPs)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int mf = 0; mf < SMF; ++mf)
#pragma unroll
                for (int nf = 0; nf < NF; ++nf)
                  dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], h ? af[mf].y : af[mf].x,
                             h ? bv[nf].y : bv[nf].x);
          } else {  // Bs[k][n]
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double bv[NF];
#pragma unroll
              for (int nf = 0; nf < NF; ++nf) bv[nf] = B[(8 * s + 2 * t + h) * NPB + 8 * nf + g];
#pragma unroll
              for (int mf = 0; mf < SMF; ++mf)
#pragma unroll
                for (int nf = 0; nf < NF; ++nf)
                  dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], h ? af[mf].y : af[mf].x, bv[nf]);
            }
          }
        }
      }
      // publish the previous strip once this one's first DMMAs are issued
      if (kk == 0 && prev_ra >= 0) {
        warp_signal(p, prev_ra, prev_ra + prev_nr, j);
        prev_ra = -1;
      }
    } else {  // C item: C - sum, stores (Cholesky diagonal tiles: row >= col only)
      const int lower_off = CHOL ? ra - jT : kNoLower;
#pragma unroll
      for (int mf = 0; mf < SMF; ++mf) {
        const int r = mf * 8 + g;
        if (r < nr) {
          double* crow = p.a + static_cast<long long>(ra + r) * ld + jT;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) {
            const int c = nf * 8 + 2 * t;
            const double2 cv = *reinterpret_cast<const double2*>(slot + r * SA + c);
            const double v0 = cv.x - acc[mf][nf][0], v1 = cv.y - acc[mf][nf][1];
            const bool ok0 = c < T && r + lower_off >= c, ok1 = c + 1 < T && r + lower_off >= c + 1;
            if (vec && ok0 && ok1) {
              *reinterpret_cast<double2*>(crow + c) = make_double2(v0, v1);
            } else {
              if (ok0) crow[c] = v0;
              if (ok1) crow[c + 1] = v1;
            }
          }
        }
      }
#pragma unroll
      for (int mf = 0; mf < SMF; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) acc[mf][nf][0] = acc[mf][nf][1] = 0.0;
      if (first_done && lane == 0) {
        first_done[0] = globaltimer();
        first_done = nullptr;
      }
      if (eager) {
        warp_signal(p, ra, ra + nr, j);
      } else {
        prev_ra = ra;
        prev_nr = nr;
      }
    }
    __syncwarp();  // every lane's reads of this slot done before it is refilled
    if (++kk == per) {
      kk = 0;
      ++i;
    }
  }
  if (prev_ra >= 0) warp_signal(p, prev_ra, prev_ra + prev_nr, j);
}

// ---------------------------------------------------------------- DIAG
// Reciprocal: MUFU seed + two Newton steps (~50 cycles vs ~110 for the IEEE
// division sequence) — the pivot reciprocal sits on the factorisation's
// serial chain.  Within 1 ulp of 1/x for the normal pivots that pass the
// reference's failure checks.
// MUFU reciprocal seed.  rcp.approx.ftz.f64 flushes results below 2^-1022
// to zero, i.e. every |x| > 2^1022 would get r = 0 (and a zero multiplier,
// where the reference divides exactly, kernels.cpp:191): such pivots (a
// warp-uniform, never-taken-in-practice branch) take the seed of x/4, scaled
// back by 1/4 — a subnormal reciprocal with >= 50 significant bits.
__device__ __forceinline__ double rcp_seed(double x) {
  double r;
  if (fabs(x) > 0x1p1021) {
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x * 0.25));
    return r * 0.25;
  }
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

__device__ __forceinline__ double rcp_nr(double x) {
  double r = rcp_seed(x);
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}



// Blocked factorisation of the diagonal tile (T <= 64, NB = ceil(T/8) blocks)
// resident in shared memory D (64 x kNP, identity-padded):
//   per 8-column block b:  warp 0 factors the 8x8 diagonal block in DMMA
//   fragment layout with shuffles (the only per-pivot serial chain: shuffle,
//   reciprocal, multiply, FMA) and forms inv(U_bb), inv(L_bb) (kept in
//   `inv` for the solves); then all warps solve the L and U panels
//   (X = A inv(U_bb), Y = inv(L_bb) A) and apply the rank-8 trailing update
//   on the fp64 tensor cores (DMMA 8x8x4).
// Three __syncthreads per 8 pivots instead of one per pivot.  Cholesky runs
// the same elimination on the symmetric tile (A = L U with U = diag(u) L^T);
// tile_store scales l_ij = L_ij sqrt(u_jj).  Failure predicates are the
// reference's on the same Schur-complement pivots (kernels.cpp:187-190,
// :297-302; NaN passes).
// inv: [b*64, +64) inv(U_bb) row-major, [512 + b*64, +64) inv(L_bb) row-major.
// rk[c] = 1/u_cc.
template <bool CHOL, int NTH = kThreads>
__device__ __forceinline__ void tile_load(double* D, const double* __restrict__ dk, long long ld,
                                          int T) {
  if (!(T & 1)) {  // element pairs (16-byte loads); Cholesky mirrors the lower triangle
    constexpr int kPer = (64 * 32 + NTH - 1) / NTH;
    double2 v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = threadIdx.x + u * NTH, i = e >> 5, c = 2 * (e & 31);
      if (e < 64 * 32 && i < T && c < T && (!CHOL || c <= i))
        v[u] = __ldcg(reinterpret_cast<const double2*>(dk + static_cast<long long>(i) * ld + c));
      else
        v[u] = make_double2(i == c ? 1.0 : 0.0, i == c + 1 ? 1.0 : 0.0);
      if (i >= T || c >= T) v[u] = make_double2(i == c ? 1.0 : 0.0, i == c + 1 ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = threadIdx.x + u * NTH, i = e >> 5, c = 2 * (e & 31);
      if (e >= 64 * 32) break;
      if (!CHOL) {
        *reinterpret_cast<double2*>(D + i * kNP + c) = v[u];
      } else {
        if (c <= i) {
          D[i * kNP + c] = v[u].x;
          D[c * kNP + i] = v[u].x;
        }
        if (c + 1 <= i) {
          D[i * kNP + c + 1] = v[u].y;
          D[(c + 1) * kNP + i] = v[u].y;
        }
      }
    }
    return;
  }
  constexpr int kPer = (64 * 64 + NTH - 1) / NTH;
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {  // Cholesky: mirror the lower triangle
    const int e = threadIdx.x + u * NTH, i = e >> 6, c = e & 63;
    const int si = (CHOL && c > i) ? c : i, sc = (CHOL && c > i) ? i : c;
    v[u] = (e < 4096 && i < T && c < T) ? __ldcg(dk + static_cast<long long>(si) * ld + sc)
                                        : (i == c ? 1.0 : 0.0);
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = threadIdx.x + u * NTH;
    if (e < 4096) D[(e >> 6) * kNP + (e & 63)] = v[u];
  }
}

// tile_load from the raw rows in shared memory (the walker's prefetch buffer P):
// Cholesky mirrors the lower triangle, identity padding outside T x T.
template <bool CHOL, int NTH = kThreads>
__device__ __forceinline__ void tile_from_raw(double* D, const double* P, int T) {
  for (int e = threadIdx.x; e < 4096; e += NTH) {
    const int i = e >> 6, c = e & 63;
    const int si = (CHOL && c > i) ? c : i, sc = (CHOL && c > i) ? i : c;
    D[i * kNP + c] = (i < T && c < T) ? P[si * kNP + sc] : (i == c ? 1.0 : 0.0);
  }
}

// 8x8 diagonal block b (one warp, fragment layout, shuffles) + inv(U_bb),
// inv(L_bb).  Called by warp 0 only.
template <bool CHOL>
__device__ __forceinline__ void factor_block8(double* D, int T, int gcol, int* info, double* inv,
                                              double* rk, int b, int* sfail) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int p = 8 * b;
  double* invU = inv + b * 64;
  double* invL = inv + 512 + b * 64;
  __syncwarp();  // converged warp: keeps the shuffles on the fast path
  double v0 = D[(p + g) * kNP + p + 2 * t], v1 = D[(p + g) * kNP + p + 2 * t + 1];
  double rr[8];
  int fail = INT_MAX;  // first failing pivot (warp-uniform: pivots come by shuffle)
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const double sel = (kk & 1) ? v1 : v0;
    const double piv = __shfl_sync(0xffffffffu, sel, kk * 4 + (kk >> 1));
    // rows above the pivot take a zero multiplier: mask the operand (off the chain)
    const double agk_all = __shfl_sync(0xffffffffu, sel, g * 4 + (kk >> 1));  // all lanes
    const double agk = g > kk ? -agk_all : 0.0;
    const double u0 = __shfl_sync(0xffffffffu, v0, kk * 4 + t);
    const double u1 = __shfl_sync(0xffffffffu, v1, kk * 4 + t);
    // m = agk / piv off a short chain: MUFU seed r0 (rel. error e ~ 2^-23),
    // m = agk r0 (1 + e + e^2) (truncation e^3 < 2^-66): 3 dependent DFMAs
    // after the seed instead of two Newton steps and a multiply.
    const double r0 = rcp_seed(piv);
    const double e = fma(-piv, r0, 1.0);
    const double tq = fma(e, e, e);
    const double nm0 = agk * r0;             // -m0 (agk is negated)
    const double nm = fma(nm0, tq, nm0);     // -m, no select on the chain
    const double r = fma(r0, tq, r0);
    if (2 * t > kk) v0 = fma(nm, u0, v0);
    if (2 * t + 1 > kk) v1 = fma(nm, u1, v1);
    if (g > kk && 2 * t == kk) v0 = -nm;
    if (g > kk && 2 * t + 1 == kk) v1 = -nm;
    rr[kk] = r;
    // the reference's failure predicates (kernels.cpp:187-190 / :297-302; NaN passes)
    if (p + kk < T && (CHOL ? piv <= 0.0 : fabs(piv) < 1e-300)) fail = min(fail, kk);
  }
  D[(p + g) * kNP + p + 2 * t] = v0;
  D[(p + g) * kNP + p + 2 * t + 1] = v1;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
    if (p + kk < T) rk[p + kk] = rr[kk];  // same value from every lane
  if (fail != INT_MAX && lane == 0) {
    atomicMin(info, gcol + p + fail);
    *sfail = 1;  // the walker checks this shared flag, not the global status word
  }
  __syncwarp();
  // inv(U_bb) (lanes 0..7) and inv(L_bb) (lanes 8..15), one column per lane,
  // by back substitution without divisions.  Both run the same instruction
  // stream: lanes 8..15 read the unit lower L through its reversal J L J
  // (upper; staged in `rev`), whose inverse is J inv(L) J.  (Keeping inv(L)
  // out of the pivot loop saves two double shuffles per pivot.)
  double* rev = invL;  // the 8x8 reversal, overwritten by inv(L) below
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int col = 2 * t + h;
    if (g > col) rev[(7 - g) * 8 + 7 - col] = h ? v1 : v0;  // strict upper part of J L J
  }
  __syncwarp();
  if (lane < 16) {
    const bool lo = lane >= 8;
    const int c = lane & 7;
    const double* m = lo ? rev : D + p * kNP + p;
    const int ms = lo ? 8 : kNP;
    double x[8];
#pragma unroll
    for (int ii = 7; ii >= 0; --ii) {
      double acc = ii == c ? 1.0 : 0.0;
#pragma unroll
      for (int mm = 7; mm > ii; --mm) acc = fma(-m[ii * ms + mm], x[mm], acc);  // newest term last
      x[ii] = lo ? acc : acc * (p + ii < T ? rr[ii] : 1.0);
    }
    __syncwarp(0x0000ffffu);  // all reads of `rev` done before inv(L) overwrites it
    double* dst = lo ? invL : invU;
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) {
      const int r = lo ? 7 - ii : ii, cc = lo ? 7 - c : c;
      dst[r * 8 + cc] = x[ii];
    }
  }
}

// One warp: trailing update of block row ir (of step b) over block columns
// jr in [jlo, nr): block (b+1+ir, b+1+jr) -= L(b+1+ir, b) * U(b, b+1+jr).
__device__ __forceinline__ void trail_row(double* D, int b, int nr, int ir, int jlo) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int p = 8 * b, ib = 8 * (b + 1 + ir);
  const double a0 = -D[(ib + g) * kNP + p + t], a1 = -D[(ib + g) * kNP + p + 4 + t];
  double c0[7], c1[7];
#pragma unroll
  for (int jr = 0; jr < 7; ++jr) {
    if (jr >= jlo && jr < nr) {
      const int jb = 8 * (b + 1 + jr);
      c0[jr] = D[(ib + g) * kNP + jb + 2 * t];
      c1[jr] = D[(ib + g) * kNP + jb + 2 * t + 1];
      const double b0 = D[(p + t) * kNP + jb + g], b1 = D[(p + 4 + t) * kNP + jb + g];
      dmma_8x8x4(c0[jr], c1[jr], a0, b0);
      dmma_8x8x4(c0[jr], c1[jr], a1, b1);
    }
  }
#pragma unroll
  for (int jr = 0; jr < 7; ++jr) {
    if (jr >= jlo && jr < nr) {
      const int jb = 8 * (b + 1 + jr);
      D[(ib + g) * kNP + jb + 2 * t] = c0[jr];
      D[(ib + g) * kNP + jb + 2 * t + 1] = c1[jr];
    }
  }
}

// Barrier over the first NW warps of the CTA (all 8: __syncthreads; fewer:
// named barrier 1 — the walker's compute warps while warp 7 publishes).
template <int NW>
__device__ __forceinline__ void csync() {
  if (NW == kWarps)
    __syncthreads();
  else
    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}
// The same barrier, AND-reducing a predicate over the participating threads.
template <int NW>
__device__ __forceinline__ bool csync_and(bool pred) {
  if (NW == kWarps) return __syncthreads_and(pred);
  int r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.s32 p, %1, 0;\n"
      " bar.red.and.pred q, 1, %2, p;\n selp.s32 %0, 1, 0, q;\n}"
      : "=r"(r)
      : "r"(pred ? 1 : 0), "n"(NW * 32)
      : "memory");
  return r != 0;
}

// Blocked elimination of the tile in shared memory with look-ahead: while
// warps 1..7 apply step b's trailing update, warp 0 updates the next
// diagonal block first and factors it, so the serial 8x8 chain of block b+1
// overlaps the bulk of step b.  Two __syncthreads per 8 pivots.
template <bool CHOL, int NW = kWarps>
__device__ __forceinline__ void diag_blocked(double* D, int T, int gcol, int* info, double* inv,
                                             double* rk, int* sfail) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int NB = (T + 7) >> 3;
  if (warp == 0) factor_block8<CHOL>(D, T, gcol, info, inv, rk, 0, sfail);
  csync<NW>();
  for (int b = 0; b + 1 < NB; ++b) {
    const int p = 8 * b, nr = NB - b - 1;
    const double* invU = inv + b * 64;
    const double* invL = inv + 512 + b * 64;
    // ---- panels: job < nr: L block (b+1+job, b) = A * inv(U_bb);
    //               job >= nr: U block (b, b+1+job-nr) = inv(L_bb) * A
    for (int job = warp; job < 2 * nr; job += NW) {
      double c0 = 0.0, c1 = 0.0;
      if (job < nr) {
        const int rb = 8 * (b + 1 + job);
        const double a0 = D[(rb + g) * kNP + p + t], a1 = D[(rb + g) * kNP + p + 4 + t];
        const double b0 = invU[t * 8 + g], b1 = invU[(4 + t) * 8 + g];
        dmma_8x8x4(c0, c1, a0, b0);
        dmma_8x8x4(c0, c1, a1, b1);
        __syncwarp();
        D[(rb + g) * kNP + p + 2 * t] = c0;
        D[(rb + g) * kNP + p + 2 * t + 1] = c1;
      } else {
        const int cb = 8 * (b + 1 + job - nr);
        const double a0 = invL[g * 8 + t], a1 = invL[g * 8 + 4 + t];
        const double b0 = D[(p + t) * kNP + cb + g], b1 = D[(p + 4 + t) * kNP + cb + g];
        dmma_8x8x4(c0, c1, a0, b0);
        dmma_8x8x4(c0, c1, a1, b1);
        __syncwarp();
        D[(p + g) * kNP + cb + 2 * t] = c0;
        D[(p + g) * kNP + cb + 2 * t + 1] = c1;
      }
    }
    csync<NW>();
    if (warp == 0) {  // look-ahead: diagonal block (b+1,b+1) first, then factor it
      trail_row(D, b, 1, 0, 0);
      __syncwarp();
      factor_block8<CHOL>(D, T, gcol, info, inv, rk, b + 1, sfail);
    } else {  // the rest of step b's trailing update
      // warps 1-3, 5-7 only: warp 4 shares warp 0's SM sub-partition; keeping
      // its DMMAs off it measured a slightly shorter DIAG (9.8 vs 10.1 us/step)
      if (warp != 4) {
        const int wi = warp < 4 ? warp - 1 : warp - 2;
        for (int ir = wi; ir < nr; ir += NW - 2) trail_row(D, b, nr, ir, ir == 0 ? 1 : 0);
      }
    }
    csync<NW>();
  }
  // Cholesky: l_jj = sqrt(u_jj) (rk[64 + j]) and 1/l_jj (rk[j]) for the solves
  if (CHOL && tid < T) {
    const double l = sqrt(D[tid * kNP + tid]);
    rk[64 + tid] = l;
    rk[tid] = rcp_nr(l);
  }
  csync<NW>();
}

// Factored tile -> global (Cholesky: lower only, scaled) and the diagonal
// reciprocals -> the step's solve slot (read by the TRSM tasks).
template <bool CHOL, int NTH = kThreads>
__device__ __forceinline__ void tile_store(const double* D, double* __restrict__ dk, long long ld,
                                           int T, const double* rk, double* solve) {
  for (int e = threadIdx.x; e < 64 * 64; e += NTH) {
    const int i = e >> 6, c = e & 63;
    if (i < T && c < T && (!CHOL || c <= i)) {
      double v = D[i * kNP + c];
      if (CHOL) v = c == i ? rk[64 + c] : v * rk[64 + c];
      dk[static_cast<long long>(i) * ld + c] = v;
    }
  }
  if (threadIdx.x < 64) solve[threadIdx.x] = rk[threadIdx.x];
}

// ---------------------------------------------------------------- TRSM
// In place X * M = S for one 16-row strip: element (r, c) of S/X lives at
// base + r*rs + c*cs (rs = ld, cs = 1 for row strips; rs = 1, cs = ld for the
// transposed U12 solve).  M (Tp x Tp upper triangular, identity-padded) and
// the inverses of its 8x8 diagonal blocks are in shared memory.  Blocked by
// 8 columns: R_b = S_b - X_<b * M_<b,b (DMMA), X_b = R_b * inv(M_bb) (DMMA).
// MMODE: 0 = M[r][c] = Ms[r*kNP + c]; 1 = M[r][c] = Ms[c*kNP + r] (M is the
// transpose of the stored tile); 2 = as 1, scaled by msc[r] (Cholesky L^T).
template <int NF, bool SMEM = false, int MMODE = 0, int MF = kMF>
__device__ __forceinline__ void warp_trsm(double* __restrict__ base, long long rs, long long cs,
                                          int nrows, int T, const double* __restrict__ Ms,
                                          const double* __restrict__ Minv,
                                          const double* __restrict__ msc = nullptr) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  // global row strips: element pairs as 16-byte accesses when aligned
  const bool vec = !SMEM && cs == 1 && !(rs & 1) && !(T & 1) &&
                   !(reinterpret_cast<uintptr_t>(base) & 15);
  double ra[NF][MF][2];
#pragma unroll
  for (int mf = 0; mf < MF; ++mf) {
    const int r = mf * 8 + g;
    const bool rv = r < nrows;
    const double* row = base + static_cast<long long>(rv ? r : 0) * rs;
    if (vec) {
#pragma unroll
      for (int b = 0; b < NF; ++b) {
        const int c = b * 8 + 2 * t;
        double2 v = make_double2(0.0, 0.0);
        if (rv && c < T) v = __ldcg(reinterpret_cast<const double2*>(row + c));
        ra[b][mf][0] = v.x;
        ra[b][mf][1] = v.y;
      }
    } else {
#pragma unroll
      for (int b = 0; b < NF; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = b * 8 + 2 * t + h;
          const double* src = row + static_cast<long long>(c) * cs;
          ra[b][mf][h] = (rv && c < T) ? (SMEM ? *src : __ldcg(src)) : 0.0;
        }
    }
  }
  // source lanes of the accumulator -> A-fragment relayout inside a quad:
  // A-layout k-step s needs column 4s + t, held by lane (g, 2s + t/2), half t&1.
  const int src0 = (lane & ~3) | (t >> 1), src1 = (lane & ~3) | (2 + (t >> 1));
  const bool odd = t & 1;
  // Right-looking over the 8-column blocks: once X_b is known it is applied
  // to every later block's accumulator (R_c -= X_b M_bc), so the serial
  // chain per block is relayout -> inv(M_bb) DMMA -> relayout -> one update
  // DMMA pair; the other blocks' updates overlap it.  Each R_c receives the
  // X_b M_bc terms in ascending b, the same order as the left-looking form.
#pragma unroll
  for (int b = 0; b < NF; ++b) {
    double rf[MF][2];
#pragma unroll
    for (int mf = 0; mf < MF; ++mf) {
      const double v0 = __shfl_sync(0xffffffffu, ra[b][mf][0], src0);
      const double v1 = __shfl_sync(0xffffffffu, ra[b][mf][1], src0);
      const double w0 = __shfl_sync(0xffffffffu, ra[b][mf][0], src1);
      const double w1 = __shfl_sync(0xffffffffu, ra[b][mf][1], src1);
      rf[mf][0] = odd ? v1 : v0;
      rf[mf][1] = odd ? w1 : w0;
    }
    double xo[MF][2] = {};
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double m = Minv[b * 64 + (4 * s + t) * 8 + g];
#pragma unroll
      for (int mf = 0; mf < MF; ++mf) dmma_8x8x4(xo[mf][0], xo[mf][1], rf[mf][s], m);
    }
    if (b + 1 < NF) {
      double xa[MF][2];  // -X_b in A-fragment layout
#pragma unroll
      for (int mf = 0; mf < MF; ++mf) {
        const double v0 = __shfl_sync(0xffffffffu, xo[mf][0], src0);
        const double v1 = __shfl_sync(0xffffffffu, xo[mf][1], src0);
        const double w0 = __shfl_sync(0xffffffffu, xo[mf][0], src1);
        const double w1 = __shfl_sync(0xffffffffu, xo[mf][1], src1);
        xa[mf][0] = -(odd ? v1 : v0);
        xa[mf][1] = -(odd ? w1 : w0);
      }
#pragma unroll
      for (int c = b + 1; c < NF; ++c)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int mr = b * 8 + 4 * s + t, mc = c * 8 + g;
          double m = MMODE == 0 ? Ms[mr * kNP + mc] : Ms[mc * kNP + mr];
          if (MMODE == 2) m *= msc[mr];
#pragma unroll
          for (int mf = 0; mf < MF; ++mf) dmma_8x8x4(ra[c][mf][0], ra[c][mf][1], xa[mf][s], m);
        }
    }
#pragma unroll
    for (int mf = 0; mf < MF; ++mf) {
      const int r = mf * 8 + g;
      if (r < nrows) {
        double* row = base + static_cast<long long>(r) * rs;
        const int c = b * 8 + 2 * t;
        if (vec) {
          if (c < T) *reinterpret_cast<double2*>(row + c) = make_double2(xo[mf][0], xo[mf][1]);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (c + h < T) row[static_cast<long long>(c + h) * cs] = xo[mf][h];
        }
      }
    }
  }
}

// Shared-memory step counters of the walker hand-off: release store / acquire
// load at CTA scope (the PTX pattern for a flag protecting prior writes).
__device__ __forceinline__ void st_release_cta(volatile int* f, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_u32(const_cast<int*>(f))), "r"(v)
               : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(volatile int* f) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(const_cast<int*>(f)))
               : "memory");
  return v;
}

// ---------------------------------------------------------------- walker
// The walker's publisher warp (tiles <= 48, see walker): the compute warps
// store the factored diagonal tile and the solved panel tiles themselves (224
// threads, no waiting), hand over at a barrier + shared step counter, and
// lane 0 of warp 7 issues the release reductions — whose fence waits for
// those stores to reach L2 (~1 us) — off the chain.  Cumulativity: the
// stores precede the compute warps' barrier, thread 0's flag write (after a
// CTA fence) and this warp's flag read (before a CTA fence), so the
// gpu-scope release covers them, as it covers a CTA's stores after a
// __syncthreads in warp_signal's pattern.
// Returns when the compute warps stop (wabort), a pivot failed (raises the
// schedule's abort flag), or after the last step.
template <int NF, bool CHOL>
__device__ void walker_publisher(const Params& p, const int* sfail, volatile int* dready,
                                 volatile int* luready, volatile int* wabort) {
  if ((threadIdx.x & 31) != 0) return;
  const int T = p.T, nt = p.nt;
  auto await = [&](volatile int* f, int k) -> bool {
    while (ld_acquire_cta(f) < k) {
      if (*wabort) return false;
      __nanosleep(32);
    }
    return true;
  };
  for (int k = 0; k < nt; ++k) {
    if (!await(dready, k)) return;
    if (*reinterpret_cast<const volatile int*>(sfail)) {
      atomicExch(p.abort, 1);
      return;
    }
    red_release_add(&p.cnt[k * nt + k], k >= 1 ? 2 * T : T);  // stage k-1 + DIAG(k)
    if (k + 1 >= nt) return;
    if (!await(luready, k)) return;
    red_release_add(&p.cnt[(k + 1) * nt + k], T);
    if (!CHOL) red_release_add(&p.cnt[k * nt + k + 1], T);
  }
}

template <int NF, bool CHOL>
__device__ void walker(const Params& p, double* dsm) {
  constexpr int Tp = NF * 8;
  double* D = dsm;                          // tile (k,k)
  double* Lt = dsm + kSmemB;                // tile (k+1,k): A21 -> L21
  double* Ut = Lt + kSmemB;                 // tile (k,k+1): A12 -> U12 (LU)
  double* rk = Ut + kSmemB;                 // 128
  double* inv = rk + 128;                   // 1024: DIAG block inverses
  double* invX = inv + 1024;                // 512: inverses for the second solve
  double* P = invX + 512;                   // prefetched tile (k+1,k+1), raw rows
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int T = p.T, nt = p.nt;
  const long long ld = p.ld;
  // PUB (Cholesky, tiles <= 48): warp 7 is the walker's publisher — it releases the
  // counters of the tiles the compute warps 0-6 stored (walker_publisher), so
  // the release fences (~1 us each, two per step) leave the chain.
  constexpr bool PUB = CHOL && NF <= 6;  // measured: Cholesky XL -1%, LU +3% (7 compute warps)
  constexpr int NW = PUB ? kWarps - 1 : kWarps;  // compute warps
  constexpr int NC = NW * 32;
  __shared__ int s_pf, s_pl, s_pu, s_fail;
  __shared__ volatile int s_dready, s_luready, s_wabort;
  if (tid == 0) {
    s_fail = 0;
    s_dready = s_luready = -1;
    s_wabort = 0;
  }
  __syncthreads();
  if (PUB && warp == kWarps - 1) {
    walker_publisher<NF, CHOL>(p, &s_fail, &s_dready, &s_luready, &s_wabort);
    return;
  }
  bool pref = false;  // tile (k,k) of this step was prefetched into P (stages < k-1)
  // Thread 0 waits on one counter (or two: c2 != nullptr); the barrier
  // AND-reduces its verdict (no shared status word to race on).
  auto wait1 = [&](const int* c, int need, const int* c2 = nullptr, int need2 = 0) -> bool {
    bool ok = true;
    if (tid == 0) {
      ok = wait_ge(p, c, need) && (!c2 || wait_ge(p, c2, need2));
      if (!ok) s_wabort = 1;  // the publisher stops too
    }
    return csync_and<NW>(ok);
  };
  auto stamp = [&](int k, int i) {
    if (p.trace && tid == 0)
      p.trace[8 * (static_cast<long long>(p.ntasks) + k) + i] = globaltimer();
  };
  for (int k = 0; k < nt; ++k) {
    const int kT = k * T;
    double* dk = p.a + static_cast<long long>(kT) * ld + kT;
    stamp(k, 0);
    // the updates of steps < k-1 of tile (k,k) come from the queue's GEMM
    // tasks (step k-1 is always a single step: the walker applies it)
    if (pref) {  // copies issued during the previous step's panel solves
      cp_async_wait<0>();
      csync<NW>();
      stamp(k, 1);
      tile_from_raw<CHOL, NC>(D, P, T);
    } else {
      if (k >= 2 && !wait1(&p.cnt[k * nt + k], need_before(p, k, k, k - 1))) return;
      stamp(k, 1);
      tile_load<CHOL, NC>(D, dk, ld, T);
    }
    csync<NW>();
    if (k >= 1) {  // stage k-1: D -= L(k,k-1) * U(k-1,k) (Cholesky: L L^T), DMMA in smem
      if (8 * warp < Tp) {
        const int r = 8 * warp;
        double acc[NF][2];
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          acc[nf][0] = D[(r + g) * kNP + nf * 8 + 2 * t];
          acc[nf][1] = D[(r + g) * kNP + nf * 8 + 2 * t + 1];
        }
#pragma unroll
        for (int s4 = 0; s4 < 2 * NF; ++s4) {
          if (4 * s4 < T) {
            const double a = -Lt[(r + g) * kNP + 4 * s4 + t];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              const double bv = CHOL ? Lt[(nf * 8 + g) * kNP + 4 * s4 + t]
                                     : Ut[(4 * s4 + t) * kNP + nf * 8 + g];
              dmma_8x8x4(acc[nf][0], acc[nf][1], a, bv);
            }
          }
        }
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          D[(r + g) * kNP + nf * 8 + 2 * t] = acc[nf][0];
          D[(r + g) * kNP + nf * 8 + 2 * t + 1] = acc[nf][1];
        }
      }
      csync<NW>();
    }
    stamp(k, 2);
    diag_blocked<CHOL, NW>(D, T, kT, p.info, inv, rk, &s_fail);
    stamp(k, 3);
    // Polls next to the tile store (warps 1-3, one lane each): the panel inputs
    // A(k+1,k) (and A(k,k+1)) at stage k-1, and the next diagonal tile at
    // stage k-1 (the walker applies stage k itself).  What is already final is
    // copied into shared memory (cp.async, warps 1-7) while thread 0's release
    // of DIAG(k) drains, instead of a poll and a load round trip after it.
    const bool more = k + 1 < nt;
    if (more && tid == 32)
      s_pf = !(T & 1) && ld_acquire(&p.cnt[(k + 1) * nt + k + 1]) >= need_before(p, k + 1, k + 1, k);
    if (more && tid == 64)
      s_pl = T == Tp && !(T & 1) && ld_acquire(&p.cnt[(k + 1) * nt + k]) >= need_before(p, k, k, k);
    if (more && tid == 96)
      s_pu = CHOL || (T == Tp && !(T & 1) &&
                      ld_acquire(&p.cnt[k * nt + k + 1]) >= need_before(p, k, k + 1, k));
    tile_store<CHOL, NC>(D, dk, ld, T, rk, p.solve + static_cast<long long>(k) * kSolveSlot);
    // publish: the CTA barrier orders every thread's stores before thread 0's
    // release reduction (cumulative), so one fence instead of one per warp.
    // A failing pivot (factor_block8, warp 0) raised s_fail before DIAG's last
    // barrier: no global read of the status word on the chain.
    csync<NW>();
    if (PUB) {  // hand D(k) to the publisher (release of tile (k,k))
      if (tid == 0) {
        st_release_cta(&s_dready, k);
      }
      if (s_fail) return;  // the publisher raises the abort flag
    }
    const bool pan = more && s_pl && s_pu;
    pref = more && s_pf;
    if (warp > 0 && (pan || pref)) {  // (warp 0 issues none: thread 0's fence below)
      const int hp = T >> 1, t7 = tid - 32;
      if (pan) {
        const double* al = p.a + static_cast<long long>(kT + T) * ld + kT;
        for (int e = t7; e < T * hp; e += NC - 32) {
          const int i = e / hp, c = 2 * (e - i * hp);
          cp_async16(Lt + i * kNP + c, al + static_cast<long long>(i) * ld + c);
          if (!CHOL) cp_async16(Ut + i * kNP + c, dk + T + static_cast<long long>(i) * ld + c);
        }
      }
      if (pref) {
        const double* dn = dk + static_cast<long long>(T) * ld + T;
        for (int e = t7; e < T * hp; e += NC - 32) {
          const int i = e / hp, c = 2 * (e - i * hp);
          cp_async16(P + i * kNP + c, dn + static_cast<long long>(i) * ld + c);
        }
      }
      cp_async_commit();
    }
    if (!PUB) {
      // s_fail is visible to every thread since the barrier above: no second
      // barrier here, warp 0's release fence overlaps the other warps' panel work
      if (tid == 0) {
        if (s_fail)
          atomicExch(p.abort, 1);
        else
          red_release_add(&p.cnt[k * nt + k], k >= 1 ? 2 * T : T);  // stage k-1 + DIAG(k)
      }
      if (s_fail) return;
    }
    if (!more) break;
    // ---- first tiles of the panel: L(k+1,k) = A(k+1,k) U11^-1, U(k,k+1) = L11^-1 A(k,k+1)
    if (pan) {
      cp_async_wait<0>();
      stamp(k, 4);
      for (int e = tid; e < NF * 64; e += NC) {  // inverses for the second solve (below)
        const int b = e >> 6, ii = (e >> 3) & 7, c = e & 7;
        const double v = inv[512 + b * 64 + c * 8 + ii];
        invX[e] = CHOL ? v * (8 * b + c < T ? rk[8 * b + c] : 1.0) : v;
      }
    } else {
    if (!wait1(&p.cnt[(k + 1) * nt + k], need_before(p, k, k, k),
               CHOL ? nullptr : &p.cnt[k * nt + k + 1], need_before(p, k, k + 1, k)))
      return;
    stamp(k, 4);
    {
      const double* al = p.a + static_cast<long long>(kT + T) * ld + kT;
      const double* au = dk + T;
      // element pairs (16-byte loads; T even keeps every pair aligned, T odd
      // loads the odd tail element alone)
      constexpr int kHP = Tp / 2, kPer = (Tp * kHP + NC - 1) / NC;
      double2 vl[kPer], vu[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = tid + u * NC, x = e / kHP, y = 2 * (e - x * kHP);
        const bool in = e < Tp * kHP && x < T && y < T;
        vl[u] = vu[u] = make_double2(0.0, 0.0);
        if (in && !(T & 1)) {
          vl[u] = __ldcg(reinterpret_cast<const double2*>(al + static_cast<long long>(x) * ld + y));
          if (!CHOL) vu[u] = __ldcg(reinterpret_cast<const double2*>(au + static_cast<long long>(x) * ld + y));
        } else if (in) {
          vl[u].x = __ldcg(al + static_cast<long long>(x) * ld + y);
          if (y + 1 < T) vl[u].y = __ldcg(al + static_cast<long long>(x) * ld + y + 1);
          if (!CHOL) {
            vu[u].x = __ldcg(au + static_cast<long long>(x) * ld + y);
            if (y + 1 < T) vu[u].y = __ldcg(au + static_cast<long long>(x) * ld + y + 1);
          }
        }
      }
      // the solves read M straight from the factored tile D: U11 = upper(D),
      // L11^T = lower(D)^T (Cholesky scaled by l_kk); only strictly-upper
      // entries of M between 8-blocks are read, and D is identity-padded
      // block inverses of the second M: LU inv(L_bb^T) = inv(L_bb)^T;
      // Cholesky inv(diag(l) L_bb^T) = inv(L_bb)^T diag(1/l)
      for (int e = tid; e < NF * 64; e += NC) {
        const int b = e >> 6, ii = (e >> 3) & 7, c = e & 7;
        const double v = inv[512 + b * 64 + c * 8 + ii];
        invX[e] = CHOL ? v * (8 * b + c < T ? rk[8 * b + c] : 1.0) : v;
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = tid + u * NC, x = e / kHP, y = 2 * (e - x * kHP);
        if (e < Tp * kHP) {
          *reinterpret_cast<double2*>(Lt + x * kNP + y) = vl[u];
          if (!CHOL) *reinterpret_cast<double2*>(Ut + x * kNP + y) = vu[u];
        }
      }
    }
    }  // panel not prefetched
    csync<NW>();
    stamp(k, 6);
    // warps 0..3: L21 strips (X * M = A21); warps 4..7: U12 strips on the
    // transposed view (X * L11^T = A12^T)
    if (CHOL && NF <= NW) {
      // Cholesky (T <= 8 NW): 8-row strips, one per compute warp — the serial
      // chain over the 8-column blocks carries half the work per block of a
      // 16-row strip (measured 2.5 us for three 16-row strips)
      const int c0 = warp * 8;
      if (c0 < T)
        warp_trsm<NF, true, 2, 1>(Lt + c0 * kNP, kNP, 1, min(8, T - c0), T, D, invX, rk + 64);
    } else if (!CHOL && NF <= 5) {
      // LU (T <= 40): L21 on 8-row strips (warps 0-4), U12 on 16-row strips
      // of the transposed view (warps 5-7)
      if (warp < 5) {
        const int c0 = warp * 8;
        if (c0 < T)
          warp_trsm<NF, true, 0, 1>(Lt + c0 * kNP, kNP, 1, min(8, T - c0), T, D, inv);
      } else {
        const int c0 = (warp - 5) * kStrip;
        if (c0 < T) warp_trsm<NF, true, 1>(Ut + c0, 1, kNP, min(kStrip, T - c0), T, D, invX);
      }
    } else {
      const int sw = warp & 3;
      const int c0 = sw * kStrip;
      if (c0 < T) {
        const int nr = min(kStrip, T - c0);
        if (warp < 4) {
          if (CHOL)
            warp_trsm<NF, true, 2>(Lt + c0 * kNP, kNP, 1, nr, T, D, invX, rk + 64);
          else
            warp_trsm<NF, true, 0>(Lt + c0 * kNP, kNP, 1, nr, T, D, inv);
        } else if (!CHOL) {
          warp_trsm<NF, true, 1>(Ut + c0, 1, kNP, nr, T, D, invX);
        }
      }
    }
    csync<NW>();
    stamp(k, 7);
    {  // the solved tiles -> global
      double* gl = p.a + static_cast<long long>(kT + T) * ld + kT;
      double* gu = dk + T;
      if (!(T & 1)) {  // 16-byte stores of element pairs
        constexpr int kHP = Tp / 2;
        for (int e = tid; e < Tp * kHP; e += NC) {
          const int x = e / kHP, y = 2 * (e - x * kHP);
          if (x < T && y < T) {
            *reinterpret_cast<double2*>(gl + static_cast<long long>(x) * ld + y) =
                *reinterpret_cast<const double2*>(Lt + x * kNP + y);
            if (!CHOL)
              *reinterpret_cast<double2*>(gu + static_cast<long long>(x) * ld + y) =
                  *reinterpret_cast<const double2*>(Ut + x * kNP + y);
          }
        }
      } else {
        for (int e = tid; e < T * T; e += NC) {
          const int x = e / T, y = e - x * T;
          gl[static_cast<long long>(x) * ld + y] = Lt[x * kNP + y];
          if (!CHOL) gu[static_cast<long long>(x) * ld + y] = Ut[x * kNP + y];
        }
      }
    }
    csync<NW>();
    if (tid == 0) {
      if (PUB) {  // the publisher releases them
        st_release_cta(&s_luready, k);
      } else {
        red_release_add(&p.cnt[(k + 1) * nt + k], T);
        if (!CHOL) red_release_add(&p.cnt[k * nt + k + 1], T);
      }
    }
    stamp(k, 5);
  }
}

// ---------------------------------------------------------------- kernel

template <int NF, bool CHOL>
__global__ void __launch_bounds__(kThreads, 1) dag_kernel(Params p) {
  constexpr int Tp = NF * 8;
  extern __shared__ __align__(16) double dsm[];
  double* sm = dsm;                      // B (GEMM) / M (TRSM): Tp x kNP
  double* minv = dsm + kSmemB;           // TRSM: 8 x (8x8) block inverses + 64 diagonal reciprocals
  double* abuf = dsm + kSmemB;           // single-step GEMM: per-warp A strips
  __shared__ int4 s_task[2];
  __shared__ int s_id[2];
  __shared__ int s_go;
  __shared__ unsigned long long s_t0, s_t1, s_ph[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int T = p.T, nt = p.nt;
  auto stamp = [&](int i) {
    if (p.trace && tid == 0) s_ph[i] = globaltimer();
  };
  const long long ld = p.ld;
  const int4 kNone = make_int4(-1, 0, 0, 0);
  if (tid == 0) atomicAdd(p.abort + 2, 1);  // CTAs started (watchdog diagnostics)

  if (blockIdx.x == 0) {
    if (!p.nodeps) walker<NF, CHOL>(p, dsm);
    return;
  }
  // queue of this CTA: [qlo, qhi) of the task array, its own counter
  const bool urgent_q = blockIdx.x <= p.nuw;
  const int qlo = urgent_q ? 0 : p.nurgent, qhi = urgent_q ? p.nurgent : p.ntasks;
  int* qnext = urgent_q ? p.next : p.next + 2;
  if (tid == 0) {
    const int id = qlo + atomicAdd(qnext, 1);
    s_id[0] = id;
    s_task[0] = id < qhi ? p.tasks[id] : kNone;
  }
  __syncthreads();
  // Early fetch hides the queue atomic behind the dependency wait but binds
  // the next task to this CTA while the current one may still be waiting on
  // its inputs (head-of-line blocking); late fetch (warp 0, after its share
  // of the task) keeps queued tasks free for idle CTAs.
  const bool early = (p.pf_mask >> (urgent_q ? 0 : 1)) & 1;
  for (int it = 0;; ++it) {
    const int cur = it & 1;
    const int4 tk = s_task[cur];
    if (warp == 0) {
      int nid = 0;
      if (lane == 0) {
        if (p.trace) s_t0 = globaltimer();
        if (early && tk.x >= 0) nid = qlo + atomicAdd(qnext, 1);
      }
      const bool ok = tk.x >= 0 && wait_deps<CHOL>(p, tk);
      // the polling lanes' acquires reach the other threads through the warp
      // and CTA barriers (both morally strong: causality order is transitive),
      // so no gpu-scope fence here (TT_DAG_FENCE=1 restores one)
      __syncwarp();
      if (lane == 0) {
        if (p.fence) __threadfence();
        s_go = ok;
        if (early) {
          s_id[cur ^ 1] = nid;
          s_task[cur ^ 1] = (tk.x >= 0 && nid < qhi) ? p.tasks[nid] : kNone;
        }
        if (p.trace) s_t1 = globaltimer();
      }
    }
    __syncthreads();
    if (!s_go) break;
    const int kind = tk.x & 3, j = tk.x >> 2, k = task_k0(tk), r0 = tk.z, r1 = tk.w;
    const int kT = k * T;
    double* dk = p.a + static_cast<long long>(kT) * ld + kT;  // diagonal tile (k,k)

    stamp(0);
    stamp(1);
    stamp(2);
    stamp(3);
    if (kind == kGemm && p.pipe) {  // pipelined strips, any q
      stage_b_async<NF, CHOL>(p, sm, j, k, task_q(tk));
      stamp(0);
      // p.eager_sig: 0 none, 1 all GEMM tasks, 2 urgent-queue CTAs only, 3 bulk only
      const bool eager =
          p.eager_sig == 1 || (p.eager_sig == 2 && urgent_q) || (p.eager_sig == 3 && !urgent_q);
      // 32-row strips for large bulk-queue tasks (T <= 40, >= 512 rows: two
      // strips per warp; NODEPS 1.35 -> 1.24 ms on Cholesky XL); the urgent
      // band and smaller tasks keep 16-row strips (finer dataflow: LU N=2000
      // with 400-row tasks measured 3% slower on 32-row strips)
      if (wide_strips_ok(NF) && p.wide && !urgent_q && r1 - r0 >= 512)
        gemm_pipe<NF, CHOL, (wide_strips_ok(NF) ? 4 : kMF)>(p, j, k, task_q(tk), r0, r1, sm, eager,
                                                        (p.trace && warp == 0) ? &s_ph[1] : nullptr);
      else
        gemm_pipe<NF, CHOL, kMF>(p, j, k, task_q(tk), r0, r1, sm, eager,
                                 (p.trace && warp == 0) ? &s_ph[1] : nullptr);
    } else if (kind == kGemm && task_q(tk) > 1) {  // chunked: q steps, K = q*T
      const int q = task_q(tk);
      stage_b<NF, CHOL>(p, sm, j, k, q);
      __syncthreads();
      stamp(0);
      // p.eager_sig: 0 none, 1 all GEMM tasks, 2 urgent-queue CTAs only, 3 bulk only
      const bool eager =
          p.eager_sig == 1 || (p.eager_sig == 2 && urgent_q) || (p.eager_sig == 3 && !urgent_q);
      gemm_task<NF, CHOL>(p, j, k, q, r0, r1, sm, eager, (p.trace && warp == 0) ? &s_ph[1] : nullptr);
    } else if (kind == kGemm) {  // single step
      // B = U(k, j) (LU) or L(j, k)^T (Cholesky), zero-padded to Tp x Tp
      const double* bsrc = CHOL ? p.a + static_cast<long long>(j * T) * ld + kT
                                : p.a + static_cast<long long>(kT) * ld + j * T;
      if (!(T & 1)) {  // element pairs, 16-byte loads; all in flight before any store
        constexpr int kHP = Tp / 2, kPer = (Tp * kHP + kThreads - 1) / kThreads;
        double2 v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int e = tid + u * kThreads, x = e / kHP, y = 2 * (e - x * kHP);  // x: slow index
          v[u] = (e < Tp * kHP && x < T && y < T)
                     ? __ldcg(reinterpret_cast<const double2*>(bsrc + static_cast<long long>(x) * ld + y))
                     : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int e = tid + u * kThreads, x = e / kHP, y = 2 * (e - x * kHP);
          if (e < Tp * kHP) {
            if (CHOL) {  // B[k][n] = L[n][k]
              sm[y * kNP + x] = v[u].x;
              sm[(y + 1) * kNP + x] = v[u].y;
            } else {
              *reinterpret_cast<double2*>(sm + x * kNP + y) = v[u];
            }
          }
        }
      } else {  // all loads in flight before any store: one L2 round trip
        constexpr int kPer = (Tp * Tp + kThreads - 1) / kThreads;
        double v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int e = tid + u * kThreads, x = e / Tp, y = e - x * Tp;  // x: slow index
          v[u] = (e < Tp * Tp && x < T && y < T) ? __ldcg(bsrc + static_cast<long long>(x) * ld + y)
                                                 : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int e = tid + u * kThreads, x = e / Tp, y = e - x * Tp;
          if (e < Tp * Tp) {
            if (CHOL)
              sm[y * kNP + x] = v[u];  // B[k][n] = L[n][k]
            else
              sm[x * kNP + y] = v[u];
          }
        }
      }
      __syncthreads();
      stamp(0);
      StripOps op;
      op.A0 = p.a + static_cast<long long>(r0) * ld + kT;
      op.lda = ld;
      op.C0 = p.a + static_cast<long long>(r0) * ld + j * T;
      op.ldc = ld;
      op.cj = j;
      op.gemm = true;
      op.beta = true;
      // p.eager_sig: 0 none, 1 all GEMM tasks, 2 urgent-queue CTAs only, 3 bulk only
      op.eager = p.eager_sig == 1 || (p.eager_sig == 2 && urgent_q) || (p.eager_sig == 3 && !urgent_q);
      gemm_strips<NF>(p, r0, r1, k, op, sm, abuf + warp * 2 * kABuf, CHOL,
                      (p.trace && warp == 0) ? &s_ph[1] : nullptr);
    } else {  // TRSM
      const bool lsolve = kind == kTrsmL;
      {  // M from the factored diagonal tile (one batched L2 round trip), then
         // the inverses of its 8x8 diagonal blocks (no divisions: DIAG(k)
         // published the diagonal reciprocals)
        const bool upper = !CHOL && lsolve, unit = !CHOL && !lsolve;
        constexpr int kPer = (Tp * Tp + kThreads - 1) / kThreads;
        double v[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {  // element (x, y) of the tile, row-contiguous
          const int e = tid + u * kThreads, x = e / Tp, y = e - x * Tp;
          const bool need = e < Tp * Tp && x < T && y < T && (upper ? y > x : y < x);
          v[u] = need ? __ldcg(dk + static_cast<long long>(x) * ld + y) : 0.0;
        }
        const double* rdg = p.solve + static_cast<long long>(k) * kSolveSlot;
        if (tid < Tp) minv[8 * 64 + tid] = tid < T ? __ldcg(rdg + tid) : 1.0;  // 1/diag
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int e = tid + u * kThreads, x = e / Tp, y = e - x * Tp;
          if (e < Tp * Tp) {
            // M[kk][c]: U11 (upper) or L11^T; diagonal: 1 if unit / padding, else 1/rdiag
            if (upper) sm[x * kNP + y] = v[u];
            else sm[y * kNP + x] = v[u];
          }
        }
        __syncthreads();  // (M's diagonal is never read: the solve applies inv(M_bb))
        const int job = tid >> 3, c = tid & 7;
        if (job < NF) {  // inverse of block `job`, column c: back substitution
          const int b = job;
          double xr[8];
#pragma unroll
          for (int ii = 7; ii >= 0; --ii) {
            double acc = ii == c ? 1.0 : 0.0;
#pragma unroll
            for (int m = 7; m > ii; --m) acc = fma(-sm[(8 * b + ii) * kNP + 8 * b + m], xr[m], acc);
            const int gi = 8 * b + ii;
            xr[ii] = acc * ((unit || gi >= T) ? 1.0 : minv[8 * 64 + gi]);
          }
#pragma unroll
          for (int ii = 0; ii < 8; ++ii) minv[b * 64 + ii * 8 + c] = xr[ii];
        }
      }
      __syncthreads();
      stamp(0);
      stamp(1);
      if (lsolve) {
        for (int ra = r0 + warp * kStrip; ra < r1; ra += kWarps * kStrip) {
          const int nr = min(kStrip, r1 - ra);
          if (!strip_deps(p, ra, ra + nr, k, k, -1, true)) break;
          warp_trsm<NF>(p.a + static_cast<long long>(ra) * ld + kT, ld, 1, nr, T, sm, minv);
          warp_signal(p, ra, ra + nr, k);
        }
      } else {  // U12 tile (k, j): strip rows are the tile's columns
        for (int c0 = warp * kStrip; c0 < T; c0 += kWarps * kStrip) {
          const int nc = min(kStrip, T - c0);
          warp_trsm<NF>(dk + static_cast<long long>(j - k) * T + c0, 1, ld, nc, T, sm, minv);
          __syncwarp();
          if (lane == 0) red_release_add(&p.cnt[k * nt + j], nc);
        }
      }
    }
    if (!early && warp == 0 && lane == 0) {
      const int nid = qlo + atomicAdd(qnext, 1);
      s_id[cur ^ 1] = nid;
      s_task[cur ^ 1] = nid < qhi ? p.tasks[nid] : kNone;
    }
    __syncthreads();  // shared tiles and the task slot are reused next iteration
    if (p.trace && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* tr = p.trace + 8 * static_cast<long long>(s_id[cur]);
      tr[0] = s_t0;
      tr[1] = s_t1;
      tr[2] = globaltimer();
      tr[3] = smid;
      tr[4] = s_ph[0];
      tr[5] = s_ph[1];
      tr[6] = s_ph[2];
      tr[7] = s_ph[3];
    }
  }
}

template <int NF, bool CHOL>
cudaError_t optin() {
  static std::atomic<unsigned long long> configured{0};  // one bit per device
  return smem_optin(dag_kernel<NF, CHOL>, kSmemBytes, configured);
}

template <int NF, bool CHOL>
cudaError_t launch(const Params& prm, int grid, cudaStream_t s) {
  const cudaError_t e = optin<NF, CHOL>();
  if (e != cudaSuccess) return e;
  // Cooperative launch: all CTAs are co-resident before any runs.  The CTAs
  // spin on each other's counters, so a partially resident grid (another
  // context's persistent kernel holding SMs, e.g. two tuning workers on one
  // GPU) could otherwise wait on tasks no resident CTA serves.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dag_kernel<NF, CHOL>, prm);
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

template <bool CHOL>
cudaError_t optin_all() {
  cudaError_t e = optin<1, CHOL>();
  if (e == cudaSuccess) e = optin<2, CHOL>();
  if (e == cudaSuccess) e = optin<3, CHOL>();
  if (e == cudaSuccess) e = optin<4, CHOL>();
  if (e == cudaSuccess) e = optin<5, CHOL>();
  if (e == cudaSuccess) e = optin<6, CHOL>();
  if (e == cudaSuccess) e = optin<7, CHOL>();
  if (e == cudaSuccess) e = optin<8, CHOL>();
  return e;
}

long long count_tasks(bool chol, int n, int by, int bx) {
  bx = tile_for(n, bx);
  if (bx == 0) return kMaxTasks + 1;
  by = region_rows(by, bx);
  const int nt = n / bx;
  long long total = 0;
  for (int k = 0; k + 1 < nt; ++k) {
    const int pe = (k + 1) * bx;
    const long long regions = (n - 1) / by - pe / by + 1;
    const long long cols = nt - k - 1;
    // + carved pieces; chunked and single GEMMs may each split a region in two runs
    total += regions + (chol ? 0 : cols) + 4 * regions * cols + 4;
  }
  return total;
}

}  // namespace

cudaError_t configure_device() {
  const cudaError_t e = optin_all<false>();
  return e != cudaSuccess ? e : optin_all<true>();
}

// Knob -> persistent schedule.  The reference's panel width
// bx (kernels.cpp:181-182) is the rank of the bulk trailing update; the
// diagonal chain is blocked at T <= 64 (what the walker's shared-memory tiles
// hold), like LAPACK factoring an nb-wide panel with an inner blocking:
//   8 <= bx <= 64: T = bx;
//   bx > 64:       T = the largest divisor of bx in [8, 64], bulk tiles take
//                  their updates bx/T steps at a time (rank bx, as in the reference);
//   bx < 8:        T = the smallest multiple of bx in [8, 64] dividing n (the
//                  8-wide DMMA atom: sub-atom panels are packed, as 3mm packs
//                  sub-atom regions).
// 0 when no such T exists (the graph schedule runs).
int tile_for(int n, int bx) {
  if (bx < 1 || n % bx) return 0;
  if (bx >= kMinTile && bx <= kMaxTile) return bx;
  if (bx > kMaxTile) {
    for (int t = kMaxTile; t >= kMinTile; --t)
      if (bx % t == 0) return t;
    return 0;
  }
  for (int t = bx * ((kMinTile + bx - 1) / bx); t <= kMaxTile; t += bx)
    if (n % t == 0) return t;
  return 0;
}

// The reference's trailing row tile by (kernels.cpp:205-216) is the row
// extent of the update / solve tasks, packed to at least
// max(kMinRegion, kMinTaskElems / T) rows (one 16-row strip per warp, and
// enough output elements per task for narrow tiles): a CTA owns adjacent
// by-row regions, as the GEMM packs sub-atom knob regions.
int region_rows(int by, int T) {
  if (by < 1 || T < 1) return 0;
  const char* v = std::getenv("TT_DAG_MINROWS");  // tuning aid: minimum task rows
  const int mr = v && std::atoi(v) > 0 ? std::atoi(v) : kMinRegion;
  const int lo = std::max(mr, (kMinTaskElems + T - 1) / T);
  return by >= lo ? by : by * ((lo + by - 1) / by);
}

bool eligible(int n, int by, int bx) {
  if (by < 1 || n % by || tile_for(n, bx) == 0) return false;
  return count_tasks(false, n, by, bx) <= kMaxTasks;
}

// The walker CTA owns DIAG(k), L(k+1,k), U(k,k+1) and the update of the
// diagonal tiles; the queue holds everything else: per step k the L21 row
// regions below tile row k+1, the U12 tiles right of column k+1, and the
// trailing GEMM regions.  Row regions are `by` rows (the reference's
// trailing row tile, kernels.cpp:205-216) aligned to multiples of by and
// clipped to the trailing rows, so a region's tiles are updated by the same
// region task at every step.
//
// Width (in tiles beyond the walker's) of the band carved into the urgent
// queue; TT_DAG_BAND overrides (tuning aid).
int urgent_band() {
  static const int b = [] {
    const char* v = std::getenv("TT_DAG_BAND");
    const int x = v ? std::atoi(v) : 0;
    return x >= 1 && x <= 16 ? x : 3;
  }();
  return b;
}

// TT_DAG_PREFETCH: bit 0 urgent, bit 1 bulk queue CTAs fetch early (default 0: both late).
int prefetch_mask() {
  static const int m = [] {
    const char* v = std::getenv("TT_DAG_PREFETCH");
    return v ? (std::atoi(v) & 3) : 0;
  }();
  return m;
}

// TT_DAG_MERGE="rows,thresh": steps with >= thresh GEMM region-tasks group
// consecutive row regions into GEMM tasks of >= rows rows (rows 0: off).
// Round 1 (step-by-step updates) used 750,250 (profiles/dag_merge_sweep_r01.txt);
// with chunked bulk updates (K = d*bx) merging measured slower, so the
// default is off (profiles/chunk_sweep_r02.txt).
struct GemmMerge {
  int rows = 0;  // off: with chunked bulk updates merging measured slower (profiles/chunk_sweep_r02.txt)
  long long thresh = 250;
};
GemmMerge gemm_merge() {
  static const GemmMerge g = [] {
    GemmMerge r;
    if (const char* v = std::getenv("TT_DAG_MERGE")) {
      int f = 0;
      long long t = 0;
      if (std::sscanf(v, "%d,%lld", &f, &t) >= 1 && f >= 0) {
        r.rows = f;
        r.thresh = t;
      }
    }
    return r;
  }();
  return g;
}

// Chunk depth: steps per bulk GEMM task, K = d*T ~ 200 (TT_DAG_CHUNK=d
// overrides; 1 = step-by-step updates), capped by the shared memory the q
// stacked B tiles take.
// TT_DAG_PIPE=0: GEMM tasks on the register path (A/B aid); default gemm_pipe.
bool pipe_gemm() {
  const char* v = std::getenv("TT_DAG_PIPE");  // read per workspace / launch (tests vary it)
  return !(v && v[0] == '0');
}

int chunk_depth(int n, int bx) {
  const int T = tile_for(n, bx);
  if (T == 0) return 1;
  const int tp = (T + 7) / 8 * 8;
  // the q stacked B tiles share the CTA's shared memory with gemm_pipe's rings
  const int room = kBudget - (pipe_gemm() ? ring_doubles(tp / 8) + 2 : 0);
  const int cap = std::max(1, room / (tp * std::max(bstride(tp, true), bstride(tp, false))));
  const char* v = std::getenv("TT_DAG_CHUNK");  // read per workspace (tests vary it)
  const int forced = v ? std::atoi(v) : 0;
  const int d = forced >= 1 ? forced : bx > kMaxTile ? bx / T : (200 + T / 2) / T;
  return std::max(1, std::min({d, cap, 0xFFFF / 2}));
}

// Two queues.  Every task has a ready step — the last panel step whose output
// it reads (TRSM_L/U(k): k; a GEMM over steps [k0, k0+q): k0+q-1) — and a
// deadline — the earliest ready step of any task (or walker step) consuming
// its output: TRSM(k): k; a single-step GEMM at step s: s+1; a chunk: the
// next chunk's ready step, or for a tile's last chunk its first single step
// (dag_factor.cuh).  Each queue is sorted by the key (deadline, ready step,
// TRSM before GEMM), generation order breaking ties.  A producer Y of a
// consumer X has deadline(Y) <= ready(X) <= deadline(X), equal keys only for
// a same-step TRSM -> GEMM pair, so the key order is a topological order of
// the task DAG, and the walker's step k consumes only tasks with deadline
// <= k while every task waiting on walker step k has ready step >= k:
// deadlock-free with in-order queues for any number of CTAs (the earliest
// unfinished task in key order always has its inputs done and is taken next
// in its queue).  The deadline order lets the queues serve what the diagonal
// chain needs next first: a chunk burst (every d steps) no longer delays the
// single-step updates of the next panel columns.
//
// The urgent queue (served by a few dedicated CTAs) holds what the walker
// needs next — the L21 rows of tile rows <= r+band and the U / GEMM pieces of
// tile columns <= r+band above the carve row (r+1+band)*bx — the bulk queue
// the rest.  Row regions are `by` rows (the reference's trailing row tile,
// kernels.cpp:205-216) aligned to multiples of by and clipped to the trailing
// rows; a GEMM region is further split at the tiles where the (chunk /
// single step) stage structure changes (dag_factor.cuh).
// Returns urgent ++ bulk; *n_urgent = urgent count.
std::vector<int4> build_tasks(bool chol, int n, int by, int bx, int* n_urgent) {
  const int d = chunk_depth(n, bx);
  bx = tile_for(n, bx);
  by = region_rows(by, bx);
  const int T = bx, nt = n / bx;
  const int band = urgent_band();
  const GemmMerge gm = gemm_merge();
  struct Keyed {
    int dl, ready, kind;
    int4 t;
  };
  std::vector<Keyed> urg, bulk;
  bulk.reserve(static_cast<size_t>(count_tasks(chol, n, by, bx)));
  // chunk of column jj (phase o = jj mod d) that closes at step r+1, if any:
  // [k0, r+1) with q = r+1-k0
  auto chunk_closing = [&](int jj, int r, int* k0) {
    const int o = jj % d, b = r + 1;
    if (d == 1) return false;
    if (o > 0 && b == o) {
      *k0 = 0;
      return true;
    }
    if (b > o && b >= d && (b - o) % d == 0) {
      *k0 = b - d;
      return true;
    }
    return false;
  };
  // is [k0, k0+q) one stage of tile (i, j)?  (a chunk of column j ending at or
  // before the tile's first single step, or a single step before m)
  auto is_stage = [&](int i, int jj, int k0, int q, bool chunk) {
    const int m = std::min(i, jj), e = chunk_end(m, d, jj % d);
    return chunk ? k0 + q <= e : (q == 1 && k0 >= e && k0 < m);
  };
  // earliest ready step of the next stage of tile (i, j) after [k0, k0+q)
  auto deadline = [&](int i, int jj, int k0, int q, bool chunk) {
    if (!chunk) return k0 + 1;
    const int e = chunk_end(std::min(i, jj), d, jj % d), end = k0 + q;
    return end < e ? end + d - 1 : e;  // the next chunk's ready step, or the first single
  };
  for (int r = 0; r + 1 < nt; ++r) {
    const int pe = (r + 1) * T;
    const int carve = std::min(n, (r + 1 + band) * T);  // rows above: tile rows <= r+band
    auto task = [&](int kind, int r0, int r1, int j, int k0, int q, int dl) {
      if (r0 >= r1) return;
      const int y = k0 | (q << 16);
      const int ko = kind == kGemm ? 1 : 0;
      const bool near = kind == kTrsmU ? j <= r + band : (kind == kTrsmL || j <= r + band);
      if (near && r0 < carve) {  // split at the carve row
        urg.push_back({dl, r, ko, make_int4(kind | (j << 2), y, r0, kind == kTrsmU ? r1 : std::min(r1, carve))});
        if (kind != kTrsmU && r1 > carve)
          bulk.push_back({dl, r, ko, make_int4(kind | (j << 2), y, carve, r1)});
      } else {
        bulk.push_back({dl, r, ko, make_int4(kind | (j << 2), y, r0, r1)});
      }
    };
    std::vector<std::pair<int, int>> reg;  // row regions: multiples of by, clipped
    for (int x = (pe / by) * by; x < n; x += by) reg.emplace_back(std::max(x, pe), std::min(n, x + by));
    for (const auto& rg : reg) task(kTrsmL, std::max(rg.first, pe + T), rg.second, 0, r, 1, r);  // row r+1: walker
    if (!chol)
      for (int j = r + 2; j < nt; ++j) task(kTrsmU, 0, 1, j, r, 1, r);
    // GEMMs ready at step r, per tile column: the single step r, and the
    // column's chunk closing at r+1 (if its phase puts a boundary there)
    const int ncols = nt - r - 1, nreg = static_cast<int>(reg.size());
    const bool merge = gm.rows > 0 && static_cast<long long>(nreg) * ncols >= gm.thresh;
    // row regions outer: a region's GEMMs need only that region's L21 rows
    // (plus the U12 tiles), so the first GEMMs taken are the first ready.
    // Steps with many GEMM tasks may group consecutive regions into one
    // single-step task (TT_DAG_MERGE; off by default).
    for (int pass = 0; pass < 2; ++pass) {  // singles, then chunks
      const bool chunk = pass == 1;
      for (int g0 = 0, g1; g0 < nreg; g0 = g1) {
        g1 = g0 + 1;  // regions [g0, g1) form one task: at least gm.rows rows when merging
        while (merge && !chunk && g1 < nreg && reg[g1 - 1].second - reg[g0].first < gm.rows) ++g1;
        const int lo = reg[g0].first, hi = reg[g1 - 1].second;
        for (int j = r + 1; j < nt; ++j) {
          int k0 = r, q = 1;
          if (chunk) {
            if (!chunk_closing(j, r, &k0)) continue;
            q = r + 1 - k0;
          }
          int r0 = std::max(lo, chol ? j * T : pe);  // Cholesky: lower triangle only
          if (!chunk && j == r + 1) r0 = std::max(r0, pe + T);  // tile (r+1,r+1): the walker
          // maximal runs of tiles for which [k0, k0+q) is a stage
          for (int x = r0; x < hi;) {
            const int i = x / T;
            const int xe = std::min(hi, (i + 1) * T);
            if (!is_stage(i, j, k0, q, chunk)) {
              x = xe;
              continue;
            }
            int y = xe, dl = deadline(i, j, k0, q, chunk);
            while (y < hi && is_stage(y / T, j, k0, q, chunk)) {
              dl = std::min(dl, deadline(y / T, j, k0, q, chunk));
              y = std::min(hi, (y / T + 1) * T);
            }
            task(kGemm, x, y, j, k0, q, dl);
            x = y;
          }
        }
      }
    }
  }
  auto order = [](std::vector<Keyed>& v) {
    std::stable_sort(v.begin(), v.end(), [](const Keyed& a, const Keyed& b) {
      if (a.dl != b.dl) return a.dl < b.dl;
      if (a.ready != b.ready) return a.ready < b.ready;
      return a.kind < b.kind;
    });
  };
  order(urg);
  order(bulk);
  std::vector<int4> out;
  out.reserve(urg.size() + bulk.size());
  for (const auto& k : urg) out.push_back(k.t);
  for (const auto& k : bulk) out.push_back(k.t);
  if (n_urgent) *n_urgent = static_cast<int>(urg.size());
  return out;
}

cudaError_t create(Workspace* w, bool chol, int n, int by, int bx) {
  int nurg = 0;
  const std::vector<int4> tasks = build_tasks(chol, n, by, bx, &nurg);
  w->T = tile_for(n, bx);
  const int nt = n / w->T;
  w->ntasks = static_cast<int>(tasks.size());
  w->nurgent = nurg;
  w->chunk = chunk_depth(n, bx);
  w->pipe = pipe_gemm() ? 1 : 0;
  w->nsteps = nt;
  // nt*nt tile counters, then: urgent next, abort flag, bulk next, and the
  // started-CTA count, and the watchdog record {recorded, cta, counter, need, seen,
  // urgent pos, bulk pos, polls, ms, started, grid} (kDiagInts)
  w->cnt_bytes = (static_cast<size_t>(nt) * nt + 4 + kDiagInts) * sizeof(int);
  cudaError_t e = cudaMalloc(&w->tasks, tasks.size() * sizeof(int4));
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(w->tasks, tasks.data(), tasks.size() * sizeof(int4), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&w->cnt, w->cnt_bytes);
  if (e != cudaSuccess) return e;
  e = cudaMemset(w->cnt, 0, w->cnt_bytes);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(&w->solve, static_cast<size_t>(nt) * kSolveSlot * sizeof(double));
  if (e != cudaSuccess) return e;

  const char* tr = std::getenv("TT_DAG_TRACE");
  if (tr && tr[0] == '1') {
    e = cudaMalloc(&w->trace, (tasks.size() + nt) * 8 * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // walker + urgent-queue workers + bulk-queue workers
  {
    // measured (tools/gpu_knobs2.sh): with >= 80 panel steps the bulk queue
    // is the bound in the early steps and 4 urgent CTAs beat 8 (Cholesky XL
    // 1.83 -> 1.81 ms, LU XL 3.07 -> 3.01 ms); LU N=2000 (50 steps) wants 6-8
    const char* v = std::getenv("TT_DAG_URGENT_CTAS");
    const int want = v ? std::atoi(v) : (nt >= 80 ? 4 : 8);
    w->nuw = nurg > 0 ? std::max(1, std::min(want, sms / 2)) : 0;
  }
  const int nbulk = w->ntasks - nurg;
  w->grid = 1 + w->nuw + std::max(0, std::min(sms - 1 - w->nuw, nbulk));
  // The uploads and the memset above run on the legacy default stream, which
  // does not order with the context's non-blocking stream: a pageable
  // cudaMemcpy may return before its DMA lands and cudaMemset is asynchronous.
  // Without this wait the first launch of a new workspace could read task
  // descriptors or counters that were still being written (long knob sweeps
  // saw rare watchdog aborts with counters zeroed under a running schedule,
  // and one illegal address).
  e = cudaStreamSynchronize(cudaStreamLegacy);
  if (e != cudaSuccess) return e;
  return cudaSuccess;
}

std::string watchdog_info(const Workspace& w) {
  if (!w.cnt) return {};
  const int nt = w.nsteps;
  int rec[kDiagInts] = {};
  if (cudaMemcpy(rec, w.cnt + static_cast<size_t>(nt) * nt + 4, sizeof(rec),
                 cudaMemcpyDeviceToHost) != cudaSuccess || rec[0] == 0)
    return {};
  char buf[256];
  std::snprintf(buf, sizeof(buf),
                "cta %d waited on tile (%d, %d) for %d rows, saw %d (T %d; queue positions: "
                "urgent %d of %d, bulk %d of %d; %d polls, %d ms; %d of %d CTAs started)",
                rec[1], rec[2] / nt, rec[2] % nt, rec[3], rec[4], w.T, rec[5], w.nurgent, rec[6],
                w.ntasks - w.nurgent, rec[7], rec[8], rec[9], rec[10]);
  return buf;
}

void destroy(Workspace* w) {
  if (w->tasks) cudaFree(w->tasks);
  if (w->cnt) cudaFree(w->cnt);
  if (w->trace) cudaFree(w->trace);
  if (w->solve) cudaFree(w->solve);
  *w = Workspace{};
}

cudaError_t enqueue(const Workspace& w, bool chol, double* a, int n, long long ld, int* info,
                    cudaStream_t s) {
  const int bx = w.T, nt = n / bx;
  static const bool nodeps = [] {
    const char* v = std::getenv("TT_DAG_NODEPS");
    return v && v[0] == '1';
  }();
  const size_t tiles = static_cast<size_t>(nt) * nt * sizeof(int);
  cudaError_t e = cudaMemsetAsync(w.cnt, nodeps ? 0x3F : 0, tiles, s);
  // queue positions, the abort flag and the started-CTA count; the watchdog
  // record after them is kept across launches (zeroed at create): it names the
  // first timeout
  if (e == cudaSuccess) e = cudaMemsetAsync(w.cnt + static_cast<size_t>(nt) * nt, 0, 4 * sizeof(int), s);
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
  prm.next = w.cnt + static_cast<size_t>(nt) * nt;  // [0] urgent, [2] bulk
  prm.abort = prm.next + 1;
  prm.info = info;
  prm.trace = w.trace;
  prm.nurgent = w.nurgent;
  prm.nuw = w.nuw;
  prm.pf_mask = prefetch_mask();
  prm.nodeps = nodeps ? 1 : 0;
  prm.fence = [] {
    const char* v = std::getenv("TT_DAG_FENCE");
    return v && v[0] == '1' ? 1 : 0;
  }();
  prm.wide = [] {
    const char* v = std::getenv("TT_DAG_WIDE");
    return v && v[0] == '0' ? 0 : 1;
  }();
  prm.pipe = w.pipe;  // fixed at create(): the chunk depth's shared-memory budget depends on it
  prm.d = w.chunk;
  // measured default: publishing each GEMM strip right after its stores
  // (round 1: Cholesky +2%; round 2, 4 urgent CTAs: LU XL 3.01 -> 2.94 ms,
  // LU N=2000 neutral)
  prm.eager_sig = [] {
    const char* v = std::getenv("TT_DAG_EAGER_SIGNAL");
    return v ? std::atoi(v) : 1;
  }();
  prm.solve = w.solve;
  const int nf = (bx + 7) / 8;
  return chol ? launch_nf<true>(nf, prm, w.grid, s) : launch_nf<false>(nf, prm, w.grid, s);
}

}  // namespace dag
}  // namespace tt
