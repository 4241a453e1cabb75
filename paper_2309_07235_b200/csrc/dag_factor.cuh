// Persistent tile-DAG schedule for LU (no pivoting) and Cholesky (sm_100a).
//
// The graph schedule (schedules.cu) issues ~4 dependent launches per panel
// step, so at PolyBench sizes the factorisation is bound by launch and
// panel latency.  This schedule runs the WHOLE factorisation as
// one launch: one CTA per SM pulls tasks from a host-built, priority-ordered
// task list and waits on per-tile completion counters in L2, so the next
// panel's diagonal block is factored while the current trailing update is
// still running (look-ahead), with no kernel boundaries on the critical path.
//
// Tiles are bx x bx (the reference's panel width, kernels.cpp:181-182); the
// trailing-update and panel-solve tasks cover row regions of `by` rows
// anchored at the panel end, exactly the reference's trailing tiling
// (kernels.cpp:205-216).  Task kinds, per panel step k:
//   DIAG(k)           getrf / potrf of tile (k,k) in shared memory
//   TRSM_L(k, rows)   L21 = A21 U11^-1 (LU) / A21 L11^-T (Cholesky)
//   TRSM_U(k, j)      U12 = L11^-1 A12 (LU only)
//   GEMM(k, rows, j)  A(rows, j) -= L(rows, k) * U(k, j)   (Cholesky: L(j,k)^T)
// GEMM and TRSM run on the fp64 tensor cores (DMMA m8n8k4); the triangular
// solves are blocked by 8 columns with 8x8 diagonal-block inverses.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace tt {
namespace dag {

enum TaskKind : int { kDiag = 0, kTrsmL = 1, kTrsmU = 2, kGemm = 3 };

// Chunked trailing updates.  A GEMM task applies the updates of q
// consecutive panel steps [k0, k0+q) to its rows at once (C stays in
// registers; K = q*bx), so the C round trip, the task's dependency waits and
// its operand staging are paid once per q steps.  Tile column j groups its
// steps into chunks ending at the boundaries o, o+d, o+2d, ... with phase
// o = j mod d (the first chunk [0, o) may be short): the columns' chunks
// close on different steps, so the bulk work arrives evenly instead of in a
// burst every d steps.  Tile (i, j), with m = min(i, j) updates before its own
// DIAG/TRSM, gets
//   the chunks of column j that end at or before step m-1,
//   then single steps up to m-1,
// so the last update of every tile — the one the diagonal chain waits for —
// is always a single step.  Each chunk / single / the final op is one
// "stage"; the tile counter counts finished rows over stages.  Per element
// the products are accumulated in ascending step order in both cases: the
// result is bitwise that of step-by-step updates (same DMMA sequence).
// Number of chunks of a tile with m updates in a column of phase o.
__host__ __device__ inline int nchunks(int m, int d, int o) {
  if (m < 1 || d <= 1) return 0;  // d = 1: every update a single step
  if (o == 0) return (m - 1) / d;
  return o <= m - 1 ? 1 + (m - 1 - o) / d : 0;
}
// End (exclusive) of the last chunk: the first single step.
__host__ __device__ inline int chunk_end(int m, int d, int o) {
  const int nc = nchunks(m, d, o);
  if (o == 0) return nc * d;
  return nc == 0 ? 0 : o + (nc - 1) * d;
}
// Stages of a tile with m updates that cover the steps < s (s a chunk
// boundary or a single step of that tile, s <= m).
__host__ __device__ inline int stages_before(int m, int s, int d, int o) {
  const int e = chunk_end(m, d, o);
  if (s > e) return nchunks(m, d, o) + (s - e);
  if (s == 0) return 0;
  return o == 0 ? s / d : 1 + (s - o) / d;
}
// Stages of a tile with m updates, its final DIAG/TRSM included.
__host__ __device__ inline int stages_total(int m, int d, int o) {
  return stages_before(m, m, d, o) + 1;
}

// Widest tile the persistent kernel handles (the diag block is factored by
// the warp-register code of diag_factor.cuh, <= 64).
constexpr int kMaxTile = 64;
constexpr int kMinTile = 8;
constexpr int kMinRegion = 128;      // rows per update / solve task, at least ...
constexpr int kMinTaskElems = 5120;  // ... and output elements (rows x T)
constexpr long long kMaxTasks = 8LL << 20;

// Watchdog: a dependency wait longer than this aborts the schedule with
// info = kTimeout (a scheduling bug must never hang the GPU).
constexpr long long kWatchdogNs = 4000000000LL;
constexpr int kTimeout = -2147483647 - 1;  // INT_MIN
// Ints after the abort flag kept for the watchdog record (see watchdog_info).
constexpr int kDiagInts = 11;


// Opts every persistent-kernel variant into its shared memory on the
// current device (called per context: the attribute is per device).
cudaError_t configure_device();

// True when the persistent schedule covers (n, by, bx).
bool eligible(int n, int by, int bx);
// Tile T the schedule runs for panel width bx (0: none), and the row extent
// of its update / solve tasks for row tile by (see dag_factor.cu).
int tile_for(int n, int bx);
int region_rows(int by, int T);

// Host-built task list in dependency-respecting priority order
// (int4 {kind | j << 2, k, r0, r1}).
// Urgent queue first, then bulk; *n_urgent (may be null) gets the urgent count.
// (int4 {kind | j << 2, k0 | q << 16, r0, r1}: GEMM tasks apply steps
// [k0, k0 + q), every other task q = 1.)
std::vector<int4> build_tasks(bool chol, int n, int by, int bx, int* n_urgent);

// Chunk depth d used for (n, by, bx) (TT_DAG_CHUNK overrides; 1 = step by step).
int chunk_depth(int n, int bx);

struct Workspace {
  int4* tasks = nullptr;   // device task list
  int ntasks = 0;
  int T = 0;               // tile (tile_for(n, bx))
  int nsteps = 0;          // n / T: walker steps (trace rows after the tasks)
  int nurgent = 0;         // urgent-queue tasks (the first nurgent of the list)
  int nuw = 0;             // CTAs serving the urgent queue
  int* cnt = nullptr;      // nt*nt tile counters + urgent counter, abort flag, bulk counter
  size_t cnt_bytes = 0;
  int grid = 0;
  int chunk = 1;           // chunk depth d
  int pipe = 1;            // GEMM tasks through the shared-memory pipeline (TT_DAG_PIPE)
  unsigned long long* trace = nullptr;  // TT_DAG_TRACE=1: per-task timestamps
  double* solve = nullptr;              // per-step diagonal reciprocals written by DIAG
};

// Allocates and uploads the workspace for one (kernel, n, by, bx, buffer).
cudaError_t create(Workspace* w, bool chol, int n, int by, int bx);
void destroy(Workspace* w);

// After a kTimeout: "cta C waited on tile (i, j) for N rows, saw V" (synchronous
// read of the workspace; empty when nothing was recorded).
std::string watchdog_info(const Workspace& w);

// Enqueues counter reset + the persistent kernel on `s` (graph-capturable).
cudaError_t enqueue(const Workspace& w, bool chol, double* a, int n, long long ld, int* info,
                    cudaStream_t s);

}  // namespace dag
}  // namespace tt
