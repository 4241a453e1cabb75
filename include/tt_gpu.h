/* tt_gpu.h — C ABI of the B200-native fp64 kernel library (libtt_gpu.so).
 *
 * Drop-in boundary for the reference's timed kernel entry points
 * (/root/reference/proj/core/include/tiletuner/kernels.hpp) and for its
 * run-and-time objective (harness.hpp / harness.cpp:89-164).  The reference
 * has no FFI; its boundary is a C++ free-function API over
 * `tiletuner::Matrix` (dense row-major std::vector<double>, matrix.hpp:9-26).
 * This header replaces it with plain pointers and sizes; the C++ shim in
 * paper_2309_07235_b200/csrc/tiletuner_gpu.hpp re-exports the exact
 * reference signatures on top of it, and INTEGRATION.md shows the one-line
 * change to KernelRunner::run_once.
 *
 * Error convention (no exceptions cross the ABI):
 *   TT_OK        success
 *   TT_EINVAL    -> std::invalid_argument   (bad arity, non-dividing factor,
 *                   non-square input, bad protocol; kernels.cpp:21-34,124-126,
 *                   harness.cpp:81-86)
 *   TT_ENUMERIC  -> tiletuner::NumericalError (|pivot| < 1e-300 or Cholesky
 *                   diag <= 0; kernels.cpp:15,187-190,297-302)
 *   TT_EDEVICE   -> tiletuner::MeasurementError (CUDA error, nonpositive
 *                   timer reading; harness.cpp:133-135)
 *   TT_ENOMEM    device allocation failed
 * tt_last_error(ctx) returns a message in the reference's wording, e.g.
 * "lu_tiled: tile factor 3 does not divide extent 64".
 *
 * Threading: one tt_ctx per host thread; contexts on different devices run
 * concurrently (the batched evaluator uses one per GPU).
 */
#ifndef TT_GPU_H
#define TT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TT_OK = 0,
  TT_EINVAL = 1,
  TT_ENUMERIC = 2,
  TT_EDEVICE = 3,
  TT_ENOMEM = 4,
};

/* Kernel ids follow tiletuner::Kernel (problem.hpp:9): lu, cholesky, mm3. */
enum { TT_KERNEL_LU = 0, TT_KERNEL_CHOLESKY = 1, TT_KERNEL_MM3 = 2 };

/* Aggregates follow tiletuner::Aggregate (harness.hpp:22). */
enum { TT_AGG_MEDIAN = 0, TT_AGG_MIN = 1, TT_AGG_MEAN = 2 };

typedef struct tt_ctx tt_ctx;

/* ---- context: one per GPU, owns a stream, events, device buffers and the
 *      per-config instantiation cache (variant + launch geometry + TMA
 *      descriptors + captured CUDA graph). ---- */
int tt_ctx_create(int device, tt_ctx** out);
int tt_ctx_destroy(tt_ctx* ctx);
const char* tt_last_error(const tt_ctx* ctx);
int tt_ctx_device(const tt_ctx* ctx);
/* Number of cached instantiations (graphs) currently held. */
int tt_cache_size(const tt_ctx* ctx);

/* ---- one-shot drop-ins for the reference entry points (host buffers).
 *      Each uploads, runs the sm_100a schedule for the knob setting and
 *      downloads the result.  Semantics match the reference exactly:
 *      validation order, in-place packed LU (kernels.cpp:178-218),
 *      lower-only Cholesky with the upper triangle untouched
 *      (kernels.cpp:264-308), fresh zero-initialised G (kernels.cpp:122-131). */

/* kernels.hpp:65  void lu_factor_inplace(Matrix& a, int by, int bx) */
int tt_lu_factor_inplace(tt_ctx* ctx, double* a, int rows, int cols, int by,
                         int bx, int* fail_index);
/* kernels.hpp:66  void cholesky_factor_inplace(Matrix& a, int by, int bx) */
int tt_cholesky_factor_inplace(tt_ctx* ctx, double* a, int rows, int cols,
                               int by, int bx, int* fail_index);
/* Pipelined batches of the two drop-ins: `count` row-major n x n host
 * matrices (page-locked for full overlap), each factored in place; upload,
 * factorisation and download of neighbouring matrices overlap (three
 * device buffers).  fail_index (count entries, may be NULL) gets
 * each matrix's failing column or -1; the status is that of the first
 * failing matrix. */
int tt_lu_factor_batch(tt_ctx* ctx, double* const* mats, int count, int n,
                       int by, int bx, int* fail_index);
int tt_cholesky_factor_batch(tt_ctx* ctx, double* const* mats, int count,
                             int n, int by, int bx, int* fail_index);
/* kernels.hpp:43  Matrix mm3_tiled(a, b, c, d, const Configuration&)
 * dims (n,l,m,o,p) positional: A n x l, B l x m, C m x o, D o x p, G n x p. */
int tt_mm3_tiled(tt_ctx* ctx, const double* a, const double* b,
                 const double* c, const double* d, int n, int l, int m, int o,
                 int p, const int* cfg, int ncfg, double* g);

/* ---- objective harness (KernelRunner twin, harness.cpp:89-143).
 *      setup uploads the case's inputs once per tuning run (the ctor);
 *      run executes one schedule on a fresh copy; measure times
 *      `warmups` + `reps` runs with CUDA events on the context stream
 *      (D2D restore of the pristine input outside the event pair) and
 *      reduces them like aggregate_samples (harness.cpp:53-71). */
int tt_setup_host(tt_ctx* ctx, int kernel, int n, int l, int m, int o, int p,
                  const double* a, const double* b, const double* c,
                  const double* d);
/* Same case generated on the device, bitwise equal to gen_spd /
 * gen_3mm_inputs (kernels.cpp:38-69): mt19937_64 draws on the host, the
 * B*B^T + n*I product on the device in ascending-k, unfused order. */
int tt_setup_seeded(tt_ctx* ctx, int kernel, int n, int l, int m, int o, int p,
                    uint64_t seed);
/* Runs the schedule once on a fresh copy; `out` (host, may be NULL) gets
 * the packed LU / the factored matrix / G. */
int tt_run(tt_ctx* ctx, const int* cfg, int ncfg, double* out, int* fail_index);
int tt_measure(tt_ctx* ctx, const int* cfg, int ncfg, int warmups, int reps,
               int aggregate, double* seconds);
/* Like tt_measure but returns every timed sample (reps of them). */
int tt_measure_samples(tt_ctx* ctx, const int* cfg, int ncfg, int warmups,
                       int reps, double* samples);
/* Downloads the setup's pristine input (A for lu/cholesky, A,B,C,D for 3mm
 * when the pointers are non-NULL). */
int tt_get_input(tt_ctx* ctx, double* a, double* b, double* c, double* d);
/* Device-side residuals of the last tt_run output against the pristine input:
 * max|L*U - A| / max|A| (kernels.cpp:326-338), max|L*L^T - A| / max|A|
 * (:340-352).  For 3mm, max|G - ref| / max|ref| against `ref_g` (host). */
int tt_residual(tt_ctx* ctx, const double* ref_g, double* out);

/* ---- device-pointer API (inputs already resident; used by the bench and
 *      the sharded 3mm driver).  `stream` is a cudaStream_t (NULL = the
 *      context stream).  Matrices are row-major with leading dimension
 *      ld >= cols, ld even, base 16-byte aligned. ---- */
int tt_dev_lu(tt_ctx* ctx, double* a, int n, int ld, int by, int bx,
              int* fail_index, void* stream);
int tt_dev_cholesky(tt_ctx* ctx, double* a, int n, int ld, int by, int bx,
                    int* fail_index, void* stream);
/* 3mm on resident operands; e and f are caller-provided scratch. */
int tt_dev_mm3(tt_ctx* ctx, const double* a, int lda, const double* b,
               int ldb, const double* c, int ldc, const double* d, int ldd,
               double* e, int lde, double* f, int ldf, double* g, int ldg,
               int n, int l, int m, int o, int p, const int* cfg, int ncfg,
               void* stream);
/* One knob-driven fp64 DMMA GEMM: C (+)= alpha * A[M x K] * B[K x N]
 * (b_trans: B given as N x K).  beta in {0,1}, alpha in {+1,-1}; (fy, fx) is
 * the output region per CTA (the reference's (yo,xo) tile). */
int tt_dev_gemm(tt_ctx* ctx, const double* a, int lda, const double* b,
                int ldb, int b_trans, double* c, int ldc, int M, int N, int K,
                int fy, int fx, int alpha, int beta, void* stream);

/* Shard-invariant device input generator for the scaled 3mm (no CPU oracle
 * exists at N = 32768): element (i, j) of rows [row0, row0+rows) of global
 * matrix `stream_id` is splitmix64(seed, stream_id, row0+i, j) >> 11 * 2^-53. */
int tt_dev_fill_uniform(tt_ctx* ctx, double* a, int rows, int cols, int ld, long long row0,
                        uint64_t seed, int stream_id, void* stream);

/* Persistent tile-DAG schedule (dag_factor.cu), host-side introspection:
 * writes up to `cap` tasks as int quadruples {kind | j << 2, k0 | q << 16,
 * r0, r1} (kind 0 DIAG, 1 TRSM_L, 2 TRSM_U, 3 GEMM; a GEMM applies the
 * updates of panel steps [k0, k0+q) to rows [r0, r1) of tile column j, every
 * other task has q = 1) and returns the task count, or -1 when (n, by, bx)
 * runs on the launch-per-kernel graph schedule instead.  Needs no device. */
int tt_dag_tasks(int kernel, int n, int by, int bx, int* out, int cap);
/* Chunk depth d of that schedule: bulk tiles receive their updates d steps
 * at a time (K = d * T, T = tt_dag_tile), the last 1..d steps of each tile
 * singly; -1 when the graph schedule runs. */
int tt_dag_chunk_depth(int n, int by, int bx);
/* Tile T of that schedule for panel width bx: bx itself for 8 <= bx <= 64,
 * the largest divisor of bx in [8, 64] for wider panels (whose bulk tiles
 * take bx/T steps per update, the reference's rank-bx trailing update), the
 * smallest multiple of bx in [8, 64] dividing n for bx < 8; -1 when the
 * graph schedule runs. */
int tt_dag_tile(int n, int by, int bx);
/* Row extent of that schedule's update / solve tasks: by packed to at least
 * max(128, 5120 / T) rows (adjacent by-row regions per task); -1 when the
 * graph schedule runs. */
int tt_dag_region_rows(int n, int by, int bx);
/* DMMA GEMM (3mm, graph-schedule updates), host-side introspection: the CTA
 * region a knob region (fy, fx) of an m x n product maps to and the tile
 * variant that sweeps it — out = {reg_y, reg_x, bm, bn, consumer warps}.
 * Knob edges in [32, 128] are kept; smaller ones are packed (floor(64 / f)
 * knob regions per CTA region), larger ones split into equal parts <= 128
 * (replaces the reference's matmul_tiled outer loops, kernels.cpp:91-111).
 * Needs no device. */
int tt_gemm_plan(int m, int n, int fy, int fx, int* out);
/* Number of leading tasks of that list forming the urgent queue (the rest is
 * the bulk queue); -1 when the graph schedule runs instead. */
int tt_dag_urgent(int kernel, int n, int by, int bx);

/* With TT_DAG_TRACE=1 in the environment the persistent schedule records,
 * per task, {fetch, dependencies-ready, done} (%globaltimer ns) and the SM
 * id and four phase stamps; this copies the most recently run schedule's
 * trace (8 u64 per task, in task-list order, then one row per walker step:
 * start, tile ready, updated, factored, panel ready, panel published) and
 * returns the row count (-1: no trace). */
int tt_dag_trace(tt_ctx* ctx, unsigned long long* out, int cap);

/* Counter of kernel launches issued by this context (graph nodes count once
 * per graph launch); the bench reports it as gpu_launches. */
uint64_t tt_launch_count(const tt_ctx* ctx);

/* Library build info ("sm_100a ..."). */
const char* tt_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TT_GPU_H */
