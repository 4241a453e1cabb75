// libtt_gpu.so — C ABI (include/tt_gpu.h) over the sm_100a kernels.
//
// Owns the per-GPU context: streams, events, device buffers laid out for
// HBM (row-major, leading dimension padded to 16 doubles = 128 B so every
// row starts on a TMA/L2-sector boundary), the status word for numerical
// failures, and the per-config instantiation cache: one captured
// CUDA graph per (kernel, buffer, shape, knob setting), each holding its
// TMA descriptors and launch geometry.  No CPU fallback: every compute entry
// point requires the CUDA device and fails with TT_EDEVICE without one.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tt_gpu.h"
#include "dag_factor.cuh"
#include "factor_kernels.cuh"
#include "gemm.hpp"
#include "schedules.cuh"

namespace {

constexpr int kLdAlign = 16;  // doubles: 128-byte rows

long long padded_ld(int cols) {
  return (static_cast<long long>(cols) + kLdAlign - 1) / kLdAlign * kLdAlign;
}

struct DevMat {
  double* p = nullptr;
  int rows = 0, cols = 0;
  long long ld = 0;
  size_t capacity = 0;  // bytes
  size_t bytes() const { return static_cast<size_t>(rows) * ld * sizeof(double); }
};

enum GraphKind { kGraphLu = 0, kGraphChol = 1, kGraphMm3 = 2 };

// (kind, every buffer address, shape, knobs): a graph bakes in pointers and TMA maps.
using GraphKey = std::tuple<int, std::vector<long long>>;

}  // namespace

struct tt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr, stream2 = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, fork = nullptr, join = nullptr;
  std::string err;
  // setup (KernelRunner twin)
  int kernel = -1;
  int dims[5] = {0, 0, 0, 0, 0};
  DevMat pristine[4];  // lu/chol: [0] = A ; mm3: A, B, C, D
  DevMat work;         // lu/chol factorisation target
  DevMat e, f, g;      // mm3 outputs
  DevMat scratch_l, scratch_u;  // residual workspaces
  DevMat oneshot;      // one-shot drop-in buffer
  DevMat batch[3];     // triple-buffered device matrices of the pipelined batch API
  cudaStream_t cin = nullptr, cout = nullptr;  // batch copy streams (H2D, D2H)
  DevMat oneshot_in[4];
  int* info = nullptr;           // device status word
  int* info_host = nullptr;      // pinned mirror(s)
  int info_host_slots = 0;
  unsigned long long* red = nullptr;  // residual reduction slots
  double* ws = nullptr;          // panel scratch (kIB x kIB)
  tt::TmapCache tmaps;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, long long> graph_nodes;
  std::map<GraphKey, tt::dag::Workspace> dag_ws;  // persistent-schedule task lists + counters
  const tt::dag::Workspace* dag_last = nullptr;    // most recently enqueued (for tt_dag_trace)
  unsigned long long launches = 0;
  bool have_output = false;
};

namespace {

int fail(tt_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

// Makes the context's device current for the scope of a device-pointer entry
// point and restores the caller's device afterwards (the caller's thread may
// have another GPU current: the workspace allocation and the SM count of the
// persistent schedule, and graph capture, must all happen on ctx->device).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
    if (prev == dev) prev = -1;  // nothing to restore
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int cuda_fail(tt_ctx* ctx, cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation)
    return fail(ctx, TT_ENOMEM, "%s: %s", where, cudaGetErrorString(e));
  return fail(ctx, TT_EDEVICE, "%s: %s", where, cudaGetErrorString(e));
}

#define TT_CUDA(ctx, x, where)                              \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, where); \
  } while (0)

// kernels.cpp:27-34 require_tile, same message.
bool tile_ok(int f, int extent) { return f >= 1 && f <= extent && extent % f == 0; }

int require_tile(tt_ctx* ctx, int f, int extent, const char* who) {
  if (!tile_ok(f, extent))
    return fail(ctx, TT_EINVAL, "%s: tile factor %d does not divide extent %d", who, f, extent);
  return TT_OK;
}

cudaError_t ensure(DevMat& m, int rows, int cols) {
  const long long ld = padded_ld(cols);
  const size_t need = static_cast<size_t>(std::max(rows, 1)) * ld * sizeof(double);
  if (m.p && m.capacity >= need) {
    m.rows = rows;
    m.cols = cols;
    m.ld = ld;
    return cudaSuccess;
  }
  if (m.p) cudaFree(m.p);
  m.p = nullptr;
  m.capacity = 0;
  cudaError_t e = cudaMalloc(&m.p, need);
  if (e != cudaSuccess) return e;
  m.capacity = need;
  m.rows = rows;
  m.cols = cols;
  m.ld = ld;
  return cudaSuccess;
}

void release(DevMat& m) {
  if (m.p) cudaFree(m.p);
  m = DevMat{};
}

cudaError_t upload(const DevMat& m, const double* host, cudaStream_t s) {
  return cudaMemcpy2DAsync(m.p, m.ld * sizeof(double), host, m.cols * sizeof(double),
                           m.cols * sizeof(double), m.rows, cudaMemcpyHostToDevice, s);
}

cudaError_t download(double* host, const DevMat& m, cudaStream_t s) {
  return cudaMemcpy2DAsync(host, m.cols * sizeof(double), m.p, m.ld * sizeof(double),
                           m.cols * sizeof(double), m.rows, cudaMemcpyDeviceToHost, s);
}

cudaError_t copy_d2d(const DevMat& dst, const DevMat& src, cudaStream_t s) {
  return cudaMemcpyAsync(dst.p, src.p, src.bytes(), cudaMemcpyDeviceToDevice, s);
}

const char* lu_name = "lu_tiled";
const char* chol_name = "cholesky_tiled";

// Validation in the reference order: require_square, require_tile(by),
// require_tile(bx) (kernels.cpp:179-182, 265-268).
int validate_factor(tt_ctx* ctx, int kernel, int rows, int cols, int by, int bx) {
  const char* who = kernel == TT_KERNEL_LU ? lu_name : chol_name;
  if (rows != cols || rows < 1) return fail(ctx, TT_EINVAL, "%s: square matrix required", who);
  int rc = require_tile(ctx, by, rows, who);
  if (rc) return rc;
  return require_tile(ctx, bx, rows, who);
}

// mm3: arity first (kernels.cpp:124-126), then each product's (fy, fx) in
// schedule order (:95-96 via :128-130).
int validate_mm3(tt_ctx* ctx, int n, int l, int m, int o, int p, const int* cfg, int ncfg) {
  (void)l;
  (void)o;
  if (ncfg != 6) return fail(ctx, TT_EINVAL, "mm3_tiled: six tile factors required");
  const int ext[6] = {n, m, m, p, n, p};
  for (int i = 0; i < 6; ++i) {
    int rc = require_tile(ctx, cfg[i], ext[i], "matmul_tiled");
    if (rc) return rc;
  }
  return TT_OK;
}

int ensure_info_slots(tt_ctx* ctx, int slots) {
  if (ctx->info_host_slots >= slots) return TT_OK;
  // grow geometrically (>= 256 slots): cudaFreeHost synchronises the device
  // and page-locking is slow, so a batch call must not hit this every time
  slots = std::max({slots, 256, 2 * ctx->info_host_slots});
  if (ctx->info_host) cudaFreeHost(ctx->info_host);
  ctx->info_host = nullptr;
  TT_CUDA(ctx, cudaMallocHost(&ctx->info_host, sizeof(int) * slots), "cudaMallocHost");
  ctx->info_host_slots = slots;
  return TT_OK;
}

// Captures (or fetches) the graph for one schedule on one buffer.
// TT_EAGER=1 (debug aid): no capture; the schedule is enqueued directly
// on the context stream every run and *out stays null.
bool eager_mode() {
  static const bool eager = [] {
    const char* v = std::getenv("TT_EAGER");
    return v && v[0] == '1';
  }();
  return eager;
}

template <class Enqueue>
int get_graph(tt_ctx* ctx, const GraphKey& key, Enqueue&& enq, cudaGraphExec_t* out,
              long long* nodes) {
  if (eager_mode()) {
    tt::ScheduleStats st;
    TT_CUDA(ctx, cudaMemsetAsync(ctx->info, 0x7F, sizeof(int), ctx->stream), "memset");
    TT_CUDA(ctx, enq(&st), "eager schedule");
    *out = nullptr;
    *nodes = st.launches;
    return TT_OK;
  }
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end()) {
    *out = it->second;
    *nodes = ctx->graph_nodes[key];
    return TT_OK;
  }
  cudaGraph_t graph = nullptr;
  TT_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal),
          "cudaStreamBeginCapture");
  tt::ScheduleStats st;
  // status word reset is the first node: 0x7F7F7F7F = "no failure"
  cudaError_t e = cudaMemsetAsync(ctx->info, 0x7F, sizeof(int), ctx->stream);
  if (e == cudaSuccess) e = enq(&st);
  cudaError_t e2 = cudaStreamEndCapture(ctx->stream, &graph);
  if (e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    return cuda_fail(ctx, e, "schedule capture");
  }
  TT_CUDA(ctx, e2, "cudaStreamEndCapture");
  if (const char* dot = std::getenv("TT_GRAPH_DOT"))  // debug aid: the captured graph
    cudaGraphDebugDotPrint(graph, dot, cudaGraphDebugDotFlagsVerbose);
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  TT_CUDA(ctx, e, "cudaGraphInstantiate");
  ctx->graphs[key] = exec;
  ctx->graph_nodes[key] = st.launches;
  *out = exec;
  *nodes = st.launches;
  return TT_OK;
}

// Factorisation schedule: TT_FACTOR_SCHEDULE=graph forces the launch-per-kernel
// graph (schedules.cu); otherwise the persistent tile-DAG kernel
// (dag_factor.cu) runs whenever it covers (n, by, bx).
bool use_dag_schedule(int n, int by, int bx) {
  const char* v = std::getenv("TT_FACTOR_SCHEDULE");  // per call: tests switch it
  const bool graph_only = v && std::strcmp(v, "graph") == 0;
  return !graph_only && tt::dag::eligible(n, by, bx);
}

int factor_graph(tt_ctx* ctx, int kernel, double* a, int n, long long ld, int by, int bx,
                 cudaGraphExec_t* g, long long* nodes) {
  const bool chol = kernel != TT_KERNEL_LU;
  const bool dag = use_dag_schedule(n, by, bx);
  GraphKey key{chol ? kGraphChol : kGraphLu,
               {reinterpret_cast<long long>(a), n, ld, by, bx, dag ? 1 : 0}};
  tt::dag::Workspace* w = nullptr;
  if (dag) {  // allocated outside stream capture
    w = &ctx->dag_ws[key];
    if (!w->tasks) TT_CUDA(ctx, tt::dag::create(w, chol, n, by, bx), "dag workspace");
    ctx->dag_last = w;
  }
  return get_graph(
      ctx, key,
      [&](tt::ScheduleStats* st) {
        if (dag) {
          ctx->dag_last = w;
          st->launches += 1;
          return tt::dag::enqueue(*w, chol, a, n, ld, ctx->info, ctx->stream);
        }
        const tt::Streams ss{ctx->stream, ctx->stream2, ctx->fork, ctx->join};
        return !chol ? tt::enqueue_lu(ctx->tmaps, a, n, ld, by, bx, ctx->ws, ctx->info, ss, st)
                     : tt::enqueue_cholesky(ctx->tmaps, a, n, ld, by, bx, ctx->ws, ctx->info, ss,
                                            st);
      },
      g, nodes);
}

int mm3_graph(tt_ctx* ctx, const tt::Mm3Bufs& b, const int* d, const int* cfg,
              cudaGraphExec_t* g, long long* nodes) {
  auto ptr = [](const void* q) { return reinterpret_cast<long long>(q); };
  GraphKey key{kGraphMm3,
               {ptr(b.a), ptr(b.b), ptr(b.c), ptr(b.d), ptr(b.e), ptr(b.f), ptr(b.g), b.lda, b.ldb,
                b.ldc, b.ldd, b.lde, b.ldf, b.ldg, d[0], d[1], d[2], d[3], d[4], cfg[0], cfg[1],
                cfg[2], cfg[3], cfg[4], cfg[5]}};
  return get_graph(
      ctx, key,
      [&](tt::ScheduleStats* st) {
        const tt::Streams ss{ctx->stream, ctx->stream2, ctx->fork, ctx->join};
        return tt::enqueue_mm3(ctx->tmaps, b, d[0], d[1], d[2], d[3], d[4], cfg, ss, st);
      },
      g, nodes);
}

tt::Mm3Bufs setup_mm3_bufs(tt_ctx* ctx) {
  tt::Mm3Bufs b;
  b.a = ctx->pristine[0].p;
  b.lda = ctx->pristine[0].ld;
  b.b = ctx->pristine[1].p;
  b.ldb = ctx->pristine[1].ld;
  b.c = ctx->pristine[2].p;
  b.ldc = ctx->pristine[2].ld;
  b.d = ctx->pristine[3].p;
  b.ldd = ctx->pristine[3].ld;
  b.e = ctx->e.p;
  b.lde = ctx->e.ld;
  b.f = ctx->f.p;
  b.ldf = ctx->f.ld;
  b.g = ctx->g.p;
  b.ldg = ctx->g.ld;
  return b;
}

int check_cfg(tt_ctx* ctx, const int* cfg, int ncfg) {
  if (ctx->kernel < 0) return fail(ctx, TT_EINVAL, "no case set up (call tt_setup_* first)");
  if (ctx->kernel == TT_KERNEL_MM3)
    return validate_mm3(ctx, ctx->dims[0], ctx->dims[1], ctx->dims[2], ctx->dims[3],
                        ctx->dims[4], cfg, ncfg);
  if (ncfg < 2) return fail(ctx, TT_EINVAL, "configuration needs two factors (by, bx)");
  return validate_factor(ctx, ctx->kernel, ctx->dims[0], ctx->dims[0], cfg[0], cfg[1]);
}

// Enqueue one run of the configured case on ctx->stream: (restore +) graph.
// `restore` happens before `ev_start` is recorded when ev_start != nullptr.
int enqueue_run(tt_ctx* ctx, const int* cfg, cudaEvent_t ev_start, cudaEvent_t ev_end,
                int* info_slot) {
  cudaGraphExec_t g = nullptr;
  long long nodes = 0;
  int rc;
  // build (or fetch) the instantiation first: workspace allocation, capture
  // and cudaGraphInstantiate stay outside the event pair even with 0 warm-ups
  // (TT_EAGER=1 has no graph: the schedule is enqueued inside the pair)
  auto build = [&] {
    return ctx->kernel == TT_KERNEL_MM3
               ? mm3_graph(ctx, setup_mm3_bufs(ctx), ctx->dims, cfg, &g, &nodes)
               : factor_graph(ctx, ctx->kernel, ctx->work.p, ctx->dims[0], ctx->work.ld, cfg[0],
                              cfg[1], &g, &nodes);
  };
  if (!eager_mode() && (rc = build()) != TT_OK) return rc;
  if (ctx->kernel != TT_KERNEL_MM3)  // fresh copy of the pristine input, untimed
    TT_CUDA(ctx, copy_d2d(ctx->work, ctx->pristine[0], ctx->stream), "restore copy");
  if (ev_start) TT_CUDA(ctx, cudaEventRecord(ev_start, ctx->stream), "cudaEventRecord");
  if (eager_mode() && (rc = build()) != TT_OK) return rc;
  if (g) TT_CUDA(ctx, cudaGraphLaunch(g, ctx->stream), "cudaGraphLaunch");
  if (ev_end) TT_CUDA(ctx, cudaEventRecord(ev_end, ctx->stream), "cudaEventRecord");
  ctx->launches += static_cast<unsigned long long>(nodes);
  if (info_slot)
    TT_CUDA(ctx,
            cudaMemcpyAsync(info_slot, ctx->info, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream),
            "status readback");
  return TT_OK;
}

int numeric_status(tt_ctx* ctx, int info, int* fail_index) {
  if (info == tt::kNoFailure) return TT_OK;
  if (info == tt::dag::kTimeout) {
    const std::string why = ctx->dag_last ? tt::dag::watchdog_info(*ctx->dag_last) : std::string();
    return fail(ctx, TT_EDEVICE, "persistent schedule watchdog: dependency wait timed out%s%s",
                why.empty() ? "" : ": ", why.c_str());
  }
  if (fail_index) *fail_index = info;
  if (ctx->kernel == TT_KERNEL_CHOLESKY)
    return fail(ctx, TT_ENUMERIC, "cholesky: non-positive diagonal at row %d", info);
  return fail(ctx, TT_ENUMERIC, "lu: vanishing pivot at column %d", info);
}

// One-shot factorisation through host memory (drop-in for the reference).
int oneshot_factor(tt_ctx* ctx, int kernel, double* a, int rows, int cols, int by, int bx,
                   int* fail_index) {
  int rc = validate_factor(ctx, kernel, rows, cols, by, bx);
  if (rc) return rc;
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  TT_CUDA(ctx, ensure(ctx->oneshot, rows, cols), "cudaMalloc");
  TT_CUDA(ctx, upload(ctx->oneshot, a, ctx->stream), "H2D");
  cudaGraphExec_t g = nullptr;
  long long nodes = 0;
  rc = factor_graph(ctx, kernel, ctx->oneshot.p, rows, ctx->oneshot.ld, by, bx, &g, &nodes);
  if (rc) return rc;
  if (g) TT_CUDA(ctx, cudaGraphLaunch(g, ctx->stream), "cudaGraphLaunch");
  ctx->launches += static_cast<unsigned long long>(nodes);
  rc = ensure_info_slots(ctx, 1);
  if (rc) return rc;
  TT_CUDA(ctx,
          cudaMemcpyAsync(ctx->info_host, ctx->info, sizeof(int), cudaMemcpyDeviceToHost,
                          ctx->stream),
          "status readback");
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "factorisation");
  const int saved_kernel = ctx->kernel;
  ctx->kernel = kernel;
  rc = numeric_status(ctx, ctx->info_host[0], fail_index);
  ctx->kernel = saved_kernel;
  if (rc) return rc;
  TT_CUDA(ctx, download(a, ctx->oneshot, ctx->stream), "D2H");
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "D2H");
  return TT_OK;
}

// Pipelined batch of one-shot factorisations through host memory: matrix i
// is uploaded (copy stream), factored (context stream) and downloaded (a
// second copy stream) while its neighbours are in flight, triple-buffered
// on the device — the host<->device traffic overlaps the factorisations.
// Host buffers should be page-locked for the copies to be asynchronous.
int batch_factor(tt_ctx* ctx, int kernel, double* const* mats, int count, int n, int by, int bx,
                 int* fail_index) {
  int rc = validate_factor(ctx, kernel, n, n, by, bx);
  if (rc) return rc;
  if (count < 0 || (count > 0 && !mats)) return fail(ctx, TT_EINVAL, "batch: bad matrix list");
  if (eager_mode()) {  // debug aid: no graphs to pipeline, run the one-shot path per matrix
    for (int i = 0; i < count; ++i) {
      int idx = -1;
      rc = oneshot_factor(ctx, kernel, mats[i], n, n, by, bx, &idx);
      if (fail_index) fail_index[i] = idx;
      if (rc) return rc;
    }
    return TT_OK;
  }
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  if (!ctx->cin) TT_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cin, cudaStreamNonBlocking), "stream");
  if (!ctx->cout) TT_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cout, cudaStreamNonBlocking), "stream");
  // Three device buffers: a buffer is re-uploaded only after its previous
  // matrix was downloaded, so with two the upload and download of one buffer
  // would sit between its factorisations (measured 1.07 ms per matrix at
  // N=2000 against 0.88 ms for the kernel); with three the copies of the
  // other buffers run while one factorises.
  constexpr int kBufs = 3;
  cudaGraphExec_t g[kBufs] = {};
  long long nodes[kBufs] = {};
  for (int b = 0; b < kBufs && b < count; ++b) {
    TT_CUDA(ctx, ensure(ctx->batch[b], n, n), "cudaMalloc");
    rc = factor_graph(ctx, kernel, ctx->batch[b].p, n, ctx->batch[b].ld, by, bx, &g[b], &nodes[b]);
    if (rc) return rc;
  }
  rc = ensure_info_slots(ctx, std::max(count, 1));
  if (rc) return rc;
  std::vector<cudaEvent_t> ev(3 * kBufs, nullptr);  // per buffer: uploaded, factored, downloaded
  for (auto& e : ev) TT_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  auto cleanup = [&] {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  };
  cudaError_t err = cudaSuccess;
  for (int i = 0; i < count && err == cudaSuccess; ++i) {
    const int b = i % kBufs;
    cudaEvent_t up = ev[3 * b], fac = ev[3 * b + 1], down = ev[3 * b + 2];
    if (i >= kBufs) err = cudaStreamWaitEvent(ctx->cin, down, 0);  // buffer b free again
    if (err == cudaSuccess) err = upload(ctx->batch[b], mats[i], ctx->cin);
    if (err == cudaSuccess) err = cudaEventRecord(up, ctx->cin);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(ctx->stream, up, 0);
    if (err == cudaSuccess && g[b]) err = cudaGraphLaunch(g[b], ctx->stream);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(&ctx->info_host[i], ctx->info, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->stream);
    if (err == cudaSuccess) err = cudaEventRecord(fac, ctx->stream);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(ctx->cout, fac, 0);
    if (err == cudaSuccess) err = download(mats[i], ctx->batch[b], ctx->cout);
    if (err == cudaSuccess) err = cudaEventRecord(down, ctx->cout);
    ctx->launches += static_cast<unsigned long long>(nodes[b]);
  }
  if (err == cudaSuccess) err = cudaStreamSynchronize(ctx->cout);
  if (err == cudaSuccess) err = cudaStreamSynchronize(ctx->stream);
  cleanup();
  if (err != cudaSuccess) return cuda_fail(ctx, err, "batch factorisation");
  const int saved = ctx->kernel;
  ctx->kernel = kernel;
  for (int i = 0; i < count; ++i) {
    if (fail_index) fail_index[i] = -1;
    if (ctx->info_host[i] != tt::kNoFailure) {
      int idx = -1;
      rc = numeric_status(ctx, ctx->info_host[i], &idx);
      if (fail_index) fail_index[i] = idx;
      if (rc) {
        ctx->kernel = saved;
        return rc;  // the first failing matrix decides the status (its index in *fail_index)
      }
    }
  }
  ctx->kernel = saved;
  return TT_OK;
}

double ordered_to_double(unsigned long long u) {
  double d;
  std::memcpy(&d, &u, sizeof d);
  return d;
}

}  // namespace

extern "C" {

const char* tt_build_info(void) {
  return "libtt_gpu sm_100a: fp64 DMMA m8n8k4 GEMM family (TMA 128B-swizzle, mbarrier "
         "pipeline), LU/Cholesky panel kernels, CUDA-graph instantiation cache";
}

int tt_ctx_create(int device, tt_ctx** out) {
  if (!out) return TT_EINVAL;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return TT_EDEVICE;  // no CPU fallback: the product path needs the GPU
  if (device < 0 || device >= count) return TT_EINVAL;
  tt_ctx* ctx = new tt_ctx();
  ctx->device = device;
  auto cleanup = [&](int code) {
    tt_ctx_destroy(ctx);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return cleanup(TT_EDEVICE);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming) != cudaSuccess)
    return cleanup(TT_EDEVICE);
  if (cudaMalloc(&ctx->info, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&ctx->ws, sizeof(double) * tt::kIB * tt::kIB) != cudaSuccess ||
      cudaMalloc(&ctx->red, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return cleanup(TT_ENOMEM);
  // (legacy default stream: wait, so it cannot land after work on ctx->stream)
  if (cudaMemset(ctx->info, 0x7F, sizeof(int)) != cudaSuccess ||
      cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess)
    return cleanup(TT_EDEVICE);
  // Set the dynamic-smem attribute of every GEMM variant up front (so graph
  // capture never meets a first-use attribute call).
  for (int bt = 0; bt < 2; ++bt)
    for (int bm : {8, 16, 32, 64, 128})
      for (int bn : {8, 16, 32, 64, 128}) {
        tt::GemmArgs dummy{};
        CUtensorMap m{};
        cudaError_t r = bt ? tt::launch_nt(bm, bn, m, m, m, dummy, 0, ctx->stream)
                           : tt::launch_nn(bm, bn, m, m, m, dummy, 0, ctx->stream);
        if (r != cudaSuccess) return cleanup(TT_EDEVICE);
      }
  // and every persistent-schedule variant (the attribute is per device)
  if (tt::dag::configure_device() != cudaSuccess) return cleanup(TT_EDEVICE);
  *out = ctx;
  return TT_OK;
}

int tt_ctx_destroy(tt_ctx* ctx) {
  if (!ctx) return TT_OK;
  cudaSetDevice(ctx->device);
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : ctx->dag_ws) tt::dag::destroy(&kv.second);
  for (auto* m : {&ctx->work, &ctx->e, &ctx->f, &ctx->g, &ctx->scratch_l, &ctx->scratch_u,
                  &ctx->oneshot, &ctx->batch[0], &ctx->batch[1], &ctx->batch[2]})
    release(*m);
  if (ctx->cin) cudaStreamDestroy(ctx->cin);
  if (ctx->cout) cudaStreamDestroy(ctx->cout);
  for (auto& m : ctx->pristine) release(m);
  for (auto& m : ctx->oneshot_in) release(m);
  if (ctx->info) cudaFree(ctx->info);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->red) cudaFree(ctx->red);
  if (ctx->info_host) cudaFreeHost(ctx->info_host);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->join) cudaEventDestroy(ctx->join);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  delete ctx;
  return TT_OK;
}

const char* tt_last_error(const tt_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int tt_ctx_device(const tt_ctx* ctx) { return ctx ? ctx->device : -1; }
int tt_cache_size(const tt_ctx* ctx) { return ctx ? static_cast<int>(ctx->graphs.size()) : 0; }
uint64_t tt_launch_count(const tt_ctx* ctx) { return ctx ? ctx->launches : 0; }

int tt_lu_factor_inplace(tt_ctx* ctx, double* a, int rows, int cols, int by, int bx,
                         int* fail_index) {
  if (!ctx || !a) return TT_EINVAL;
  return oneshot_factor(ctx, TT_KERNEL_LU, a, rows, cols, by, bx, fail_index);
}

int tt_cholesky_factor_inplace(tt_ctx* ctx, double* a, int rows, int cols, int by, int bx,
                               int* fail_index) {
  if (!ctx || !a) return TT_EINVAL;
  return oneshot_factor(ctx, TT_KERNEL_CHOLESKY, a, rows, cols, by, bx, fail_index);
}

int tt_lu_factor_batch(tt_ctx* ctx, double* const* mats, int count, int n, int by, int bx,
                       int* fail_index) {
  if (!ctx) return TT_EINVAL;
  return batch_factor(ctx, TT_KERNEL_LU, mats, count, n, by, bx, fail_index);
}

int tt_cholesky_factor_batch(tt_ctx* ctx, double* const* mats, int count, int n, int by, int bx,
                             int* fail_index) {
  if (!ctx) return TT_EINVAL;
  return batch_factor(ctx, TT_KERNEL_CHOLESKY, mats, count, n, by, bx, fail_index);
}

int tt_mm3_tiled(tt_ctx* ctx, const double* a, const double* b, const double* c,
                 const double* d, int n, int l, int m, int o, int p, const int* cfg, int ncfg,
                 double* g) {
  if (!ctx || !a || !b || !c || !d || !g) return TT_EINVAL;
  if (n < 1 || l < 1 || m < 1 || o < 1 || p < 1)
    return fail(ctx, TT_EINVAL, "matmul: inner dimensions disagree");
  int rc = validate_mm3(ctx, n, l, m, o, p, cfg, ncfg);
  if (rc) return rc;
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  const int shp[4][2] = {{n, l}, {l, m}, {m, o}, {o, p}};
  const double* src[4] = {a, b, c, d};
  for (int i = 0; i < 4; ++i) {
    TT_CUDA(ctx, ensure(ctx->oneshot_in[i], shp[i][0], shp[i][1]), "cudaMalloc");
    TT_CUDA(ctx, upload(ctx->oneshot_in[i], src[i], ctx->stream), "H2D");
  }
  TT_CUDA(ctx, ensure(ctx->scratch_l, n, m), "cudaMalloc");
  TT_CUDA(ctx, ensure(ctx->scratch_u, m, p), "cudaMalloc");
  TT_CUDA(ctx, ensure(ctx->oneshot, n, p), "cudaMalloc");
  tt::Mm3Bufs bufs;
  bufs.a = ctx->oneshot_in[0].p;
  bufs.lda = ctx->oneshot_in[0].ld;
  bufs.b = ctx->oneshot_in[1].p;
  bufs.ldb = ctx->oneshot_in[1].ld;
  bufs.c = ctx->oneshot_in[2].p;
  bufs.ldc = ctx->oneshot_in[2].ld;
  bufs.d = ctx->oneshot_in[3].p;
  bufs.ldd = ctx->oneshot_in[3].ld;
  bufs.e = ctx->scratch_l.p;
  bufs.lde = ctx->scratch_l.ld;
  bufs.f = ctx->scratch_u.p;
  bufs.ldf = ctx->scratch_u.ld;
  bufs.g = ctx->oneshot.p;
  bufs.ldg = ctx->oneshot.ld;
  const int dims[5] = {n, l, m, o, p};
  cudaGraphExec_t gx = nullptr;
  long long nodes = 0;
  rc = mm3_graph(ctx, bufs, dims, cfg, &gx, &nodes);
  if (rc) return rc;
  if (gx) TT_CUDA(ctx, cudaGraphLaunch(gx, ctx->stream), "cudaGraphLaunch");
  ctx->launches += static_cast<unsigned long long>(nodes);
  TT_CUDA(ctx, download(g, ctx->oneshot, ctx->stream), "D2H");
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "3mm");
  return TT_OK;
}

static int setup_common(tt_ctx* ctx, int kernel, int n, int l, int m, int o, int p) {
  if (kernel < TT_KERNEL_LU || kernel > TT_KERNEL_MM3)
    return fail(ctx, TT_EINVAL, "unknown kernel id %d", kernel);
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->kernel = -1;
  ctx->have_output = false;
  if (kernel == TT_KERNEL_MM3) {
    if (n < 1 || l < 1 || m < 1 || o < 1 || p < 1)
      return fail(ctx, TT_EINVAL, "gen_3mm_inputs: all five extents must be >= 1");
    const int shp[4][2] = {{n, l}, {l, m}, {m, o}, {o, p}};
    for (int i = 0; i < 4; ++i)
      TT_CUDA(ctx, ensure(ctx->pristine[i], shp[i][0], shp[i][1]), "cudaMalloc");
    TT_CUDA(ctx, ensure(ctx->e, n, m), "cudaMalloc");
    TT_CUDA(ctx, ensure(ctx->f, m, p), "cudaMalloc");
    TT_CUDA(ctx, ensure(ctx->g, n, p), "cudaMalloc");
  } else {
    if (n < 1) return fail(ctx, TT_EINVAL, "gen_spd: n must be >= 1");
    TT_CUDA(ctx, ensure(ctx->pristine[0], n, n), "cudaMalloc");
    TT_CUDA(ctx, ensure(ctx->work, n, n), "cudaMalloc");
  }
  ctx->dims[0] = n;
  ctx->dims[1] = l;
  ctx->dims[2] = m;
  ctx->dims[3] = o;
  ctx->dims[4] = p;
  return TT_OK;
}

int tt_setup_host(tt_ctx* ctx, int kernel, int n, int l, int m, int o, int p, const double* a,
                  const double* b, const double* c, const double* d) {
  if (!ctx || !a) return TT_EINVAL;
  int rc = setup_common(ctx, kernel, n, l, m, o, p);
  if (rc) return rc;
  if (kernel == TT_KERNEL_MM3) {
    if (!b || !c || !d) return fail(ctx, TT_EINVAL, "3mm setup needs A, B, C, D");
    const double* src[4] = {a, b, c, d};
    for (int i = 0; i < 4; ++i) TT_CUDA(ctx, upload(ctx->pristine[i], src[i], ctx->stream), "H2D");
  } else {
    TT_CUDA(ctx, upload(ctx->pristine[0], a, ctx->stream), "H2D");
  }
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "setup");
  ctx->kernel = kernel;
  return TT_OK;
}

int tt_setup_seeded(tt_ctx* ctx, int kernel, int n, int l, int m, int o, int p, uint64_t seed) {
  if (!ctx) return TT_EINVAL;
  int rc = setup_common(ctx, kernel, n, l, m, o, p);
  if (rc) return rc;
  // tiletuner::Rng (rng.hpp:11-32) is std::mt19937_64 with next_double =
  // (u64 >> 11) * 2^-53; the standard fixes its output bit-exactly.
  std::mt19937_64 gen(seed);
  auto next_double = [&] { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
  if (kernel == TT_KERNEL_MM3) {
    const int shp[4][2] = {{n, l}, {l, m}, {m, o}, {o, p}};
    for (int i = 0; i < 4; ++i) {  // one stream fills A, B, C, D in order (kernels.cpp:64-67)
      std::vector<double> h(static_cast<size_t>(shp[i][0]) * shp[i][1]);
      for (double& v : h) v = next_double();
      TT_CUDA(ctx, upload(ctx->pristine[i], h.data(), ctx->stream), "H2D");
      TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "setup");
    }
  } else {
    std::vector<double> h(static_cast<size_t>(n) * n);
    for (double& v : h) v = next_double();
    TT_CUDA(ctx, ensure(ctx->scratch_l, n, n), "cudaMalloc");
    TT_CUDA(ctx, upload(ctx->scratch_l, h.data(), ctx->stream), "H2D");
    tt::launch_spd_product(ctx->scratch_l.p, ctx->scratch_l.ld, n, ctx->pristine[0].p,
                           ctx->pristine[0].ld, ctx->stream);
    ctx->launches += 1;
    TT_CUDA(ctx, cudaGetLastError(), "gen_spd kernel");
    TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "setup");
  }
  ctx->kernel = kernel;
  return TT_OK;
}

int tt_get_input(tt_ctx* ctx, double* a, double* b, double* c, double* d) {
  if (!ctx) return TT_EINVAL;
  if (ctx->kernel < 0) return fail(ctx, TT_EINVAL, "no case set up");
  double* dst[4] = {a, b, c, d};
  const int count = ctx->kernel == TT_KERNEL_MM3 ? 4 : 1;
  for (int i = 0; i < count; ++i)
    if (dst[i]) TT_CUDA(ctx, download(dst[i], ctx->pristine[i], ctx->stream), "D2H");
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "D2H");
  return TT_OK;
}

int tt_run(tt_ctx* ctx, const int* cfg, int ncfg, double* out, int* fail_index) {
  if (!ctx || !cfg) return TT_EINVAL;
  int rc = check_cfg(ctx, cfg, ncfg);
  if (rc) return rc;
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  rc = ensure_info_slots(ctx, 1);
  if (rc) return rc;
  rc = enqueue_run(ctx, cfg, nullptr, nullptr, &ctx->info_host[0]);
  if (rc) return rc;
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "run");
  if (ctx->kernel != TT_KERNEL_MM3) {
    rc = numeric_status(ctx, ctx->info_host[0], fail_index);
    if (rc) return rc;
  }
  ctx->have_output = true;
  if (out) {
    TT_CUDA(ctx, download(out, ctx->kernel == TT_KERNEL_MM3 ? ctx->g : ctx->work, ctx->stream),
            "D2H");
    TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "D2H");
  }
  return TT_OK;
}

int tt_measure_samples(tt_ctx* ctx, const int* cfg, int ncfg, int warmups, int reps,
                       double* samples) {
  if (!ctx || !cfg || !samples) return TT_EINVAL;
  // harness.cpp:81-86 check_protocol
  if (warmups < 0 || reps < 1)
    return fail(ctx, TT_EINVAL, "measure: warmups must be >= 0 and repetitions >= 1");
  int rc = check_cfg(ctx, cfg, ncfg);
  if (rc) return rc;
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  rc = ensure_info_slots(ctx, warmups + reps);
  if (rc) return rc;
  std::vector<cudaEvent_t> evs(2 * static_cast<size_t>(reps));
  for (auto& e : evs) TT_CUDA(ctx, cudaEventCreate(&e), "cudaEventCreate");
  auto destroy = [&] {
    for (auto& e : evs) cudaEventDestroy(e);
  };
  for (int w = 0; w < warmups && rc == TT_OK; ++w)
    rc = enqueue_run(ctx, cfg, nullptr, nullptr, &ctx->info_host[w]);
  for (int r = 0; r < reps && rc == TT_OK; ++r)
    rc = enqueue_run(ctx, cfg, evs[2 * r], evs[2 * r + 1], &ctx->info_host[warmups + r]);
  if (rc) {
    destroy();
    return rc;
  }
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    destroy();
    return cuda_fail(ctx, e, "measure");
  }
  if (ctx->kernel != TT_KERNEL_MM3) {
    for (int i = 0; i < warmups + reps; ++i) {
      rc = numeric_status(ctx, ctx->info_host[i], nullptr);
      if (rc) {
        destroy();
        return rc;
      }
    }
  }
  for (int r = 0; r < reps; ++r) {
    float ms = 0.f;
    e = cudaEventElapsedTime(&ms, evs[2 * r], evs[2 * r + 1]);
    if (e != cudaSuccess) {
      destroy();
      return cuda_fail(ctx, e, "cudaEventElapsedTime");
    }
    samples[r] = static_cast<double>(ms) * 1e-3;
    if (!(samples[r] > 0.0)) {  // harness.cpp:133-135
      destroy();
      return fail(ctx, TT_EDEVICE, "measure: nonpositive timer reading");
    }
  }
  destroy();
  ctx->have_output = true;
  return TT_OK;
}

int tt_measure(tt_ctx* ctx, const int* cfg, int ncfg, int warmups, int reps, int aggregate,
               double* seconds) {
  if (!ctx || !seconds) return TT_EINVAL;
  if (aggregate < TT_AGG_MEDIAN || aggregate > TT_AGG_MEAN)
    return fail(ctx, TT_EINVAL, "unknown aggregate enum value");
  std::vector<double> s(std::max(reps, 1));
  int rc = tt_measure_samples(ctx, cfg, ncfg, warmups, reps, s.data());
  if (rc) return rc;
  // harness.cpp:53-71 aggregate_samples
  if (aggregate == TT_AGG_MIN) {
    *seconds = *std::min_element(s.begin(), s.end());
  } else if (aggregate == TT_AGG_MEAN) {
    double acc = 0.0;
    for (double v : s) acc += v;
    *seconds = acc / static_cast<double>(s.size());
  } else {
    std::sort(s.begin(), s.end());
    const size_t n = s.size();
    *seconds = n % 2 == 1 ? s[n / 2] : 0.5 * (s[n / 2 - 1] + s[n / 2]);
  }
  return TT_OK;
}

int tt_residual(tt_ctx* ctx, const double* ref_g, double* out) {
  if (!ctx || !out) return TT_EINVAL;
  if (ctx->kernel < 0 || !ctx->have_output) return fail(ctx, TT_EINVAL, "no output to check");
  TT_CUDA(ctx, cudaSetDevice(ctx->device), "cudaSetDevice");
  TT_CUDA(ctx, cudaMemsetAsync(ctx->red, 0, 2 * sizeof(unsigned long long), ctx->stream),
          "memset");
  if (ctx->kernel == TT_KERNEL_MM3) {
    if (!ref_g) return fail(ctx, TT_EINVAL, "3mm residual needs the reference output");
    const int n = ctx->dims[0], p = ctx->dims[4];
    TT_CUDA(ctx, ensure(ctx->scratch_l, n, p), "cudaMalloc");
    TT_CUDA(ctx, upload(ctx->scratch_l, ref_g, ctx->stream), "H2D");
    tt::launch_maxdiff(ctx->g.p, ctx->g.ld, ctx->scratch_l.p, ctx->scratch_l.ld, n, p, ctx->red,
                       ctx->stream);
  } else {
    const int n = ctx->dims[0];
    TT_CUDA(ctx, ensure(ctx->scratch_l, n, n), "cudaMalloc");
    TT_CUDA(ctx, ensure(ctx->scratch_u, n, n), "cudaMalloc");
    TT_CUDA(ctx, ensure(ctx->oneshot, n, n), "cudaMalloc");
    const tt::Operand L{ctx->scratch_l.p, n, n, ctx->scratch_l.ld, 0, 0};
    if (ctx->kernel == TT_KERNEL_LU) {
      tt::launch_unpack_lu(ctx->work.p, ctx->work.ld, n, ctx->scratch_l.p, ctx->scratch_u.p,
                           ctx->scratch_l.ld, ctx->stream);
      const tt::Operand U{ctx->scratch_u.p, n, n, ctx->scratch_u.ld, 0, 0};
      TT_CUDA(ctx,
              tt::gemm(ctx->tmaps, L, U, false, ctx->oneshot.p, ctx->oneshot.ld, n, n, n, 128,
                       128, 0, 0, 0, 0, ctx->stream),
              "residual gemm");
    } else {
      tt::launch_lower_of(ctx->work.p, ctx->work.ld, n, ctx->scratch_l.p, ctx->scratch_l.ld,
                          ctx->stream);
      TT_CUDA(ctx,
              tt::gemm(ctx->tmaps, L, L, true, ctx->oneshot.p, ctx->oneshot.ld, n, n, n, 128,
                       128, 0, 0, 0, 0, ctx->stream),
              "residual gemm");
    }
    tt::launch_maxdiff(ctx->oneshot.p, ctx->oneshot.ld, ctx->pristine[0].p, ctx->pristine[0].ld,
                       n, n, ctx->red, ctx->stream);
  }
  TT_CUDA(ctx, cudaGetLastError(), "residual kernels");
  unsigned long long h[2] = {0, 0};
  TT_CUDA(ctx, cudaMemcpyAsync(h, ctx->red, sizeof h, cudaMemcpyDeviceToHost, ctx->stream),
          "D2H");
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "residual");
  const double num = ordered_to_double(h[0]), den = ordered_to_double(h[1]);
  *out = den > 0.0 ? num / den : num;  // kernels.cpp:336-337
  return TT_OK;
}

int tt_dev_lu(tt_ctx* ctx, double* a, int n, int ld, int by, int bx, int* fail_index,
              void* stream) {
  if (!ctx || !a) return TT_EINVAL;
  int rc = validate_factor(ctx, TT_KERNEL_LU, n, n, by, bx);
  if (rc) return rc;
  if (ld < n || (ld & 1)) return fail(ctx, TT_EINVAL, "leading dimension must be even and >= n");
  if (!aligned16(a)) return fail(ctx, TT_EINVAL, "matrix base must be 16-byte aligned");
  DeviceGuard dg(ctx->device);
  TT_CUDA(ctx, dg.err, "cudaSetDevice");
  cudaGraphExec_t g = nullptr;
  long long nodes = 0;
  rc = factor_graph(ctx, TT_KERNEL_LU, a, n, ld, by, bx, &g, &nodes);
  if (rc) return rc;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (g) TT_CUDA(ctx, cudaGraphLaunch(g, s), "cudaGraphLaunch");
  ctx->launches += static_cast<unsigned long long>(nodes);
  if (fail_index) {  // synchronous status check requested
    rc = ensure_info_slots(ctx, 1);
    if (rc) return rc;
    TT_CUDA(ctx, cudaMemcpyAsync(ctx->info_host, ctx->info, sizeof(int), cudaMemcpyDeviceToHost, s),
            "status readback");
    TT_CUDA(ctx, cudaStreamSynchronize(s), "lu");
    *fail_index = -1;
    const int saved = ctx->kernel;
    ctx->kernel = TT_KERNEL_LU;
    rc = numeric_status(ctx, ctx->info_host[0], fail_index);
    ctx->kernel = saved;
    return rc;
  }
  return TT_OK;
}

int tt_dev_cholesky(tt_ctx* ctx, double* a, int n, int ld, int by, int bx, int* fail_index,
                    void* stream) {
  if (!ctx || !a) return TT_EINVAL;
  int rc = validate_factor(ctx, TT_KERNEL_CHOLESKY, n, n, by, bx);
  if (rc) return rc;
  if (ld < n || (ld & 1)) return fail(ctx, TT_EINVAL, "leading dimension must be even and >= n");
  if (!aligned16(a)) return fail(ctx, TT_EINVAL, "matrix base must be 16-byte aligned");
  DeviceGuard dg(ctx->device);
  TT_CUDA(ctx, dg.err, "cudaSetDevice");
  cudaGraphExec_t g = nullptr;
  long long nodes = 0;
  rc = factor_graph(ctx, TT_KERNEL_CHOLESKY, a, n, ld, by, bx, &g, &nodes);
  if (rc) return rc;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (g) TT_CUDA(ctx, cudaGraphLaunch(g, s), "cudaGraphLaunch");
  ctx->launches += static_cast<unsigned long long>(nodes);
  if (fail_index) {
    rc = ensure_info_slots(ctx, 1);
    if (rc) return rc;
    TT_CUDA(ctx, cudaMemcpyAsync(ctx->info_host, ctx->info, sizeof(int), cudaMemcpyDeviceToHost, s),
            "status readback");
    TT_CUDA(ctx, cudaStreamSynchronize(s), "cholesky");
    *fail_index = -1;
    const int saved = ctx->kernel;
    ctx->kernel = TT_KERNEL_CHOLESKY;
    rc = numeric_status(ctx, ctx->info_host[0], fail_index);
    ctx->kernel = saved;
    return rc;
  }
  return TT_OK;
}

int tt_dev_mm3(tt_ctx* ctx, const double* a, int lda, const double* b, int ldb, const double* c,
               int ldc, const double* d, int ldd, double* e, int lde, double* f, int ldf,
               double* g, int ldg, int n, int l, int m, int o, int p, const int* cfg, int ncfg,
               void* stream) {
  if (!ctx || !a || !b || !c || !d || !e || !f || !g || !cfg) return TT_EINVAL;
  int rc = validate_mm3(ctx, n, l, m, o, p, cfg, ncfg);
  if (rc) return rc;
  for (const void* q : {static_cast<const void*>(a), static_cast<const void*>(b),
                        static_cast<const void*>(c), static_cast<const void*>(d),
                        static_cast<const void*>(e), static_cast<const void*>(f),
                        static_cast<const void*>(g)})
    if (!aligned16(q)) return fail(ctx, TT_EINVAL, "3mm: operand bases must be 16-byte aligned");
  if ((lda | ldb | ldc | ldd | lde | ldf | ldg) & 1)
    return fail(ctx, TT_EINVAL, "3mm: leading dimensions must be even");
  DeviceGuard dg(ctx->device);
  TT_CUDA(ctx, dg.err, "cudaSetDevice");
  tt::Mm3Bufs bufs{a, b, c, d, lda, ldb, ldc, ldd, e, f, g, lde, ldf, ldg};
  const int dims[5] = {n, l, m, o, p};
  cudaGraphExec_t gx = nullptr;
  long long nodes = 0;
  rc = mm3_graph(ctx, bufs, dims, cfg, &gx, &nodes);
  if (rc) return rc;
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (gx) TT_CUDA(ctx, cudaGraphLaunch(gx, s), "cudaGraphLaunch");
  ctx->launches += static_cast<unsigned long long>(nodes);
  return TT_OK;
}

int tt_dev_fill_uniform(tt_ctx* ctx, double* a, int rows, int cols, int ld, long long row0,
                        uint64_t seed, int stream_id, void* stream) {
  if (!ctx || !a || rows < 0 || cols < 0 || ld < cols) return TT_EINVAL;
  DeviceGuard dg(ctx->device);
  TT_CUDA(ctx, dg.err, "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  tt::launch_fill_uniform(a, ld, rows, cols, row0, seed, stream_id, s);
  TT_CUDA(ctx, cudaGetLastError(), "fill_uniform");
  ctx->launches += 1;
  return TT_OK;
}

int tt_dag_tasks(int kernel, int n, int by, int bx, int* out, int cap) {
  if (!tt::dag::eligible(n, by, bx)) return -1;
  const std::vector<int4> v = tt::dag::build_tasks(kernel != TT_KERNEL_LU, n, by, bx, nullptr);
  if (out) {
    const size_t m = std::min(v.size(), static_cast<size_t>(std::max(cap, 0)));
    for (size_t i = 0; i < m; ++i) {
      out[4 * i] = v[i].x;
      out[4 * i + 1] = v[i].y;
      out[4 * i + 2] = v[i].z;
      out[4 * i + 3] = v[i].w;
    }
  }
  return static_cast<int>(v.size());
}

int tt_dag_chunk_depth(int n, int by, int bx) {
  if (!tt::dag::eligible(n, by, bx)) return -1;
  return tt::dag::chunk_depth(n, bx);
}

int tt_dag_tile(int n, int by, int bx) {
  if (!tt::dag::eligible(n, by, bx)) return -1;
  return tt::dag::tile_for(n, bx);
}

int tt_dag_region_rows(int n, int by, int bx) {
  if (!tt::dag::eligible(n, by, bx)) return -1;
  return tt::dag::region_rows(by, tt::dag::tile_for(n, bx));
}

int tt_gemm_plan(int m, int n, int fy, int fx, int* out) {
  if (m < 1 || n < 1 || fy < 1 || fx < 1 || !out) return TT_EINVAL;
  const tt::GemmPlan p = tt::plan_gemm(m, n, fy, fx);
  out[0] = p.reg_y;
  out[1] = p.reg_x;
  out[2] = p.bm;
  out[3] = p.bn;
  out[4] = tt::consumer_warps(p.bm, p.bn);
  return TT_OK;
}

int tt_dag_urgent(int kernel, int n, int by, int bx) {
  if (!tt::dag::eligible(n, by, bx)) return -1;
  int nu = 0;
  tt::dag::build_tasks(kernel != TT_KERNEL_LU, n, by, bx, &nu);
  return nu;
}

int tt_dag_trace(tt_ctx* ctx, unsigned long long* out, int cap) {
  if (!ctx || !ctx->dag_last || !ctx->dag_last->trace) return -1;
  const tt::dag::Workspace* w = ctx->dag_last;
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream), "trace sync");
  const int total = w->ntasks + w->nsteps;  // queue tasks, then one row per walker step
  const int m = std::min(total, std::max(cap, 0));
  if (out && m > 0)
    TT_CUDA(ctx, cudaMemcpy(out, w->trace, static_cast<size_t>(m) * 8 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost),
            "trace copy");
  return total;
}

int tt_dev_gemm(tt_ctx* ctx, const double* a, int lda, const double* b, int ldb, int b_trans,
                double* c, int ldc, int M, int N, int K, int fy, int fx, int alpha, int beta,
                void* stream) {
  if (!ctx || !a || !b || !c) return TT_EINVAL;
  if (M < 1 || N < 1 || K < 0) return fail(ctx, TT_EINVAL, "gemm: bad extents");
  if ((alpha != 1 && alpha != -1) || (beta != 0 && beta != 1))
    return fail(ctx, TT_EINVAL, "gemm: alpha must be +/-1 and beta 0 or 1");
  int rc = require_tile(ctx, fy, M, "matmul_tiled");
  if (rc) return rc;
  rc = require_tile(ctx, fx, N, "matmul_tiled");
  if (rc) return rc;
  if ((lda & 1) || (ldb & 1)) return fail(ctx, TT_EINVAL, "gemm: leading dims must be even");
  DeviceGuard dg(ctx->device);
  TT_CUDA(ctx, dg.err, "cudaSetDevice");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const tt::Operand A{a, M, std::max(K, 1), lda, 0, 0};
  const tt::Operand B = b_trans ? tt::Operand{b, N, std::max(K, 1), ldb, 0, 0}
                                : tt::Operand{b, std::max(K, 1), N, ldb, 0, 0};
  TT_CUDA(ctx,
          tt::gemm(ctx->tmaps, A, B, b_trans != 0, c, ldc, M, N, K, fy, fx, alpha < 0 ? 1 : 0,
                   beta, 0, 0, s),
          "gemm");
  ctx->launches += 1;
  return TT_OK;
}

}  // extern "C"
