// Host side of the DMMA GEMM: TMA descriptor cache, knob -> variant plan,
// launch.  See gemm.hpp.
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "gemm.hpp"

namespace tt {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int tile_edge(int reg) {
  for (int t : {8, 16, 32, 64}) {
    if (reg <= t) return t;
  }
  return 128;
}

// Knob region -> CTA region (one CTA per region, every output element one
// full-K reduction by one CTA: the arithmetic per element is the same for
// every mapping).  The knob's region edge f (the reference's outer tile,
// kernels.cpp:91-111) is kept as the CTA edge inside [32, 128]; outside it:
//   f < 32:  floor(64 / f) adjacent knob regions are packed into one CTA
//            region (as the DMMA atom packs sub-8 regions), so a CTA never
//            runs a warp tile narrower than 32;
//   f > 128: the region is split into its s equal parts for the smallest
//            divisor s of f with f / s <= 128 (so part edges stay on region
//            edges), else into ceil(f / 128) near-equal parts — one CTA per
//            part instead of one CTA sweeping a long region alone.
int pack_region(int f, int extent) {
  int r = f;
  if (f < 32) {
    r = f * std::max(1, 64 / f);
  } else if (f > 128) {
    int s = (f + 127) / 128;
    while (f % s && f / s >= 32) ++s;
    r = f % s ? (f + (f + 127) / 128 - 1) / ((f + 127) / 128) : f / s;
  }
  return std::max(1, std::min(r, extent));
}

// A base that is only 8-byte aligned is moved back one element (origin
// column + 1) so the tensor map base is 16-byte aligned.
bool align_base(Operand& o) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(o.base);
  if (addr % 8) return false;
  if (addr % 16) {
    o.base -= 1;
    o.c0 += 1;
    o.cols += 1;
  }
  return true;
}

}  // namespace

namespace {

bool encode(CUtensorMap* m, const double* base, int rows, int cols, long long ld, int box_rows,
            int box_cols, bool swizzle) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

const CUtensorMap* TmapCache::get(const double* base, int rows, int cols, long long ld,
                                  int box_rows) {
  auto key = std::make_tuple(static_cast<const void*>(base), rows, cols, ld, box_rows, 0);
  auto it = maps_.find(key);
  if (it != maps_.end()) return &it->second;
  CUtensorMap m;
  if (!encode(&m, base, rows, cols, ld, box_rows, 16, true)) return nullptr;
  return &maps_.emplace(key, m).first->second;
}

const CUtensorMap* TmapCache::get_plain(const double* base, int rows, int cols, long long ld,
                                        int box_rows, int box_cols) {
  auto key = std::make_tuple(static_cast<const void*>(base), rows, cols, ld, box_rows, box_cols);
  auto it = maps_.find(key);
  if (it != maps_.end()) return &it->second;
  CUtensorMap m;
  if (!encode(&m, base, rows, cols, ld, box_rows, box_cols, false)) return nullptr;
  return &maps_.emplace(key, m).first->second;
}

GemmPlan plan_gemm(int M, int N, int fy, int fx) {
  GemmPlan p;
  p.reg_y = pack_region(fy, M);
  p.reg_x = pack_region(fx, N);
  p.bm = tile_edge(p.reg_y);
  p.bn = tile_edge(p.reg_x);
  p.nreg_y = (M + p.reg_y - 1) / p.reg_y;
  p.nreg_x = (N + p.reg_x - 1) / p.reg_x;
  return p;
}

cudaError_t gemm(TmapCache& tc, const Operand& A, const Operand& B, bool b_trans, double* c,
                 long long ldc, int M, int N, int K, int fy, int fx, int alpha_neg, int beta,
                 int lower, int diag_off, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const GemmPlan plan = plan_gemm(M, N, fy, fx);
  // TMA boxes must start 16-byte aligned: the matrix bases must be, and an
  // odd k origin is moved one column left with that column masked (klo).
  Operand a = A, b = B;
  if (!align_base(a) || !align_base(b)) return cudaErrorInvalidValue;
  int klo = 0;
  if (a.c0 & 1) {
    klo = 1;
    a.c0 -= 1;
    if (b_trans) {
      if (!(b.c0 & 1)) return cudaErrorInvalidValue;  // A and B^T k origins must share parity
      b.c0 -= 1;
    } else {
      b.r0 -= 1;
    }
  } else if (b_trans && (b.c0 & 1)) {
    return cudaErrorInvalidValue;
  }
  const CUtensorMap* ta = tc.get(a.base, a.rows, a.cols, a.ld, plan.bm);
  const CUtensorMap* tb = b_trans ? tc.get(b.base, b.rows, b.cols, b.ld, plan.bn)
                                  : tc.get(b.base, b.rows, b.cols, b.ld, 16);
  if (!ta || !tb) return cudaErrorInvalidValue;
  GemmArgs args;
  args.c = c;
  args.ldc = ldc;
  args.M = M;
  args.N = N;
  args.K = K;
  args.a_r0 = a.r0;
  args.a_c0 = a.c0;
  args.b_r0 = b.r0;
  args.b_c0 = b.c0;
  args.klo = klo;
  args.reg_y = plan.reg_y;
  args.reg_x = plan.reg_x;
  args.nreg_x = plan.nreg_x;
  args.alpha_neg = alpha_neg;
  args.beta = beta;
  args.lower = lower;
  args.diag_off = diag_off;
  // C prefetch map (beta = 1): over the M x N view, 16-byte aligned base, an
  // even leading dimension (TMA stride rule); otherwise plain loads.
  args.c_tma = 0;
  args.c_sh = 0;
  const CUtensorMap* tcm = ta;
  const uintptr_t caddr = reinterpret_cast<uintptr_t>(c);
  // (the 8-consumer-warp tiles, >= 128 x 64, issue TMA in line: no C prefetch)
  if (beta && plan.bm * plan.bn < 128 * 64 && (ldc % 2) == 0 && (caddr % 8) == 0) {
    const int sh = (caddr % 16) ? 1 : 0;
    const CUtensorMap* m = tc.get_plain(c - sh, M, N + sh, ldc, plan.bm, plan.bn + 2);
    if (m) {
      tcm = m;
      args.c_tma = 1;
      args.c_sh = sh;
    }
  }
  return b_trans ? launch_nt(plan.bm, plan.bn, *ta, *tb, *tcm, args, plan.grid(), stream)
                 : launch_nn(plan.bm, plan.bn, *ta, *tb, *tcm, args, plan.grid(), stream);
}

}  // namespace tt
