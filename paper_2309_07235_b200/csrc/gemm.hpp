// Host side of the knob-driven DMMA GEMM: operand views, the TMA descriptor
// cache and the knob -> variant mapping (part of the per-config
// instantiation cache).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <tuple>

#include "dgemm.cuh"

namespace tt {

// A matrix view: full row-major matrix (base, rows x cols, leading dim ld)
// plus the origin (r0, c0) of the operand inside it.  TMA descriptors are
// built for the full matrix so out-of-matrix reads zero-fill; the kernel
// masks the K edge of the view itself.
struct Operand {
  const double* base;
  int rows, cols;
  long long ld;
  int r0, c0;
};

class TmapCache {
 public:
  // 2-D fp64 map over the full matrix, box = 16 columns x box_rows rows,
  // 128B swizzle.  Returns nullptr on an encode failure.
  const CUtensorMap* get(const double* base, int rows, int cols, long long ld, int box_rows);
  // Unswizzled map with an arbitrary (even) box width, for the C prefetch.
  const CUtensorMap* get_plain(const double* base, int rows, int cols, long long ld, int box_rows,
                               int box_cols);
  void clear() { maps_.clear(); }
  size_t size() const { return maps_.size(); }

 private:
  std::map<std::tuple<const void*, int, int, long long, int, int>, CUtensorMap> maps_;
};

// Region (knob) -> launch geometry.  Sub-atom regions are packed into the
// 8x8 DMMA atom; the tile edge is the smallest of {8,16,32,64,128} covering
// the region edge (capped at 128; larger regions are swept in tile steps).
struct GemmPlan {
  int reg_y, reg_x;  // effective CTA region
  int bm, bn;        // tile variant
  int nreg_y, nreg_x;
  long long grid() const { return static_cast<long long>(nreg_y) * nreg_x; }
};
GemmPlan plan_gemm(int M, int N, int fy, int fx);
// DMMA consumer warps of the BM x BN variant (GemmShape<BM, BN>::NCW).
int consumer_warps(int bm, int bn);

// C (+)= (+/-) A * B on `stream`.  c points at the output view origin.
// lower: write only view elements with i + diag_off >= j (Cholesky).
cudaError_t gemm(TmapCache& tc, const Operand& A, const Operand& B, bool b_trans, double* c,
                 long long ldc, int M, int N, int K, int fy, int fx, int alpha_neg, int beta,
                 int lower, int diag_off, cudaStream_t stream);

// Per-variant launchers (gemm_nn.cu / gemm_nt.cu).
cudaError_t launch_nn(int bm, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& tc, const GemmArgs& args, long long grid,
                      cudaStream_t stream);
cudaError_t launch_nt(int bm, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& tc, const GemmArgs& args, long long grid,
                      cudaStream_t stream);

}  // namespace tt
