// NT instantiations of the DMMA GEMM family (Cholesky SYRK/GEMM updates, B given as N x K).
#include "gemm_variants.cuh"

namespace tt {
cudaError_t launch_nt(int bm, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& tc, const GemmArgs& args, long long grid, cudaStream_t stream) {
  TT_DISPATCH(true)
}
}  // namespace tt
