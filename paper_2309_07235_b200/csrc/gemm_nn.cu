// NN instantiations of the DMMA GEMM family (3mm products, LU updates).
#include "gemm_variants.cuh"

namespace tt {
cudaError_t launch_nn(int bm, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& tc, const GemmArgs& args, long long grid, cudaStream_t stream) {
  TT_DISPATCH(false)
}
}  // namespace tt
