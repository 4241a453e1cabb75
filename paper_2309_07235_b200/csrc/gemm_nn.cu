// NN instantiations of the DMMA GEMM family (3mm products, LU updates).
#include "gemm_variants.cuh"

namespace tt {
cudaError_t launch_nn(int bm, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                      const CUtensorMap& tc, const GemmArgs& args, long long grid, cudaStream_t stream) {
  TT_DISPATCH(false)
}

// GemmShape<bm, bn>::NCW of the instantiated variants (introspection).
int consumer_warps(int bm, int bn) {
#define TT_NCW_BN(BM)                                   \
  switch (bn) {                                         \
    case 8: return GemmShape<BM, 8, false>::NCW;        \
    case 16: return GemmShape<BM, 16, false>::NCW;      \
    case 32: return GemmShape<BM, 32, false>::NCW;      \
    case 64: return GemmShape<BM, 64, false>::NCW;      \
    case 128: return GemmShape<BM, 128, false>::NCW;    \
  }                                                     \
  return 0;
  switch (bm) {
    case 8: { TT_NCW_BN(8) }
    case 16: { TT_NCW_BN(16) }
    case 32: { TT_NCW_BN(32) }
    case 64: { TT_NCW_BN(64) }
    case 128: { TT_NCW_BN(128) }
  }
  return 0;
#undef TT_NCW_BN
}
}  // namespace tt
