// Instantiation helper for the AOT DMMA GEMM family.
#pragma once
#include "devattr.hpp"
#include "gemm.hpp"

namespace tt {

template <int BM, int BN, bool BT>
cudaError_t launch_variant(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                           const GemmArgs& args, long long grid, cudaStream_t stream) {
  using S = GemmShape<BM, BN, BT>;
  static std::atomic<unsigned long long> configured{0};  // per variant, one bit per device
  const cudaError_t e = smem_optin(dgemm_kernel<BM, BN, BT>, S::SMEM_OPT, configured);
  if (e != cudaSuccess) return e;
  if (grid <= 0) return cudaSuccess;
  const bool c_tma = args.beta && args.c_tma;
  if (c_tma && S::SMEM_OPT < S::SMEM) return cudaErrorInvalidValue;  // plan_gemm never asks
  dgemm_kernel<BM, BN, BT><<<static_cast<unsigned>(grid), S::THREADS, c_tma ? S::SMEM : S::SMEM_NOC,
                             stream>>>(ta, tb, tc, args);
  return cudaGetLastError();
}

#define TT_DISPATCH_BN(BM, BT)                                                  \
  switch (bn) {                                                                 \
    case 8: return launch_variant<BM, 8, BT>(ta, tb, tc, args, grid, stream);       \
    case 16: return launch_variant<BM, 16, BT>(ta, tb, tc, args, grid, stream);     \
    case 32: return launch_variant<BM, 32, BT>(ta, tb, tc, args, grid, stream);     \
    case 64: return launch_variant<BM, 64, BT>(ta, tb, tc, args, grid, stream);     \
    case 128: return launch_variant<BM, 128, BT>(ta, tb, tc, args, grid, stream); \
  }                                                                             \
  return cudaErrorInvalidValue;

#define TT_DISPATCH(BT)                      \
  switch (bm) {                              \
    case 8: { TT_DISPATCH_BN(8, BT) }        \
    case 16: { TT_DISPATCH_BN(16, BT) }      \
    case 32: { TT_DISPATCH_BN(32, BT) }      \
    case 64: { TT_DISPATCH_BN(64, BT) }      \
    case 128: { TT_DISPATCH_BN(128, BT) }    \
  }                                          \
  return cudaErrorInvalidValue;

}  // namespace tt
