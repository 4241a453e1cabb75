// Per-device opt-in to large dynamic shared memory.  The attribute set by
// cudaFuncSetAttribute belongs to the CURRENT device, so a process driving
// several GPUs (one tt_ctx per device) must set it once per (kernel,
// device); `done` holds one bit per device ordinal.  Racing setters are
// harmless (the call is idempotent).
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace tt {

template <class K>
cudaError_t smem_optin(K* kernel, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

}  // namespace tt
