// tiletuner_gpu.hpp — header-only C++ drop-in for the reference's timed kernel
// entry points, implemented over the C ABI of libtt_gpu.so (include/tt_gpu.h).
//
//   reference (kernels.hpp)                         this header
//   void lu_factor_inplace(Matrix&, int, int)       tiletuner_gpu::lu_factor_inplace
//   void cholesky_factor_inplace(Matrix&, int, int) tiletuner_gpu::cholesky_factor_inplace
//   Matrix mm3_tiled(a, b, c, d, Configuration)     tiletuner_gpu::mm3_tiled
//   KernelRunner::measure (harness.cpp:99-105)      tiletuner_gpu::GpuKernelRunner::measure
//
// The functions are templates over the matrix type so they take the
// reference's tiletuner::Matrix (rows, cols, std::vector<double> data,
// row-major) unchanged.  When the reference headers are on the include path
// the errors are the reference's own types (std::invalid_argument,
// tiletuner::NumericalError, tiletuner::MeasurementError); otherwise local
// equivalents with the same names are declared.  See INTEGRATION.md.
#pragma once

#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tt_gpu.h"

#if __has_include("tiletuner/errors.hpp")
#include "tiletuner/errors.hpp"
namespace tiletuner_gpu {
using NumericalError = tiletuner::NumericalError;
using MeasurementError = tiletuner::MeasurementError;
}  // namespace tiletuner_gpu
#else
namespace tiletuner_gpu {
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class MeasurementError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
}  // namespace tiletuner_gpu
#endif

namespace tiletuner_gpu {

// One context per (host thread, device): tt_ctx is single-owner state.
inline tt_ctx* context(int device = 0) {
  struct Holder {
    tt_ctx* h[64] = {};
    ~Holder() {
      for (tt_ctx* c : h)
        if (c) tt_ctx_destroy(c);
    }
  };
  thread_local Holder holder;
  if (device < 0 || device >= 64) throw std::invalid_argument("device index out of range");
  if (!holder.h[device]) {
    const int rc = tt_ctx_create(device, &holder.h[device]);
    if (rc != TT_OK) throw MeasurementError("tt_ctx_create: no usable CUDA device (no CPU fallback)");
  }
  return holder.h[device];
}

inline void check(tt_ctx* c, int rc) {
  switch (rc) {
    case TT_OK: return;
    case TT_EINVAL: throw std::invalid_argument(tt_last_error(c));
    case TT_ENUMERIC: throw NumericalError(tt_last_error(c));
    case TT_ENOMEM: throw std::bad_alloc();
    default: throw MeasurementError(tt_last_error(c));
  }
}

// kernels.hpp:65
template <class MatrixT>
void lu_factor_inplace(MatrixT& a, int by, int bx, int device = 0) {
  tt_ctx* c = context(device);
  int idx = -1;
  check(c, tt_lu_factor_inplace(c, a.data.data(), a.rows, a.cols, by, bx, &idx));
}

// kernels.hpp:66
template <class MatrixT>
void cholesky_factor_inplace(MatrixT& a, int by, int bx, int device = 0) {
  tt_ctx* c = context(device);
  int idx = -1;
  check(c, tt_cholesky_factor_inplace(c, a.data.data(), a.rows, a.cols, by, bx, &idx));
}

// kernels.hpp:43-44 (config: anything with .values, e.g. tiletuner::Configuration)
template <class MatrixT, class ConfigT>
MatrixT mm3_tiled(const MatrixT& a, const MatrixT& b, const MatrixT& c, const MatrixT& d,
                  const ConfigT& config, int device = 0) {
  if (a.cols != b.rows || b.cols != c.rows || c.cols != d.rows)
    throw std::invalid_argument("matmul: inner dimensions disagree");
  tt_ctx* ctx = context(device);
  MatrixT g(a.rows, d.cols);
  const std::vector<int>& v = config.values;
  check(ctx, tt_mm3_tiled(ctx, a.data.data(), b.data.data(), c.data.data(), d.data.data(),
                          a.rows, a.cols, b.cols, c.cols, d.cols, v.data(),
                          static_cast<int>(v.size()), g.data.data()));
  return g;
}

// The KernelRunner twin (harness.cpp:89-143): inputs generated once on the
// device (bitwise gen_spd / gen_3mm_inputs), every sample a fresh copy,
// CUDA-event timing, the reference's aggregation.
class GpuKernelRunner {
 public:
  // kernel: 0 lu, 1 cholesky, 2 3mm; dims (n, l, m, o, p) as ProblemSize.
  GpuKernelRunner(int kernel, int n, int l, int m, int o, int p, unsigned long long seed,
                  int device = 0)
      : ctx_(context(device)) {
    check(ctx_, tt_setup_seeded(ctx_, kernel, n, l, m, o, p, seed));
  }
  // aggregate: 0 median, 1 min, 2 mean (harness.hpp:22)
  double measure(const std::vector<int>& config, int warmups = 1, int reps = 3,
                 int aggregate = TT_AGG_MEDIAN) {
    double s = 0.0;
    check(ctx_, tt_measure(ctx_, config.data(), static_cast<int>(config.size()), warmups, reps,
                           aggregate, &s));
    return s;
  }

 private:
  tt_ctx* ctx_;
};

}  // namespace tiletuner_gpu
