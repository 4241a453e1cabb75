// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/core/src/*.cpp (see oracle/Makefile; output goes to
// oracle/_ref/libtiletuner_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference arm load it, as the checker and
// the CPU baseline.  Every wrapper forwards to the reference symbol named in
// its comment; exceptions are mapped to the same status codes the product
// C-ABI uses (include/tt_gpu.h): 0 ok, 1 invalid_argument, 2 NumericalError,
// 3 MeasurementError, 9 anything else.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "tiletuner/errors.hpp"
#include "tiletuner/harness.hpp"
#include "tiletuner/kernels.hpp"
#include "tiletuner/problem.hpp"
#include "tiletuner/space.hpp"
#include "tiletuner/tuners.hpp"

using namespace tiletuner;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const MeasurementError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Matrix to_matrix(const double* p, int r, int c) {
  Matrix m(r, c);
  std::memcpy(m.data.data(), p, sizeof(double) * static_cast<std::size_t>(r) * c);
  return m;
}

void from_matrix(const Matrix& m, double* p) {
  std::memcpy(p, m.data.data(), sizeof(double) * m.data.size());
}

Kernel kernel_of(int k) {
  switch (k) {
    case 0: return Kernel::lu;
    case 1: return Kernel::cholesky;
    case 2: return Kernel::mm3;
  }
  throw std::invalid_argument("ref_capi: unknown kernel id");
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// kernels.cpp:38 gen_spd
int ref_gen_spd(int n, std::uint64_t seed, double* out) {
  return guarded([&] { from_matrix(gen_spd(n, seed), out); });
}

// kernels.cpp:57 gen_3mm_inputs
int ref_gen_3mm(int n, int l, int m, int o, int p, std::uint64_t seed, double* a,
                double* b, double* c, double* d) {
  return guarded([&] {
    ProblemSize s{Kernel::mm3, "custom", n, l, m, o, p};
    Mm3Inputs in = gen_3mm_inputs(s, seed);
    from_matrix(in.a, a);
    from_matrix(in.b, b);
    from_matrix(in.c, c);
    from_matrix(in.d, d);
  });
}

// kernels.cpp:115 mm3_reference
int ref_mm3_reference(const double* a, const double* b, const double* c,
                      const double* d, int n, int l, int m, int o, int p,
                      double* g) {
  return guarded([&] {
    from_matrix(mm3_reference(to_matrix(a, n, l), to_matrix(b, l, m),
                              to_matrix(c, m, o), to_matrix(d, o, p)),
                g);
  });
}

// kernels.cpp:122 mm3_tiled
int ref_mm3_tiled(const double* a, const double* b, const double* c,
                  const double* d, int n, int l, int m, int o, int p,
                  const int* cfg, int ncfg, double* g) {
  return guarded([&] {
    Configuration config;
    config.values.assign(cfg, cfg + ncfg);
    from_matrix(mm3_tiled(to_matrix(a, n, l), to_matrix(b, l, m),
                          to_matrix(c, m, o), to_matrix(d, o, p), config),
                g);
  });
}

// kernels.cpp:178 lu_factor_inplace (rows x cols lets tests hit require_square)
int ref_lu_factor_inplace(double* a, int rows, int cols, int by, int bx) {
  return guarded([&] {
    Matrix m = to_matrix(a, rows, cols);
    lu_factor_inplace(m, by, bx);
    from_matrix(m, a);
  });
}

// kernels.cpp:264 cholesky_factor_inplace
int ref_cholesky_factor_inplace(double* a, int rows, int cols, int by, int bx) {
  return guarded([&] {
    Matrix m = to_matrix(a, rows, cols);
    cholesky_factor_inplace(m, by, bx);
    from_matrix(m, a);
  });
}

// kernels.cpp:171 lu_reference -> packed (L strictly below, U on/above)
int ref_lu_reference_packed(const double* a, int n, double* packed) {
  return guarded([&] {
    LuFactors f = lu_reference(to_matrix(a, n, n));
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        packed[static_cast<std::size_t>(i) * n + j] = j < i ? f.l(i, j) : f.u(i, j);
  });
}

// kernels.cpp:257 cholesky_reference (lower, zeros above)
int ref_cholesky_reference(const double* a, int n, double* l) {
  return guarded([&] { from_matrix(cholesky_reference(to_matrix(a, n, n)), l); });
}

// kernels.cpp:326 lu_residual, fed the packed factor (unpacked like unpack_lu :158)
int ref_lu_residual_packed(const double* a, const double* packed, int n, double* out) {
  return guarded([&] {
    LuFactors f{Matrix(n, n), Matrix(n, n)};
    for (int i = 0; i < n; ++i) {
      f.l(i, i) = 1.0;
      for (int j = 0; j < i; ++j) f.l(i, j) = packed[static_cast<std::size_t>(i) * n + j];
      for (int j = i; j < n; ++j) f.u(i, j) = packed[static_cast<std::size_t>(i) * n + j];
    }
    *out = lu_residual(to_matrix(a, n, n), f);
  });
}

// kernels.cpp:340 cholesky_residual on the lower triangle of `fac`
int ref_cholesky_residual(const double* a, const double* fac, int n, double* out) {
  return guarded([&] {
    Matrix l(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) l(i, j) = fac[static_cast<std::size_t>(i) * n + j];
    *out = cholesky_residual(to_matrix(a, n, n), l);
  });
}

// kernels.cpp:366 residual_for(KernelCase{find_size(kernel,size), seed}, cfg)
int ref_residual_for(int kernel, const char* size, std::uint64_t seed,
                     const int* cfg, int ncfg, double* out) {
  return guarded([&] {
    KernelCase kase{find_size(kernel_of(kernel), size), seed};
    Configuration config;
    config.values.assign(cfg, cfg + ncfg);
    *out = residual_for(kase, config);
  });
}

// harness.cpp:160 measure(KernelCase, Configuration, MeasureProtocol)
int ref_measure(int kernel, const char* size, std::uint64_t seed, const int* cfg,
                int ncfg, int warmups, int reps, int aggregate, double* seconds) {
  return guarded([&] {
    KernelCase kase{find_size(kernel_of(kernel), size), seed};
    Configuration config;
    config.values.assign(cfg, cfg + ncfg);
    MeasureProtocol protocol;
    protocol.warmups = warmups;
    protocol.repetitions = reps;
    protocol.aggregate = aggregate == 1 ? Aggregate::min
                         : aggregate == 2 ? Aggregate::mean
                                          : Aggregate::median;
    *seconds = measure(kase, config, protocol);
  });
}

// harness.cpp:53 aggregate_samples
int ref_aggregate_samples(const double* s, int n, int aggregate, double* out) {
  return guarded([&] {
    std::vector<double> v(s, s + n);
    *out = aggregate_samples(v, aggregate == 1 ? Aggregate::min
                                : aggregate == 2 ? Aggregate::mean
                                                 : Aggregate::median);
  });
}

// space.cpp:10 divisor_candidates; returns the count, fills up to cap
int ref_divisor_candidates(int n, int* out, int cap) {
  std::vector<int> v;
  int rc = guarded([&] { v = divisor_candidates(n); });
  if (rc != 0) return -1;
  for (int i = 0; i < static_cast<int>(v.size()) && i < cap; ++i) out[i] = v[i];
  return static_cast<int>(v.size());
}

// space.cpp:30/:47 build_space + space_size
int ref_space_size(int kernel, const char* size, std::uint64_t* out) {
  return guarded([&] { *out = space_size(build_space(kernel_of(kernel), size)); });
}

// space.cpp:53 config_at
int ref_config_at(int kernel, const char* size, std::uint64_t flat, int* cfg) {
  return guarded([&] {
    Configuration c = config_at(build_space(kernel_of(kernel), size), flat);
    for (std::size_t i = 0; i < c.values.size(); ++i) cfg[i] = c.values[i];
  });
}

// space.cpp:78 index_of
int ref_index_of(int kernel, const char* size, const int* cfg, int ncfg,
                 std::uint64_t* out) {
  return guarded([&] {
    Configuration c;
    c.values.assign(cfg, cfg + ncfg);
    *out = index_of(build_space(kernel_of(kernel), size), c);
  });
}

// space.cpp:106 encode
int ref_encode(int kernel, const char* size, const int* cfg, int ncfg, double* out) {
  return guarded([&] {
    Configuration c;
    c.values.assign(cfg, cfg + ncfg);
    std::vector<double> f = encode(build_space(kernel_of(kernel), size), c);
    for (std::size_t i = 0; i < f.size(); ++i) out[i] = f[i];
  });
}

// harness.cpp:199 run_tuning with the synthetic objective (virtual clock):
// returns the evaluated flat indices and runtimes; used to pin the batched
// evaluator's k=1 equivalence.
int ref_run_tuning_synthetic(int kernel, const char* size, int tuner,
                             std::uint64_t seed, int max_evals,
                             std::uint64_t* flat_out, double* runtime_out,
                             int* n_out) {
  return guarded([&] {
    const ParamSpace space = build_space(kernel_of(kernel), size);
    Budget budget;
    budget.max_evals = static_cast<std::uint64_t>(max_evals);
    TuningTrace t = run_tuning(all_tuner_kinds().at(tuner), space,
                               SyntheticObjective{}, budget, MeasureProtocol{}, seed);
    *n_out = static_cast<int>(t.records.size());
    for (std::size_t i = 0; i < t.records.size(); ++i) {
      flat_out[i] = index_of(space, t.records[i].config);
      runtime_out[i] = t.records[i].runtime_s ? *t.records[i].runtime_s : -1.0;
    }
  });
}

}  // extern "C"
