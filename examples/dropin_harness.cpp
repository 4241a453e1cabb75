// The C++ drop-in exercised end to end on a GPU, inside one program that also
// links the UNMODIFIED reference core (oracle/_ref/libtiletuner_ref.so, built
// from /root/reference sources by oracle/Makefile):
//
//   1. INTEGRATION.md section 2: tiletuner_gpu::{lu,cholesky}_factor_inplace and
//      mm3_tiled take the reference's own tiletuner::Matrix / Configuration, on
//      the reference's own inputs (tiletuner::gen_spd, gen_3mm_inputs); results
//      are checked against the reference's own CPU kernels (lu_factor_inplace,
//      cholesky_factor_inplace, mm3_reference, kernels.hpp:29-66) and its own
//      residuals (lu_residual / cholesky_residual, kernels.hpp:69-70).
//   2. INTEGRATION.md section 3: the patched harness measure(KernelCase,
//      Configuration, MeasureProtocol) (harness.cpp:99-105) built on
//      tiletuner_gpu::GpuKernelRunner returns a positive device time for every
//      kernel, next to the reference's own CPU measure().
//   3. The error convention: a knob that does not divide n throws the
//      reference's std::invalid_argument through the shim.
//
// Exit code 0 = all checks passed, 1 = a check failed, 3 = no GPU
// (tiletuner::MeasurementError from the shim).
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "tiletuner/harness.hpp"
#include "tiletuner/kernels.hpp"
#include "tiletuner/matrix.hpp"
#include "tiletuner/problem.hpp"
#include "tiletuner/space.hpp"
#include "tiletuner_gpu.hpp"

namespace {

int failures = 0;

void expect(bool ok, const char* what, double v) {
  std::printf("%-58s %-4s %.3e\n", what, ok ? "ok" : "FAIL", v);
  if (!ok) ++failures;
}

double max_rel(const tiletuner::Matrix& x, const tiletuner::Matrix& y, bool lower_only) {
  double num = 0.0, den = 0.0;
  for (int i = 0; i < x.rows; ++i)
    for (int j = 0; j < x.cols; ++j) {
      if (lower_only && j > i) continue;
      num = std::fmax(num, std::fabs(x(i, j) - y(i, j)));
      den = std::fmax(den, std::fabs(y(i, j)));
    }
  return num / den;
}

// the patched harness objective.
double gpu_measure(const tiletuner::KernelCase& kase, const tiletuner::Configuration& config,
                   const tiletuner::MeasureProtocol& protocol) {
  tiletuner_gpu::GpuKernelRunner runner(static_cast<int>(kase.size.kernel), kase.size.n,
                                        kase.size.l, kase.size.m, kase.size.o, kase.size.p,
                                        kase.seed);
  return runner.measure(config.values, protocol.warmups, protocol.repetitions,
                        static_cast<int>(protocol.aggregate));
}

}  // namespace

int main() {
  using namespace tiletuner;
  try {
    // ---- 1. drop-in kernels on the reference's own inputs vs its own CPU kernels
    {
      const int n = 400;
      const Matrix a = gen_spd(n, 1);
      Matrix cpu = a, gpu = a;
      lu_factor_inplace(cpu, 100, 40);
      tiletuner_gpu::lu_factor_inplace(gpu, 100, 40);
      expect(max_rel(gpu, cpu, false) <= 1e-10, "lu_factor_inplace(400, 100, 40) vs reference", max_rel(gpu, cpu, false));
      LuFactors f{Matrix(n, n), Matrix(n, n)};
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          if (j < i) f.l(i, j) = gpu(i, j);
          else f.u(i, j) = gpu(i, j);
          if (i == j) f.l(i, j) = 1.0;
        }
      const double r = lu_residual(a, f);
      expect(r <= 1e-12, "reference lu_residual of the GPU factors", r);
    }
    {
      const int n = 400;
      const Matrix a = gen_spd(n, 2);
      Matrix cpu = a, gpu = a;
      cholesky_factor_inplace(cpu, 80, 50);
      tiletuner_gpu::cholesky_factor_inplace(gpu, 80, 50);
      expect(max_rel(gpu, cpu, true) <= 1e-10, "cholesky_factor_inplace(400, 80, 50) vs reference", max_rel(gpu, cpu, true));
      Matrix l(n, n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) l(i, j) = gpu(i, j);
      const double r = cholesky_residual(a, l);
      expect(r <= 1e-12, "reference cholesky_residual of the GPU factor", r);
      bool upper_same = true;  // the reference never writes j > i
      for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) upper_same = upper_same && gpu(i, j) == a(i, j);
      expect(upper_same, "cholesky upper triangle untouched", 0.0);
    }
    {
      ProblemSize dims;
      dims.kernel = Kernel::mm3;
      dims.n = 80; dims.l = 90; dims.m = 100; dims.o = 110; dims.p = 120;
      const Mm3Inputs in = gen_3mm_inputs(dims, 1);
      const Matrix ref = mm3_reference(in.a, in.b, in.c, in.d);
      const Configuration cfg{{16, 25, 20, 24, 40, 24}};
      const Matrix g = tiletuner_gpu::mm3_tiled(in.a, in.b, in.c, in.d, cfg);
      expect(max_rel(g, ref, false) <= 1e-10, "mm3_tiled(80..120, cfg) vs mm3_reference", max_rel(g, ref, false));
    }
    // ---- 2. the patched harness measure() (GPU) next to the reference's CPU measure()
    {
      const MeasureProtocol protocol{1, 3, Aggregate::median};
      for (const char* name : {"lu", "cholesky", "3mm"}) {
        const std::string kn(name);
        for (const ProblemSize& ps : registered_sizes()) {
          if (std::string(kernel_name(ps.kernel)) != kn || ps.name != "small") continue;
          const KernelCase kase{ps, 1};
          const ParamSpace space = build_space(ps.kernel, ps.name);
          const Configuration cfg = config_at(space, space_size(space) / 2);
          const double g = gpu_measure(kase, cfg, protocol);
          const double c = measure(kase, cfg, protocol);
          char what[96];
          std::snprintf(what, sizeof what, "measure(%s small) GPU %.3g s, reference CPU %.3g s", name, g, c);
          expect(g > 0.0 && std::isfinite(g), what, g);
        }
      }
    }
    // ---- 3. error convention through the shim
    {
      Matrix a = gen_spd(64, 1);
      bool threw = false;
      try {
        tiletuner_gpu::lu_factor_inplace(a, 7, 8);  // 7 does not divide 64
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      expect(threw, "non-divisor knob -> std::invalid_argument", 0.0);
    }
  } catch (const MeasurementError& e) {
    std::printf("no GPU: %s\n", e.what());
    return 3;
  }
  std::printf("%s\n", failures ? "FAILED" : "ALL OK");
  return failures ? 1 : 0;
}
