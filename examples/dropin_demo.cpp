// Compile-time proof that the drop-in shim takes the reference's own types:
// built against /root/reference/proj/core/include (when present) by
// tests/test_abi.py::test_cpp_shim_compiles_against_reference_types.
#include <cstdio>

#include "tiletuner/kernels.hpp"
#include "tiletuner/matrix.hpp"
#include "tiletuner/space.hpp"
#include "tiletuner_gpu.hpp"

int main() {
  tiletuner::Matrix a(2, 2);
  a(0, 0) = 4;
  a(0, 1) = 3;
  a(1, 0) = 6;
  a(1, 1) = 3;
  try {
    tiletuner_gpu::lu_factor_inplace(a, 1, 1);  // kernels_test.cpp:166-181 on the GPU
    std::printf("L21=%g U11=%g\n", a(1, 0), a(1, 1));
    tiletuner::Configuration cfg{{1, 1, 1, 1, 1, 1}};
    tiletuner::Matrix x(1, 2), y(2, 1), z(1, 1), w(1, 1);
    x(0, 0) = 1; x(0, 1) = 2; y(0, 0) = 3; y(1, 0) = 4; z(0, 0) = 5; w(0, 0) = 6;
    tiletuner::Matrix g = tiletuner_gpu::mm3_tiled(x, y, z, w, cfg);
    std::printf("G=%g\n", g(0, 0));
    return (a(1, 0) == 1.5 && a(1, 1) == -1.5 && g(0, 0) == 330.0) ? 0 : 1;
  } catch (const tiletuner::MeasurementError& e) {
    std::printf("no GPU: %s\n", e.what());
    return 3;
  }
}
