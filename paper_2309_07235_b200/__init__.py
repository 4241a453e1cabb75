"""B200-native fp64 tuned kernels of arxiv/paper_2309_07235 (3mm, LU nopiv, Cholesky).

The compute path is ``libtt_gpu.so`` (hand-written sm_100a CUDA behind the C
ABI in ``include/tt_gpu.h``); this package is the host-side mirror of the
reference's kernel / harness interface used by the tests and the bench.
"""
from .kernels import (  # noqa: F401
    Context,
    DeviceError,
    GpuKernelRunner,
    KernelCase,
    MeasureProtocol,
    MeasurementError,
    NumericalError,
    aggregate_samples,
    apply_env_overrides,
    cholesky_factor_batch,
    cholesky_factor_inplace,
    cholesky_tiled,
    default_context,
    lu_factor_batch,
    lu_factor_inplace,
    lu_tiled,
    measure,
    mm3_tiled,
    unpack_lu,
)

__all__ = [
    "Context", "DeviceError", "GpuKernelRunner", "KernelCase", "MeasureProtocol",
    "MeasurementError", "NumericalError", "aggregate_samples", "apply_env_overrides",
    "cholesky_factor_batch", "cholesky_factor_inplace", "lu_factor_batch", "cholesky_tiled", "default_context", "lu_factor_inplace",
    "lu_tiled", "measure", "mm3_tiled", "unpack_lu",
]
