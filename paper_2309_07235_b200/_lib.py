"""ctypes binding of the in-tree C-ABI library ``libtt_gpu.so`` (include/tt_gpu.h).

The product path is the CUDA library; there is no CPU fallback.  Loading
fails loudly when the library has not been built, and every compute call
fails with ``DeviceError`` when no CUDA device is present.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libtt_gpu.so"

TT_OK, TT_EINVAL, TT_ENUMERIC, TT_EDEVICE, TT_ENOMEM = 0, 1, 2, 3, 4
KERNEL_IDS = {"lu": 0, "cholesky": 1, "3mm": 2, "mm3": 2}
AGGREGATES = {"median": 0, "min": 1, "mean": 2}

# The exported surface; tests/test_abi.py checks it against include/tt_gpu.h.
EXPORTS = (
    "tt_ctx_create", "tt_ctx_destroy", "tt_last_error", "tt_ctx_device", "tt_cache_size",
    "tt_lu_factor_inplace", "tt_cholesky_factor_inplace", "tt_mm3_tiled",
    "tt_setup_host", "tt_setup_seeded", "tt_run", "tt_measure", "tt_measure_samples",
    "tt_get_input", "tt_residual", "tt_dev_lu", "tt_dev_cholesky", "tt_dev_mm3",
    "tt_dev_gemm", "tt_dev_fill_uniform", "tt_launch_count", "tt_build_info", "tt_dag_tasks",
    "tt_dag_trace", "tt_dag_urgent", "tt_dag_chunk_depth", "tt_dag_tile", "tt_dag_region_rows",
    "tt_lu_factor_batch", "tt_cholesky_factor_batch", "tt_gemm_plan",
)

_lib = None


def load() -> ctypes.CDLL:
    """Load libtt_gpu.so (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("TT_GPU_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise ImportError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(path)
    c_int, c_int_p, c_dbl_p = ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_void_p
    vp = ctypes.c_void_p
    sig = {
        "tt_ctx_create": (c_int, [c_int, ctypes.POINTER(vp)]),
        "tt_ctx_destroy": (c_int, [vp]),
        "tt_last_error": (ctypes.c_char_p, [vp]),
        "tt_ctx_device": (c_int, [vp]),
        "tt_cache_size": (c_int, [vp]),
        "tt_lu_factor_inplace": (c_int, [vp, c_dbl_p, c_int, c_int, c_int, c_int, c_int_p]),
        "tt_cholesky_factor_inplace": (c_int, [vp, c_dbl_p, c_int, c_int, c_int, c_int, c_int_p]),
        "tt_mm3_tiled": (c_int, [vp] + [c_dbl_p] * 4 + [c_int] * 5 + [c_int_p, c_int, c_dbl_p]),
        "tt_setup_host": (c_int, [vp, c_int] + [c_int] * 5 + [c_dbl_p] * 4),
        "tt_setup_seeded": (c_int, [vp, c_int] + [c_int] * 5 + [ctypes.c_uint64]),
        "tt_run": (c_int, [vp, c_int_p, c_int, c_dbl_p, c_int_p]),
        "tt_measure": (c_int, [vp, c_int_p, c_int, c_int, c_int, c_int,
                               ctypes.POINTER(ctypes.c_double)]),
        "tt_measure_samples": (c_int, [vp, c_int_p, c_int, c_int, c_int, c_dbl_p]),
        "tt_get_input": (c_int, [vp] + [c_dbl_p] * 4),
        "tt_residual": (c_int, [vp, c_dbl_p, ctypes.POINTER(ctypes.c_double)]),
        "tt_dev_lu": (c_int, [vp, vp, c_int, c_int, c_int, c_int, c_int_p, vp]),
        "tt_dev_cholesky": (c_int, [vp, vp, c_int, c_int, c_int, c_int, c_int_p, vp]),
        "tt_dev_mm3": (c_int, [vp] + [vp, c_int] * 7 + [c_int] * 5 + [c_int_p, c_int, vp]),
        "tt_dev_gemm": (c_int, [vp, vp, c_int, vp, c_int, c_int, vp, c_int] + [c_int] * 7 + [vp]),
        "tt_dev_fill_uniform": (c_int, [vp, vp, c_int, c_int, c_int, ctypes.c_longlong,
                                        ctypes.c_uint64, c_int, vp]),
        "tt_launch_count": (ctypes.c_uint64, [vp]),
        "tt_build_info": (ctypes.c_char_p, []),
        "tt_dag_tasks": (c_int, [c_int, c_int, c_int, c_int, c_int_p, c_int]),
        "tt_dag_trace": (c_int, [vp, vp, c_int]),
        "tt_dag_urgent": (c_int, [c_int, c_int, c_int, c_int]),
        "tt_dag_chunk_depth": (c_int, [c_int, c_int, c_int]),
        "tt_dag_tile": (c_int, [c_int, c_int, c_int]),
        "tt_dag_region_rows": (c_int, [c_int, c_int, c_int]),
        "tt_gemm_plan": (c_int, [c_int, c_int, c_int, c_int, ctypes.c_void_p]),
        "tt_lu_factor_batch": (c_int, [vp, vp, c_int, c_int, c_int, c_int, c_int_p]),
        "tt_cholesky_factor_batch": (c_int, [vp, vp, c_int, c_int, c_int, c_int, c_int_p]),
    }
    ab = "TT_GPU_LIB" in os.environ  # A/B against another build: tolerate older exports
    for name, (res, args) in sig.items():
        if ab and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.c_void_p)


def int_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_int * max(len(vals), 1))(*vals)


def dag_tasks(kernel: str, n: int, by: int, bx: int) -> np.ndarray | None:
    """Task list of the persistent tile-DAG schedule as an (ntasks, 4) int array
    {kind | j << 2, k0 | q << 16, r0, r1} (a GEMM applies panel steps [k0, k0+q)),
    or None when (n, by, bx) uses the graph schedule."""
    lib = load()
    kid = KERNEL_IDS[kernel]
    cnt = lib.tt_dag_tasks(kid, n, by, bx, None, 0)
    if cnt < 0:
        return None
    out = np.zeros((cnt, 4), dtype=np.int32)
    lib.tt_dag_tasks(kid, n, by, bx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), cnt)
    return out


def dag_tile(n: int, by: int, bx: int) -> int | None:
    """Tile T the persistent schedule runs for (n, by, bx), None on the graph schedule."""
    t = load().tt_dag_tile(n, by, bx)
    return None if t < 0 else int(t)


def gemm_plan(m: int, n: int, fy: int, fx: int) -> dict:
    """CTA region and tile variant a 3mm knob region (fy, fx) maps to (tt_gemm_plan)."""
    out = (ctypes.c_int * 5)()
    if load().tt_gemm_plan(m, n, fy, fx, ctypes.cast(out, ctypes.c_void_p)):
        raise ValueError("gemm_plan: invalid arguments")
    return {"reg_y": out[0], "reg_x": out[1], "bm": out[2], "bn": out[3], "warps": out[4]}


def dag_region_rows(n: int, by: int, bx: int) -> int | None:
    """Row extent of the persistent schedule's update / solve tasks (by packed to >= 128)."""
    r = load().tt_dag_region_rows(n, by, bx)
    return None if r < 0 else int(r)


def dag_chunk_depth(n: int, by: int, bx: int) -> int | None:
    """Chunk depth d of the persistent schedule for (n, by, bx), None on the graph schedule."""
    d = load().tt_dag_chunk_depth(n, by, bx)
    return None if d < 0 else int(d)
