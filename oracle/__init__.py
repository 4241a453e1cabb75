"""TEST INFRASTRUCTURE ONLY — CPU oracle for the hot path.

Python loader for ``oracle/liboracle.so`` (the plain-C restatement in
tt_oracle.c) and, when present, ``oracle/_ref/libtiletuner_ref.so`` (the
unmodified reference core compiled from /root/reference by oracle/Makefile).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module, and only as the checker / the timed CPU baseline.  The product
package (paper_2309_07235_b200) never imports it.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libtiletuner_ref.so"

_vp = ctypes.c_void_p
_orc = None
_ref = None


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


def lib():
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = ctypes.CDLL(str(ORACLE_SO))
        c_int, u64, dbl = ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        L.orc_gen_spd.argtypes = [c_int, u64, _vp]
        L.orc_gen_3mm.argtypes = [c_int] * 5 + [u64] + [_vp] * 4
        L.orc_mm3_reference.argtypes = [_vp] * 4 + [c_int] * 5 + [_vp]
        L.orc_mm3_tiled.argtypes = [_vp] * 4 + [c_int] * 5 + [_vp, c_int, _vp]
        L.orc_lu_factor_inplace.argtypes = [_vp, c_int, c_int, c_int, _vp]
        L.orc_cholesky_factor_inplace.argtypes = [_vp, c_int, c_int, c_int, _vp]
        L.orc_lu_residual_packed.argtypes = [_vp, _vp, c_int]
        L.orc_lu_residual_packed.restype = dbl
        L.orc_cholesky_residual.argtypes = [_vp, _vp, c_int]
        L.orc_cholesky_residual.restype = dbl
        L.orc_mm3_residual.argtypes = [_vp, _vp, ctypes.c_int64]
        L.orc_mm3_residual.restype = dbl
        _orc = L
    return _orc


def ref_lib():
    """The unmodified reference (None when it was not built in this container)."""
    global _ref
    if _ref is None and REF_SO.exists():
        R = ctypes.CDLL(str(REF_SO))
        c_int, u64, dbl = ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        R.ref_last_error.restype = ctypes.c_char_p
        R.ref_gen_spd.argtypes = [c_int, u64, _vp]
        R.ref_gen_3mm.argtypes = [c_int] * 5 + [u64] + [_vp] * 4
        R.ref_mm3_reference.argtypes = [_vp] * 4 + [c_int] * 5 + [_vp]
        R.ref_mm3_tiled.argtypes = [_vp] * 4 + [c_int] * 5 + [_vp, c_int, _vp]
        R.ref_lu_factor_inplace.argtypes = [_vp, c_int, c_int, c_int, c_int]
        R.ref_cholesky_factor_inplace.argtypes = [_vp, c_int, c_int, c_int, c_int]
        R.ref_lu_reference_packed.argtypes = [_vp, c_int, _vp]
        R.ref_cholesky_reference.argtypes = [_vp, c_int, _vp]
        R.ref_lu_residual_packed.argtypes = [_vp, _vp, c_int, ctypes.POINTER(dbl)]
        R.ref_cholesky_residual.argtypes = [_vp, _vp, c_int, ctypes.POINTER(dbl)]
        R.ref_residual_for.argtypes = [c_int, ctypes.c_char_p, u64, _vp, c_int, ctypes.POINTER(dbl)]
        R.ref_measure.argtypes = [c_int, ctypes.c_char_p, u64, _vp, c_int, c_int, c_int, c_int,
                                  ctypes.POINTER(dbl)]
        R.ref_aggregate_samples.argtypes = [_vp, c_int, c_int, ctypes.POINTER(dbl)]
        R.ref_divisor_candidates.argtypes = [c_int, _vp, c_int]
        R.ref_space_size.argtypes = [c_int, ctypes.c_char_p, ctypes.POINTER(u64)]
        R.ref_config_at.argtypes = [c_int, ctypes.c_char_p, u64, _vp]
        R.ref_index_of.argtypes = [c_int, ctypes.c_char_p, _vp, c_int, ctypes.POINTER(u64)]
        R.ref_encode.argtypes = [c_int, ctypes.c_char_p, _vp, c_int, _vp]
        R.ref_run_tuning_synthetic.argtypes = [c_int, ctypes.c_char_p, c_int, u64, c_int, _vp,
                                               _vp, ctypes.POINTER(c_int)]
        _ref = R
    return _ref


# ---- oracle (plain-C restatement) ------------------------------------------------

def gen_spd(n: int, seed: int) -> np.ndarray:
    a = np.empty((n, n))
    if lib().orc_gen_spd(n, seed, _p(a)) != 0:
        raise ValueError("gen_spd: n must be >= 1")
    return a


def gen_3mm(dims, seed: int):
    n, l, m, o, p = dims
    mats = [np.empty(s) for s in ((n, l), (l, m), (m, o), (o, p))]
    if lib().orc_gen_3mm(n, l, m, o, p, seed, *(_p(x) for x in mats)) != 0:
        raise ValueError("gen_3mm_inputs: all five extents must be >= 1")
    return mats


def mm3_reference(a, b, c, d) -> np.ndarray:
    g = np.empty((a.shape[0], d.shape[1]))
    lib().orc_mm3_reference(_p(a), _p(b), _p(c), _p(d), a.shape[0], a.shape[1], b.shape[1],
                            c.shape[1], d.shape[1], _p(g))
    return g


def mm3_tiled(a, b, c, d, cfg) -> np.ndarray:
    g = np.empty((a.shape[0], d.shape[1]))
    arr = (ctypes.c_int * max(len(cfg), 1))(*cfg)
    rc = lib().orc_mm3_tiled(_p(a), _p(b), _p(c), _p(d), a.shape[0], a.shape[1], b.shape[1],
                             c.shape[1], d.shape[1], ctypes.cast(arr, _vp), len(cfg), _p(g))
    if rc == 1:
        raise ValueError("mm3_tiled: invalid configuration")
    return g


class OracleNumericalError(RuntimeError):
    pass


def lu_factor_inplace(a: np.ndarray, by: int, bx: int) -> None:
    idx = ctypes.c_int(-1)
    rc = lib().orc_lu_factor_inplace(_p(a), a.shape[0], by, bx, ctypes.cast(ctypes.pointer(idx), _vp))
    if rc == 1:
        raise ValueError("lu_tiled: invalid factor")
    if rc == 2:
        raise OracleNumericalError(f"lu: vanishing pivot at column {idx.value}")


def cholesky_factor_inplace(a: np.ndarray, by: int, bx: int) -> None:
    idx = ctypes.c_int(-1)
    rc = lib().orc_cholesky_factor_inplace(_p(a), a.shape[0], by, bx,
                                           ctypes.cast(ctypes.pointer(idx), _vp))
    if rc == 1:
        raise ValueError("cholesky_tiled: invalid factor")
    if rc == 2:
        raise OracleNumericalError(f"cholesky: non-positive diagonal at row {idx.value}")


def lu_residual_packed(a, packed) -> float:
    return lib().orc_lu_residual_packed(_p(a), _p(packed), a.shape[0])


def cholesky_residual(a, fac) -> float:
    return lib().orc_cholesky_residual(_p(a), _p(fac), a.shape[0])


def mm3_residual(ref, out) -> float:
    return lib().orc_mm3_residual(_p(ref), _p(out), ref.size)
