"""Reference-shaped Python API over the sm_100a kernels (host side of the boundary).

Mirrors ``/root/reference/proj/core/include/tiletuner/kernels.hpp`` and
``harness.hpp``: same names, argument meaning and error behaviour, with
``ValueError`` standing in for ``std::invalid_argument``.  Every call goes
through the C ABI of ``libtt_gpu.so``; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import TT_EDEVICE, TT_EINVAL, TT_ENOMEM, TT_ENUMERIC, TT_OK


class NumericalError(RuntimeError):
    """errors.hpp:15-18 — vanishing LU pivot / non-positive Cholesky diagonal."""

    def __init__(self, msg: str, index: int | None = None):
        super().__init__(msg)
        self.index = index


class MeasurementError(RuntimeError):
    """errors.hpp:44-47 — device/timer failure or failed spot check."""


class DeviceError(MeasurementError):
    """No usable CUDA device (the product path never falls back to the CPU)."""


def _raise(ctx, rc: int, index: int | None = None):
    if rc == TT_OK:
        return
    lib = _lib.load()
    msg = lib.tt_last_error(ctx).decode() if ctx else "no context"
    if rc == TT_EINVAL:
        raise ValueError(msg)
    if rc == TT_ENUMERIC:
        raise NumericalError(msg, index)
    if rc == TT_ENOMEM:
        raise MemoryError(msg)
    if rc == TT_EDEVICE:
        raise DeviceError(msg)
    raise RuntimeError(f"tt_gpu status {rc}: {msg}")


class Context:
    """One ``tt_ctx``: a GPU, its streams and its instantiation cache."""

    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = ctypes.c_void_p()
        rc = lib.tt_ctx_create(int(device), ctypes.byref(h))
        if rc == TT_EDEVICE:
            raise DeviceError("tt_ctx_create: no CUDA device visible (no CPU fallback)")
        if rc != TT_OK:
            raise RuntimeError(f"tt_ctx_create failed with status {rc}")
        self.handle = h
        self.device = device
        self.lib = lib

    def close(self):
        if self.handle:
            self.lib.tt_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order varies
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.lib.tt_launch_count(self.handle))

    @property
    def cache_size(self) -> int:
        return int(self.lib.tt_cache_size(self.handle))

    def check(self, rc: int, index: int | None = None):
        _raise(self.handle, rc, index)


_default: dict[int, Context] = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        ctx = _default.get(device)
        if ctx is None:
            ctx = _default[device] = Context(device)
        return ctx


def _as_matrix(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.float64 or a.ndim != 2 or not a.flags.c_contiguous:
        raise ValueError("expected a C-contiguous 2-D float64 matrix (tiletuner::Matrix layout)")
    return a


def lu_factor_inplace(a: np.ndarray, by: int, bx: int, ctx: Context | None = None) -> None:
    """kernels.hpp:65 — packed in-place LU without pivoting (L strictly below, U on/above)."""
    a = _as_matrix(a)
    ctx = ctx or default_context()
    idx = ctypes.c_int(-1)
    rc = ctx.lib.tt_lu_factor_inplace(ctx.handle, _lib.ptr(a), a.shape[0], a.shape[1],
                                      int(by), int(bx), ctypes.byref(idx))
    ctx.check(rc, idx.value)


def cholesky_factor_inplace(a: np.ndarray, by: int, bx: int, ctx: Context | None = None) -> None:
    """kernels.hpp:66 — L in the lower triangle; the upper triangle is never written."""
    a = _as_matrix(a)
    ctx = ctx or default_context()
    idx = ctypes.c_int(-1)
    rc = ctx.lib.tt_cholesky_factor_inplace(ctx.handle, _lib.ptr(a), a.shape[0], a.shape[1],
                                            int(by), int(bx), ctypes.byref(idx))
    ctx.check(rc, idx.value)


def _factor_batch(fn, mats, by, bx, ctx):
    mats = [_as_matrix(m) for m in mats]
    if not mats:
        return
    n = mats[0].shape[0]
    if any(m.shape != (n, n) for m in mats):
        raise ValueError("batch: all matrices must be square with the same extent")
    ptrs = (ctypes.c_void_p * len(mats))(*[m.ctypes.data for m in mats])
    fails = (ctypes.c_int * len(mats))()
    rc = fn(ctx.handle, ptrs, len(mats), n, int(by), int(bx), fails)
    first = next((f for f in fails if f >= 0), -1) if rc else None
    ctx.check(rc, first)


def lu_factor_batch(mats, by: int, bx: int, ctx: Context | None = None) -> None:
    """Pipelined batch of lu_factor_inplace (kernels.hpp:65) over host matrices: the
    upload / factorisation / download of neighbouring matrices overlap.  Page-locked
    host buffers (torch pin_memory) give full overlap."""
    ctx = ctx or default_context()
    _factor_batch(ctx.lib.tt_lu_factor_batch, mats, by, bx, ctx)


def cholesky_factor_batch(mats, by: int, bx: int, ctx: Context | None = None) -> None:
    """Pipelined batch of cholesky_factor_inplace (kernels.hpp:66)."""
    ctx = ctx or default_context()
    _factor_batch(ctx.lib.tt_cholesky_factor_batch, mats, by, bx, ctx)


def mm3_tiled(a, b, c, d, config, ctx: Context | None = None) -> np.ndarray:
    """kernels.hpp:43 — G = (A*B)*(C*D) with per-product CTA regions (P0..P5)."""
    a, b, c, d = (_as_matrix(x) for x in (a, b, c, d))
    if a.shape[1] != b.shape[0] or c.shape[1] != d.shape[0] or b.shape[1] != c.shape[0]:
        raise ValueError("matmul: inner dimensions disagree")
    ctx = ctx or default_context()
    cfg = list(config)
    g = np.empty((a.shape[0], d.shape[1]), dtype=np.float64)
    rc = ctx.lib.tt_mm3_tiled(ctx.handle, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), _lib.ptr(d),
                              a.shape[0], a.shape[1], b.shape[1], c.shape[1], d.shape[1],
                              _lib.int_array(cfg), len(cfg), _lib.ptr(g))
    ctx.check(rc)
    return g


def unpack_lu(packed: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """kernels.cpp:158-167 — exact unit diagonal and exact zeros."""
    lower = np.tril(packed, -1)
    np.fill_diagonal(lower, 1.0)
    return lower, np.triu(packed)


def lu_tiled(a, by: int, bx: int, ctx: Context | None = None):
    """kernels.hpp:52 — copy, factor, unpack into (L, U)."""
    work = np.array(a, dtype=np.float64, copy=True, order="C")
    lu_factor_inplace(work, by, bx, ctx)
    return unpack_lu(work)


def cholesky_tiled(a, by: int, bx: int, ctx: Context | None = None) -> np.ndarray:
    """kernels.hpp:60 — copy, factor, keep the lower triangle (lower_of, kernels.cpp:246-253)."""
    work = np.array(a, dtype=np.float64, copy=True, order="C")
    cholesky_factor_inplace(work, by, bx, ctx)
    return np.tril(work)


# ---------------------------------------------------------------- harness twin

@dataclass
class MeasureProtocol:
    """harness.hpp:32-38 (defaults 1 warm-up, 3 repetitions, median)."""
    warmups: int = 1
    repetitions: int = 3
    aggregate: str = "median"


def apply_env_overrides(protocol: MeasureProtocol) -> MeasureProtocol:
    """harness.cpp:42-51 — TILETUNER_REPS overrides repetitions when a positive integer."""
    import os
    import re
    raw = os.environ.get("TILETUNER_REPS")
    # strtol(raw, &end, 10) accepted iff it consumed everything: leading
    # whitespace and a sign are allowed, trailing characters are not.
    if raw is not None and re.fullmatch(r"[ \t\n\r\f\v]*[+-]?[0-9]+", raw):
        v = int(raw.strip())
        if v >= 1:
            return MeasureProtocol(protocol.warmups, v, protocol.aggregate)
    return protocol


def aggregate_samples(samples, how: str = "median") -> float:
    """harness.cpp:53-71."""
    s = list(samples)
    if not s:
        raise ValueError("aggregate_samples: empty sample set")
    if how == "min":
        return min(s)
    if how == "mean":
        return _mean(s)
    if how != "median":
        raise ValueError(f"unknown aggregate: {how}")
    s.sort()
    n = len(s)
    return s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])


def _mean(s) -> float:
    acc = 0.0
    for v in s:  # std::accumulate order
        acc += v
    return acc / len(s)


@dataclass
class KernelCase:
    """kernels.hpp:11-14: a problem size + the input seed (kInputSeed = 1)."""
    kernel: str
    n: int
    l: int = 0
    m: int = 0
    o: int = 0
    p: int = 0
    seed: int = 1
    size_name: str = field(default="custom")

    @property
    def dims(self):
        return (self.n, self.l, self.m, self.o, self.p)


class GpuKernelRunner:
    """The device twin of KernelRunner (harness.cpp:89-143).

    The case's inputs are generated once (bitwise gen_spd / gen_3mm_inputs on
    the device) and kept resident; every sample runs the schedule on a fresh
    device copy, timed with CUDA events on the context stream.
    """

    def __init__(self, kase: KernelCase, ctx: Context | None = None, inputs=None):
        self.kase = kase
        self.ctx = ctx or default_context()
        kid = _lib.KERNEL_IDS[kase.kernel]
        lib = self.ctx.lib
        if inputs is None:
            rc = lib.tt_setup_seeded(self.ctx.handle, kid, *kase.dims, int(kase.seed))
        else:
            mats = [_as_matrix(x) for x in inputs] + [None] * (4 - len(inputs))
            rc = lib.tt_setup_host(self.ctx.handle, kid, *kase.dims, *(_lib.ptr(m) for m in mats))
        self.ctx.check(rc)
        self.kernel_id = kid

    def measure(self, config, protocol: MeasureProtocol = MeasureProtocol()) -> float:
        cfg = list(config)
        out = ctypes.c_double(0.0)
        rc = self.ctx.lib.tt_measure(self.ctx.handle, _lib.int_array(cfg), len(cfg),
                                     int(protocol.warmups), int(protocol.repetitions),
                                     _lib.AGGREGATES[protocol.aggregate], ctypes.byref(out))
        self.ctx.check(rc)
        return out.value

    def samples(self, config, warmups: int, reps: int) -> list[float]:
        cfg = list(config)
        buf = np.zeros(max(reps, 1), dtype=np.float64)
        rc = self.ctx.lib.tt_measure_samples(self.ctx.handle, _lib.int_array(cfg), len(cfg),
                                             int(warmups), int(reps), _lib.ptr(buf))
        self.ctx.check(rc)
        return buf[:reps].tolist()

    def run(self, config, want_output: bool = True):
        cfg = list(config)
        n, l, m, o, p = self.kase.dims
        out = None
        if want_output:
            shape = (n, p) if self.kase.kernel in ("3mm", "mm3") else (n, n)
            out = np.empty(shape, dtype=np.float64)
        idx = ctypes.c_int(-1)
        rc = self.ctx.lib.tt_run(self.ctx.handle, _lib.int_array(cfg), len(cfg), _lib.ptr(out),
                                 ctypes.byref(idx))
        self.ctx.check(rc, idx.value)
        return out

    def residual(self, ref_g: np.ndarray | None = None) -> float:
        out = ctypes.c_double(0.0)
        rc = self.ctx.lib.tt_residual(self.ctx.handle, _lib.ptr(ref_g), ctypes.byref(out))
        self.ctx.check(rc)
        return out.value

    def inputs(self):
        n, l, m, o, p = self.kase.dims
        if self.kase.kernel in ("3mm", "mm3"):
            mats = [np.empty(s) for s in ((n, l), (l, m), (m, o), (o, p))]
        else:
            mats = [np.empty((n, n))]
        ptrs = [_lib.ptr(x) for x in mats] + [None] * (4 - len(mats))
        self.ctx.check(self.ctx.lib.tt_get_input(self.ctx.handle, *ptrs))
        return mats


def measure(kase: KernelCase, config, protocol: MeasureProtocol = MeasureProtocol(),
            ctx: Context | None = None) -> float:
    """harness.cpp:160-164 — fresh runner per call."""
    return GpuKernelRunner(kase, ctx).measure(config, protocol)
