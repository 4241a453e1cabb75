"""ctypes binding of the host tuning runtime ``libtt_tuner.so`` (include/tt_tuner.h).

Mirrors the reference's space / tuner / run_tuning interface
(/root/reference/proj/core/include/tiletuner/space.hpp, tuners.hpp,
harness.hpp) with the batch extension the multi-GPU evaluator needs.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

from . import _lib

LIB_PATH = Path(__file__).resolve().parent / "libtt_tuner.so"
TUNERS = {"random": 0, "grid": 1, "genetic": 2, "boosted": 3, "bayesopt": 4}
KERNELS = {"lu": 0, "cholesky": 1, "3mm": 2, "mm3": 2}


class Record(ctypes.Structure):
    _fields_ = [("eval_index", ctypes.c_uint64), ("flat", ctypes.c_uint64),
                ("config", ctypes.c_int * 6), ("nconfig", ctypes.c_int), ("failed", ctypes.c_int),
                ("runtime_s", ctypes.c_double), ("elapsed_s", ctypes.c_double),
                ("best_so_far_s", ctypes.c_double), ("worker", ctypes.c_int),
                ("ask_s", ctypes.c_double), ("eval_s", ctypes.c_double)]


@dataclass
class EvalRecord:
    eval_index: int
    flat: int
    config: tuple
    runtime_s: float | None
    elapsed_s: float
    best_so_far_s: float
    worker: int
    ask_s: float = 0.0
    eval_s: float = 0.0


_lib_t = None


def load():
    global _lib_t
    if _lib_t is not None:
        return _lib_t
    _lib.load()  # libtt_gpu.so first (libtt_tuner links it)
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} missing: build with __graft_entry__.build()")
    L = ctypes.CDLL(str(LIB_PATH))
    u64, c_int, dbl, vp, cp = ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_char_p
    L.tt_space_divisors.argtypes = [c_int, vp, c_int]
    L.tt_space_size.argtypes = [c_int, cp, ctypes.POINTER(u64)]
    L.tt_space_config_at.argtypes = [c_int, cp, u64, vp]
    L.tt_space_index_of.argtypes = [c_int, cp, vp, c_int, ctypes.POINTER(u64)]
    L.tt_space_encode.argtypes = [c_int, cp, vp, c_int, vp]
    L.tt_space_synthetic.argtypes = [c_int, cp, vp, c_int, ctypes.POINTER(dbl)]
    L.tt_tuner_create.argtypes = [c_int, c_int, cp, u64, ctypes.POINTER(vp)]
    L.tt_tuner_ask_batch.argtypes = [vp, c_int, vp, ctypes.POINTER(c_int)]
    L.tt_tuner_tell.argtypes = [vp, u64, c_int, dbl]
    L.tt_tuner_destroy.argtypes = [vp]
    L.tt_tune_synthetic.argtypes = [c_int, c_int, cp, u64, c_int, dbl, c_int, vp, c_int,
                                    ctypes.POINTER(c_int), ctypes.POINTER(dbl)]
    L.tt_tune_measured.argtypes = [c_int, c_int, cp, u64, u64, c_int, dbl, vp, c_int, c_int, c_int,
                                   c_int, c_int, vp, c_int, ctypes.POINTER(c_int),
                                   ctypes.POINTER(dbl), ctypes.c_char_p, c_int]
    L.tt_tune_virtual.argtypes = [c_int, c_int, cp, u64, u64, c_int, dbl, c_int, c_int, c_int, c_int,
                                  c_int, c_int, vp, c_int, ctypes.POINTER(c_int),
                                  ctypes.POINTER(dbl), ctypes.c_char_p, c_int]
    _lib_t = L
    return L


def _ints(vals):
    arr = (ctypes.c_int * max(len(vals), 1))(*[int(v) for v in vals])
    return arr


def _nparams(kernel: str) -> int:
    return 6 if KERNELS[kernel] == 2 else 2


def divisor_candidates(n: int) -> list[int]:
    buf = (ctypes.c_int * 4096)()
    k = load().tt_space_divisors(n, ctypes.cast(buf, ctypes.c_void_p), 4096)
    if k < 0:
        raise ValueError("divisor_candidates: n must be >= 1")
    return list(buf[:k])


def space_size(kernel: str, size: str) -> int:
    out = ctypes.c_uint64()
    if load().tt_space_size(KERNELS[kernel], size.encode(), ctypes.byref(out)):
        raise ValueError(f"unregistered problem size: {kernel}/{size}")
    return out.value


def config_at(kernel: str, size: str, flat: int) -> tuple:
    buf = (ctypes.c_int * 6)()
    if load().tt_space_config_at(KERNELS[kernel], size.encode(), flat, ctypes.cast(buf, ctypes.c_void_p)):
        raise ValueError("config_at: flat index out of range")
    return tuple(buf[:_nparams(kernel)])


def index_of(kernel: str, size: str, cfg) -> int:
    out = ctypes.c_uint64()
    if load().tt_space_index_of(KERNELS[kernel], size.encode(), ctypes.cast(_ints(cfg), ctypes.c_void_p),
                                len(cfg), ctypes.byref(out)):
        raise ValueError("index_of: configuration not in space")
    return out.value


def encode(kernel: str, size: str, cfg) -> list[float]:
    buf = (ctypes.c_double * 6)()
    if load().tt_space_encode(KERNELS[kernel], size.encode(), ctypes.cast(_ints(cfg), ctypes.c_void_p),
                              len(cfg), ctypes.cast(buf, ctypes.c_void_p)):
        raise ValueError("encode: configuration not in space")
    return list(buf[:len(cfg)])


def synthetic_objective(kernel: str, size: str, cfg) -> float:
    out = ctypes.c_double()
    if load().tt_space_synthetic(KERNELS[kernel], size.encode(),
                                 ctypes.cast(_ints(cfg), ctypes.c_void_p), len(cfg), ctypes.byref(out)):
        raise ValueError("synthetic_objective: configuration not in space")
    return out.value


class Tuner:
    """Ask/tell handle with the batch extension (tuners.hpp:51-61 + ask_batch)."""

    def __init__(self, tuner: str, kernel: str, size: str, seed: int):
        h = ctypes.c_void_p()
        rc = load().tt_tuner_create(TUNERS[tuner], KERNELS[kernel], size.encode(), seed, ctypes.byref(h))
        if rc:
            raise ValueError(f"cannot create tuner {tuner} for {kernel}/{size}")
        self.h, self.kernel, self.size = h, kernel, size

    def ask_batch(self, k: int) -> list[int]:
        buf = (ctypes.c_uint64 * max(k, 1))()
        got = ctypes.c_int()
        if load().tt_tuner_ask_batch(self.h, k, ctypes.cast(buf, ctypes.c_void_p), ctypes.byref(got)):
            raise ValueError("ask_batch failed")
        return list(buf[:got.value])

    def ask(self) -> int:
        got = self.ask_batch(1)
        if not got:
            raise StopIteration("search space exhausted")
        return got[0]

    def tell(self, flat: int, runtime_s: float | None):
        rc = load().tt_tuner_tell(self.h, flat, 1 if runtime_s is None else 0,
                                  0.0 if runtime_s is None else float(runtime_s))
        if rc:
            raise ValueError("tell(): configuration was not asked")

    def __del__(self):  # pragma: no cover
        try:
            load().tt_tuner_destroy(self.h)
        except Exception:
            pass


def _records(buf, n) -> list[EvalRecord]:
    out = []
    for i in range(n):
        r = buf[i]
        out.append(EvalRecord(r.eval_index, r.flat, tuple(r.config[:r.nconfig]),
                              None if r.failed else r.runtime_s, r.elapsed_s, r.best_so_far_s,
                              r.worker, r.ask_s, r.eval_s))
    return out


def run_tuning_synthetic(tuner: str, kernel: str, size: str, seed: int, max_evals: int,
                         max_seconds: float | None = None, workers: int = 1):
    buf = (Record * max_evals)()
    n = ctypes.c_int()
    tot = ctypes.c_double()
    rc = load().tt_tune_synthetic(TUNERS[tuner], KERNELS[kernel], size.encode(), seed, max_evals,
                                  max_seconds or 0.0, workers, ctypes.cast(buf, ctypes.c_void_p),
                                  max_evals, ctypes.byref(n), ctypes.byref(tot))
    if rc:
        raise ValueError(f"run_tuning failed ({rc})")
    return _records(buf, n.value), tot.value


def run_tuning_measured(tuner: str, kernel: str, size: str, seed: int, max_evals: int,
                        devices=(0,), max_seconds: float | None = None, warmups: int = 1,
                        reps: int = 3, aggregate: str = "median", spot_check: bool = True,
                        input_seed: int = 1):
    """The GPU objective: one worker thread + tt_ctx per entry of `devices`."""
    buf = (Record * max_evals)()
    n = ctypes.c_int()
    tot = ctypes.c_double()
    err = ctypes.create_string_buffer(512)
    devs = _ints(devices)
    rc = load().tt_tune_measured(TUNERS[tuner], KERNELS[kernel], size.encode(), seed, input_seed,
                                 max_evals, max_seconds or 0.0, ctypes.cast(devs, ctypes.c_void_p),
                                 len(devices), warmups, reps, _lib.AGGREGATES[aggregate],
                                 1 if spot_check else 0, ctypes.cast(buf, ctypes.c_void_p),
                                 max_evals, ctypes.byref(n), ctypes.byref(tot), err, 512)
    if rc:
        raise TuningError(f"run_tuning (measured) failed ({rc}): {err.value.decode()}",
                          _records(buf, n.value))
    return _records(buf, n.value), tot.value


class TuningError(RuntimeError):
    """MeasurementError during a measured run; `records` holds the flushed partial trace
    (harness.cpp:252-256)."""

    def __init__(self, msg: str, records):
        super().__init__(msg)
        self.records = records


def run_tuning_virtual(tuner: str, kernel: str, size: str, seed: int, max_evals: int,
                       workers: int, device: int = 0, max_seconds: float | None = None,
                       warmups: int = 1, reps: int = 3, aggregate: str = "median",
                       spot_check: bool = True, input_seed: int = 1):
    """T1/T8 harness: `workers` evaluators emulated on one real device (virtual clock;
    every evaluation measured for real, host ask time charged serially)."""
    buf = (Record * max_evals)()
    n = ctypes.c_int()
    tot = ctypes.c_double()
    err = ctypes.create_string_buffer(512)
    rc = load().tt_tune_virtual(TUNERS[tuner], KERNELS[kernel], size.encode(), seed, input_seed,
                                max_evals, max_seconds or 0.0, device, workers, warmups, reps,
                                _lib.AGGREGATES[aggregate], 1 if spot_check else 0,
                                ctypes.cast(buf, ctypes.c_void_p), max_evals, ctypes.byref(n),
                                ctypes.byref(tot), err, 512)
    if rc:
        raise TuningError(f"run_tuning (virtual) failed ({rc}): {err.value.decode()}",
                          _records(buf, n.value))
    return _records(buf, n.value), tot.value


def time_to_reach(records, best_runtime: float, best_flat: int | None = None) -> float:
    """elapsed_s of the first record with runtime <= best_runtime or that
    evaluates the same configuration (best_flat)."""
    for r in records:
        if (r.runtime_s is not None and r.runtime_s <= best_runtime) or \
                (best_flat is not None and r.flat == best_flat):
            return r.elapsed_s
    return float("inf")


def best_record(records):
    """First record achieving the run's final best (its time is T1 for a 1-GPU run)."""
    ok = [r for r in records if r.runtime_s is not None]
    best = min(r.runtime_s for r in ok)
    return next(r for r in ok if r.runtime_s == best)


def time_to_best(records, target: float | None = None) -> float:
    """elapsed_s of the first record reaching `target` (default: the run's final best)."""
    best = min(r.runtime_s for r in records if r.runtime_s is not None) if target is None else target
    for r in records:
        if r.runtime_s is not None and r.runtime_s <= best:
            return r.elapsed_s
    return float("inf")
