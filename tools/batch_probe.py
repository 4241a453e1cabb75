#!/usr/bin/env python3
"""Marginal per-matrix time of the pipelined batch entry (tt_lu_factor_batch)
against the kernel alone: how much of the host<->device traffic it hides."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402  (input generator for the host copies only)
from paper_2309_07235_b200 import Context, _lib  # noqa: E402

n, by, bx = 2000, 200, 40
ctx = Context(0)
lib = ctx.lib
a = oracle.gen_spd(n, 1)
host = [torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy() for _ in range(40)]
for h in host:
    h[...] = a


def run(cnt):
    for h in host[:cnt]:
        h[...] = a
    ptrs = (ctypes.c_void_p * cnt)(*[h.ctypes.data for h in host[:cnt]])
    fails = (ctypes.c_int * cnt)()
    t0 = time.perf_counter()
    ctx.check(lib.tt_lu_factor_batch(ctx.handle, ptrs, cnt, n, by, bx, fails))
    return time.perf_counter() - t0


run(40)
for cnt in (1, 2, 5, 10, 20, 40):
    ts = sorted(run(cnt) for _ in range(3))
    print(f"batch {cnt:3d}: {ts[0] * 1e3:8.2f} ms  ({ts[0] / cnt * 1e3:.3f} ms per matrix)")
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
hp = host[0]
s = torch.cuda.Stream()
for name, fn in (("H2D 32 MB", lambda: d.copy_(torch.from_numpy(hp), non_blocking=True)),
                 ("D2H 32 MB", lambda: torch.from_numpy(hp).copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
