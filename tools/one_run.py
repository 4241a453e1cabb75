#!/usr/bin/env python3
"""Runs one schedule twice (first run captures the graph); for ncu launch lists."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kernel", default="lu")
ap.add_argument("--dims", default="2000")
ap.add_argument("--cfg", default="400,50")
ap.add_argument("--runs", type=int, default=2)
a = ap.parse_args()
dims = [int(x) for x in a.dims.split(",")] + [0] * 4
cfg = [int(x) for x in a.cfg.split(",")]
ctx = Context(0)
r = GpuKernelRunner(KernelCase(a.kernel, *dims[:5]), ctx)
for _ in range(a.runs):
    r.run(cfg, want_output=False)
print("launches", ctx.launches)
