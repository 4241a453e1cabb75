#!/usr/bin/env python3
"""Structured 3mm config grid (regions near multiples of the 128x64 DMMA tile)."""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa

size = sys.argv[1] if len(sys.argv) > 1 else "extralarge"
dims = {"large": (800, 900, 1000, 1100, 1200), "extralarge": (1600, 1800, 2000, 2200, 2400)}[size]
n, l, m, o, p = dims
fl = 2.0 * (n * l * m + m * o * p + n * m * p)


def near(ext, cands):
    return [c for c in cands if ext % c == 0]


ys_n = near(n, [32, 40, 50, 64, 80, 100, 128, 160, 200, 256, 320, 400])
xs_m = near(m, [40, 50, 100, 125, 200, 250, 500])
xs_p = near(p, [60, 64, 80, 96, 100, 120, 128, 150, 160, 200, 240, 300, 400, 480])
ys_m = near(m, [40, 50, 80, 100, 125, 200, 250])
ctx = Context(0)
r = GpuKernelRunner(KernelCase("3mm", *dims), ctx)
proto = MeasureProtocol(1, 5, "median")
best = []
# sweep each product with the others at the hand-picked values
base = list((64, 125, 125, 120, 64, 120) if size == "extralarge" else (16, 125, 125, 120, 32, 120))
for idx, (ya, xa) in enumerate([(0, 1), (2, 3), (4, 5)]):
    ycands = ys_n if idx != 1 else ys_m
    xcands = xs_m if idx == 0 else xs_p
    res = []
    for y, x in itertools.product(ycands, xcands):
        cfg = list(base)
        cfg[ya], cfg[xa] = y, x
        s = r.measure(tuple(cfg), proto)
        res.append((s, y, x))
    res.sort()
    base[ya], base[xa] = res[0][1], res[0][2]
    print(json.dumps({"product": "EFG"[idx], "best": [res[0][1], res[0][2]], "ms": res[0][0] * 1e3,
                      "top5": [(round(s * 1e3, 4), y, x) for s, y, x in res[:5]]}), flush=True)
s = r.measure(tuple(base), MeasureProtocol(2, 9, "median"))
print(json.dumps({"size": size, "config": base, "ms": s * 1e3, "tflops": fl / s / 1e12,
                  "pct": 100 * fl / s / 1e12 / 37.05}))
