#!/usr/bin/env python3
"""Random sweep of 3mm tile configs (divisor knobs, regions >= 16) at a size;
prints the top configs by median time (reference protocol, CUDA events)."""
import argparse
import json
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa

SIZES = {"large": (800, 900, 1000, 1100, 1200), "extralarge": (1600, 1800, 2000, 2200, 2400)}


def divisors(n, lo=16):
    return [d for d in range(lo, n + 1) if n % d == 0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="large")
    ap.add_argument("--samples", type=int, default=400)
    ap.add_argument("--max-seconds", type=float, default=120)
    a = ap.parse_args()
    n, l, m, o, p = SIZES[a.size]
    ctx = Context(0)
    r = GpuKernelRunner(KernelCase("3mm", n, l, m, o, p), ctx)
    fl = 2.0 * (n * l * m + m * o * p + n * m * p)
    proto = MeasureProtocol(1, 5, "median")
    rng = random.Random(1)
    axes = [divisors(n), divisors(m), divisors(m), divisors(p), divisors(n), divisors(p)]
    res, t0 = [], time.time()
    for _ in range(a.samples):
        cfg = tuple(rng.choice(ax) for ax in axes)
        s = r.measure(cfg, proto)
        res.append((s, cfg))
        if time.time() - t0 > a.max_seconds:
            break
    res.sort()
    for s, cfg in res[:10]:
        print(json.dumps({"size": a.size, "config": cfg, "ms": s * 1e3, "tflops": fl / s / 1e12,
                          "pct": 100 * fl / s / 1e12 / 37.05}))
    print(json.dumps({"evaluated": len(res)}))


if __name__ == "__main__":
    main()
