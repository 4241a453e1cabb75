#!/usr/bin/env python3
"""Exhaustive knob sweeps on the GPU (LU / Cholesky spaces are 400/576 points).

Writes one JSON line per config to stdout: kernel, size, config, median
seconds (reference protocol 1 warm-up + median of 3, CUDA events), GFLOP/s.
Used to pick the fixed bench block and to see the tuning surface.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="lu")
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--min-bx", type=int, default=1)
    ap.add_argument("--max-seconds", type=float, default=240)
    args = ap.parse_args()
    ctx = Context(0)
    kase = KernelCase(args.kernel, args.n)
    r = GpuKernelRunner(kase, ctx)
    flops = (2 / 3 if args.kernel == "lu" else 1 / 3) * args.n ** 3
    t0 = time.time()
    best = None
    for bx in divisors(args.n):
        if bx < args.min_bx:
            continue
        for by in divisors(args.n):
            if time.time() - t0 > args.max_seconds:
                break
            s = r.measure((by, bx), MeasureProtocol(1, 3, "median"))
            rec = {"kernel": args.kernel, "n": args.n, "by": by, "bx": bx, "s": s,
                   "gflops": flops / s / 1e9}
            print(json.dumps(rec), flush=True)
            if best is None or s < best["s"]:
                best = rec
    print(json.dumps({"best": best}), flush=True)


if __name__ == "__main__":
    main()
