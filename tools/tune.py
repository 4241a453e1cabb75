#!/usr/bin/env python3
"""Measured BO tuning run on the GPU(s) through the host runtime (libtt_tuner).

    python tools/tune.py --kernel 3mm --size extralarge --evals 200 --devices 0
Prints one JSON line: best config, its runtime / GFLOP/s / % of fp64 peak,
time-to-best (elapsed_s of the first record reaching the final best), total
tuning wall time, and the per-eval trace (flat, runtime, elapsed, worker).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import tuning  # noqa: E402

PEAK = 37.05
DIMS = {("lu", "large"): 2000, ("lu", "extralarge"): 4000, ("cholesky", "large"): 2000,
        ("cholesky", "extralarge"): 4000}


def flops(kernel, size):
    if kernel == "3mm":
        n, l, m, o, p = {"large": (800, 900, 1000, 1100, 1200),
                         "extralarge": (1600, 1800, 2000, 2200, 2400),
                         "small": (80, 90, 100, 110, 120), "mini": (16, 18, 20, 22, 24)}[size]
        return 2.0 * (n * l * m + m * o * p + n * m * p)
    n = DIMS.get((kernel, size)) or {"small": 400, "mini": 64}[size]
    return (2 / 3 if kernel == "lu" else 1 / 3) * n ** 3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tuner", default="bayesopt")
    ap.add_argument("--kernel", default="3mm")
    ap.add_argument("--size", default="extralarge")
    ap.add_argument("--evals", type=int, default=200)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--devices", default="0")
    ap.add_argument("--max-seconds", type=float, default=0.0)
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    devs = tuple(int(x) for x in a.devices.split(","))
    recs, total = tuning.run_tuning_measured(a.tuner, a.kernel, a.size, a.seed, a.evals,
                                             devices=devs, max_seconds=a.max_seconds or None)
    ok = [r for r in recs if r.runtime_s is not None]
    best = min(ok, key=lambda r: r.runtime_s)
    f = flops(a.kernel, a.size)
    out = {"tuner": a.tuner, "kernel": a.kernel, "size": a.size, "seed": a.seed,
           "devices": list(devs), "evals": len(recs), "failed": len(recs) - len(ok),
           "best_config": list(best.config), "best_runtime_s": best.runtime_s,
           "best_gflops": f / best.runtime_s / 1e9,
           "best_pct_of_fp64_peak": 100 * f / best.runtime_s / 1e12 / PEAK,
           "time_to_best_s": tuning.time_to_best(recs), "total_tuning_s": total}
    if a.trace:
        out["trace"] = [[r.flat, r.runtime_s, round(r.elapsed_s, 4), r.worker] for r in recs]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
