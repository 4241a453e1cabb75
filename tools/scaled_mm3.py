#!/usr/bin/env python3
"""Scaled 3mm (n=l=m=o=p=N) row-sharded over the ranks of a torchrun job.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        tools/scaled_mm3.py --n 32768 --steps 2 --warmup 1
Rank 0 prints one JSON line (aggregate TFLOP/s, Freivalds residual, per-rank
checksums for the 1-vs-G bitwise comparison)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200.sharded import run_scaled  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--kblocks", type=int, default=8)
a = ap.parse_args()
import os  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import ClockSampler  # noqa: E402

# SM clock + throttle reasons sampled over the whole run (the timed steps dominate it)
with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
    out = run_scaled(a.n, a.steps, a.warmup, a.kblocks)
if out is not None:
    out["clocks"] = clk.summary()
    out["pct_of_fp64_peak_per_gpu"] = 100.0 * out["tflops"] / out["world"] / 37.05
    print(json.dumps(out), flush=True)
