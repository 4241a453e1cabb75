#!/usr/bin/env python3
"""Watchdog stress: run (kernel, n, by, bx) configs repeatedly in one process
(measure protocol 1 warm-up + 3 reps each); stop at the first failure."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa

kern, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfgs = [tuple(map(int, c.split(','))) for c in sys.argv[4:]]
ctx = Context(0)
r = GpuKernelRunner(KernelCase(kern, n), ctx)
t0 = time.time()
runs = 0
for it in range(reps):
    for c in cfgs:
        try:
            r.measure(c, MeasureProtocol(1, 3, "median"))
            runs += 4
        except Exception as e:
            print(f"FAIL it={it} cfg={c} after {runs} runs: {e}", flush=True)
            sys.exit(1)
print(f"ok {runs} runs of {len(cfgs)} configs in {time.time() - t0:.1f}s", flush=True)
