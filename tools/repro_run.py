#!/usr/bin/env python3
"""runner.run over configs (kernel n cfg...), fresh context; reports the first failure."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase  # noqa
kern, n = sys.argv[1], int(sys.argv[2])
ctx = Context(0)
r = GpuKernelRunner(KernelCase(kern, n), ctx)
for c in sys.argv[3:]:
    cfg = tuple(map(int, c.split(',')))
    try:
        r.run(cfg)
        print(kern, n, cfg, "ok residual %.2e" % r.residual(), flush=True)
    except Exception as e:
        print(kern, n, cfg, "FAIL", e, flush=True)
        sys.exit(1)
