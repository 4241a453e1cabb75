#!/usr/bin/env python3
"""Times LU/Cholesky for one (kernel, n, by, bx) in a fresh process (the
schedule env vars are read once per process).  Prints one JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa

kern, n, by, bx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ctx = Context(0)
r = GpuKernelRunner(KernelCase(kern, n, seed=1), ctx)
s = r.measure((by, bx), MeasureProtocol(2, 7, "median"))
fl = (2 / 3 if kern == "lu" else 1 / 3) * n ** 3
import os
print(json.dumps({"kernel": kern, "n": n, "by": by, "bx": bx, "band": os.environ.get("TT_DAG_BAND"),
                  "ucta": os.environ.get("TT_DAG_URGENT_CTAS"),
                  "pf": os.environ.get("TT_DAG_PREFETCH"), "chunk": os.environ.get("TT_DAG_CHUNK"), "merge": os.environ.get("TT_DAG_MERGE"), "ms": s * 1e3, "tflops": fl / s / 1e12}))
