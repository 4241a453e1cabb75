#!/usr/bin/env python3
"""GPU sanity + timing of the persistent tile-DAG schedule vs the graph schedule."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa
from paper_2309_07235_b200 import cholesky_tiled, lu_factor_inplace, _lib  # noqa: E402

ctx = Context(0)
for n, by, bx in [(64, 8, 8), (64, 16, 32), (96, 24, 48), (120, 5, 20), (96, 3, 12)]:
    a = oracle.gen_spd(n, 1)
    w = a.copy()
    t0 = time.time()
    lu_factor_inplace(w, by, bx, ctx=ctx)
    res = oracle.lu_residual_packed(a, w)
    l = cholesky_tiled(a, by, bx, ctx=ctx)
    rc = oracle.cholesky_residual(a, l)
    dag = _lib.dag_tasks("lu", n, by, bx) is not None
    print(f"n={n} ({by},{bx}) dag={dag} lu_res={res:.2e} chol_res={rc:.2e} {time.time()-t0:.2f}s", flush=True)

proto = MeasureProtocol(2, 5, "median")
for kern, n, cfgs in [("lu", 2000, [(400, 50), (200, 40), (100, 50), (400, 40), (2000, 50), (50, 50), (400, 80)]),
                      ("cholesky", 4000, [(160, 50), (200, 40), (500, 50), (160, 32), (100, 25), (160, 160)]),
                      ("lu", 4000, [(160, 50), (200, 40), (160, 32)])]:
    r = GpuKernelRunner(KernelCase(kern, n, seed=1), ctx)
    fl = (2 / 3 if kern == "lu" else 1 / 3) * n ** 3
    for cfg in cfgs:
        try:
            s = r.measure(cfg, proto)
            r.run(cfg)
            res = r.residual()
            print(f"{kern} n={n} {cfg} dag={_lib.dag_tasks(kern, n, *cfg) is not None} "
                  f"{s*1e3:.3f} ms {fl/s/1e12:.2f} TF/s res={res:.2e}", flush=True)
        except Exception as e:
            print(f"{kern} n={n} {cfg} ERROR {e}", flush=True)
