#!/usr/bin/env python3
"""Per-task timeline of the persistent tile-DAG schedule (TT_DAG_TRACE=1).

Usage: TT_DAG_TRACE=1 python tools/dag_trace.py lu 2000 400 50 [out.npz]
Prints per-kind run/wait times and the DIAG critical-chain timeline."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

os.environ["TT_DAG_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, _lib  # noqa: E402

kern, n, by, bx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ctx = Context(0)
r = GpuKernelRunner(KernelCase(kern, n, seed=1), ctx)
for _ in range(3):
    r.run((by, bx), want_output=False)
tasks = _lib.dag_tasks(kern, n, by, bx)
nt = len(tasks)
nsteps = n // _lib.dag_tile(n, by, bx)
trall = np.zeros((nt + nsteps, 8), dtype=np.uint64)
got = ctx.lib.tt_dag_trace(ctx.handle, trall.ctypes.data_as(ctypes.c_void_p), nt + nsteps)
tr = trall[:nt]
wk = (trall[nt:, :8].astype(np.int64) - int(tr[:, 0].min())) / 1e3
t = tr[:, :3].astype(np.int64)
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
kind = tasks[:, 0] & 3
names = ["DIAG", "TRSM_L", "TRSM_U", "GEMM"]
span = max(t[:, 2].max(), wk[:, 5].max())
print(f"{kern} n={n} ({by},{bx}): {nt} tasks, span {span:.1f} us, SMs used {len(set(tr[:, 3]))}")
for k in range(4):
    m = kind == k
    if m.any():
        run = t[m, 2] - t[m, 1]
        wait = t[m, 1] - t[m, 0]
        print(f"  {names[k]:6s} n={m.sum():6d} run mean {run.mean():7.2f} max {run.max():7.2f} "
              f"| wait mean {wait.mean():7.2f} max {wait.max():7.2f} us | busy sum {run.sum():9.1f}")
w = wk[1:-1]
print("  walker per step (us): wait tile %.2f, update %.2f, DIAG %.2f, store+wait panel %.2f, L/U tiles %.2f | period %.2f" % (
    (w[:, 1] - w[:, 0]).mean(), (w[:, 2] - w[:, 1]).mean(), (w[:, 3] - w[:, 2]).mean(),
    (w[:, 4] - w[:, 3]).mean(), (w[:, 5] - w[:, 4]).mean(), np.diff(wk[:, 0]).mean()))
print("  walker step k=5: " + " ".join("%.1f" % x for x in wk[5]))
print("  walker L/U split (us): loads+sync %.2f, solves+sync %.2f, publish %.2f" % (
    (w[:, 6] - w[:, 4]).mean(), (w[:, 7] - w[:, 6]).mean(), (w[:, 5] - w[:, 7]).mean()))
for kk, nm, a_, b_ in [(2, "TRSM_U", "M load+sync", "8x8 inverses+sync"), (1, "TRSM_L", "M load+sync", "8x8 inverses+sync"), (3, "GEMM", "B load+sync", "first strip (warp 0) done")]:
    mm = kind == kk
    if mm.any():
        q = (tr[mm, 4:6].astype(np.int64) - t0) / 1e3
        print(f"  {nm} phases (us after ready): {a_} {(q[:, 0] - t[mm, 1]).mean():.2f}, {b_} +{(q[:, 1] - q[:, 0]).mean():.2f}, end +{(t[mm, 2] - q[:, 1]).mean():.2f}")
mm = kind == 3
q = (tr[mm, 4:8].astype(np.int64) - t0) / 1e3
print("  GEMM first strip (warp 0) after B: deps +%.2f, loads +%.2f, compute+store +%.2f us" % (
    (q[:, 3] - q[:, 0]).mean(), (q[:, 2] - q[:, 3]).mean(), (q[:, 1] - q[:, 2]).mean()))
busy = (t[:, 2] - t[:, 1]).sum()
grid = len(set(tr[:, 3]))
print(f"  utilisation (task run time / (SMs x span)) = {busy / (grid * span):.3f}")

if len(sys.argv) > 5:
    np.savez(sys.argv[5], tasks=tasks, trace=tr, walker=trall[nt:], nurgent=ctx.lib.tt_dag_urgent(0 if kern == "lu" else 1, n, by, bx))
