#!/usr/bin/env python3
"""Runner-path (device inputs, measure then run) error map vs the oracle."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, MeasureProtocol  # noqa

kern, n, by, bx, nmeas = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
ctx = Context(0)
r = GpuKernelRunner(KernelCase(kern, n, seed=1), ctx)
if nmeas:
    r.measure((by, bx), MeasureProtocol(1, nmeas, "median"))
w = r.run((by, bx))
(a,) = r.inputs()
ref = a.copy()
(oracle.lu_factor_inplace if kern == "lu" else oracle.cholesky_factor_inplace)(ref, n, n)
if kern != "lu":
    ref, w = np.tril(ref), np.tril(w)
nt = n // bx
bad = np.argwhere(~np.isfinite(w))
print("nonfinite", len(bad), bad[:5].tolist() if len(bad) else "")
err = np.zeros((nt, nt))
for i in range(nt):
    for j in range(nt):
        d = np.abs(w[i*bx:(i+1)*bx, j*bx:(j+1)*bx] - ref[i*bx:(i+1)*bx, j*bx:(j+1)*bx]).max()
        err[i, j] = np.log10(d + 1e-300)
np.set_printoptions(linewidth=220, precision=0, threshold=100000)
print(err[:8, :12])
print("max err", np.nanmax(err))
