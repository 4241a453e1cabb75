#!/usr/bin/env python3
"""Per-tile error map of a DAG factorisation vs the oracle (debug aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2309_07235_b200 import Context, lu_factor_inplace, cholesky_factor_inplace  # noqa

kern, n, by, bx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ctx = Context(0)
a = oracle.gen_spd(n, int(sys.argv[5]) if len(sys.argv) > 5 else 3)
ref = a.copy()
w = a.copy()
if kern == "lu":
    oracle.lu_factor_inplace(ref, n, n)
    lu_factor_inplace(w, by, bx, ctx=ctx)
else:
    oracle.cholesky_factor_inplace(ref, n, n)
    try:
        cholesky_factor_inplace(w, by, bx, ctx=ctx)
    except Exception as e:
        print("error", e)
    ref, w = np.tril(ref), np.tril(w)
nt = n // bx
np.set_printoptions(linewidth=200, precision=1)
err = np.zeros((nt, nt))
for i in range(nt):
    for j in range(nt):
        d = np.abs(w[i*bx:(i+1)*bx, j*bx:(j+1)*bx] - ref[i*bx:(i+1)*bx, j*bx:(j+1)*bx]).max()
        err[i, j] = np.log10(d + 1e-300)
print(err)
