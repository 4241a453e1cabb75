import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle
from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase, lu_factor_inplace
n, by, bx = 400, 40, 40
ctx = Context(0)
r = GpuKernelRunner(KernelCase("lu", n, seed=1), ctx)
(a,) = r.inputs()
print("inputs == gen_spd:", np.array_equal(a, oracle.gen_spd(n, 1)))
ref = a.copy(); oracle.lu_factor_inplace(ref, n, n)
def err(w): return np.abs(w - ref).max() / np.abs(ref).max()
w1 = r.run((by, bx)); print("runner run1", err(w1))
w2 = r.run((by, bx)); print("runner run2", err(w2))
w = a.copy(); lu_factor_inplace(w, by, bx, ctx=ctx); print("oneshot", err(w))
w3 = r.run((by, bx)); print("runner run3", err(w3))
ctx2 = Context(0)
w = a.copy(); lu_factor_inplace(w, by, bx, ctx=ctx2); print("oneshot fresh ctx", err(w))
r2 = GpuKernelRunner(KernelCase("lu", n, seed=1), ctx2)
print("runner after oneshot in ctx2", err(r2.run((by, bx))))
