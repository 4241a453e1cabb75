#!/usr/bin/env python3
"""Debug aid: launch every DMMA GEMM variant once (sync after each) and check
it against torch fp64; then run LU / Cholesky schedules eagerly (TT_EAGER=1)."""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase  # noqa: E402


def main():
    ctx = Context(0)
    lib = ctx.lib
    stream = torch.cuda.current_stream()
    s = ctypes.c_void_p(stream.cuda_stream)
    bad = 0
    for bt in (0, 1):
        for bm in (8, 16, 32, 64, 128):
            for bn in (8, 16, 32, 64, 128):
                M, N, K = 2 * bm, 2 * bn, 37
                A = torch.rand(M, 40, dtype=torch.float64, device="cuda")
                B = torch.rand(N, 40, dtype=torch.float64, device="cuda") if bt else \
                    torch.rand(K, N, dtype=torch.float64, device="cuda")
                C = torch.zeros(M, N, dtype=torch.float64, device="cuda")
                torch.cuda.synchronize()
                rc = lib.tt_dev_gemm(ctx.handle, ctypes.c_void_p(A.data_ptr()), 40,
                                     ctypes.c_void_p(B.data_ptr()), 40 if bt else N, bt,
                                     ctypes.c_void_p(C.data_ptr()), N, M, N, K, bm, bn, 1, 0, s)
                msg = lib.tt_last_error(ctx.handle).decode() if rc else ""
                try:
                    torch.cuda.synchronize()
                    ref = A[:, :K] @ (B[:, :K].T if bt else B)
                    err = ((C - ref).abs().max() / ref.abs().max()).item()
                except Exception as e:  # noqa
                    print(f"bt={bt} bm={bm} bn={bn}: DEVICE ERROR {e}", flush=True)
                    return 1
                ok = rc == 0 and err < 1e-13
                bad += not ok
                print(f"bt={bt} bm={bm} bn={bn}: rc={rc} {msg} err={err:.3e} {'OK' if ok else 'BAD'}",
                      flush=True)
    for kern, n, cfgs in (("lu", 2000, [(400, 50), (40, 40), (125, 125)]),
                          ("cholesky", 400, [(80, 40), (400, 400)])):
        r = GpuKernelRunner(KernelCase(kern, n), ctx)
        for cfg in cfgs:
            try:
                r.run(cfg, want_output=False)
                print(kern, n, cfg, "residual", r.residual(), flush=True)
            except Exception as e:  # noqa
                print(kern, n, cfg, "ERROR", e, flush=True)
                bad += 1
    print("bad", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    os.environ.setdefault("TT_EAGER", "1")
    sys.exit(main())
