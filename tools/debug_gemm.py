#!/usr/bin/env python3
"""Debug aid: one GEMM configuration, mismatch pattern + per-call timing."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2309_07235_b200 import Context  # noqa: E402


def run(ctx, M, N, K, fy, fx, off, bt, alpha, beta):
    lib = ctx.lib
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    torch.manual_seed(1)
    lda = (K + off + 1) // 2 * 2 + 2
    A = torch.rand(M, lda, dtype=torch.float64, device="cuda")[:, off:off + K]
    if bt:
        ldb = (K + off + 1) // 2 * 2
        B = torch.rand(N, ldb, dtype=torch.float64, device="cuda")[:, off:off + K]
        ref = A @ B.T
    else:
        ldb = (N + off + 1) // 2 * 2 + 4
        B = torch.rand(K, ldb, dtype=torch.float64, device="cuda")[:, off:off + N]
        ref = A @ B
    ldc = N + 3
    C = torch.rand(M, ldc, dtype=torch.float64, device="cuda")
    C0 = C[:, :N].clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.tt_dev_gemm(ctx.handle, ctypes.c_void_p(A.data_ptr()), lda, ctypes.c_void_p(B.data_ptr()),
                         ldb, bt, ctypes.c_void_p(C.data_ptr()), ldc, M, N, K, fy, fx, alpha, beta, s)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    want = alpha * ref + (C0 if beta else 0)
    bad = ((C[:, :N] - want).abs() > 1e-12 * want.abs().max()).nonzero()
    print(f"M={M} N={N} K={K} fy={fy} fx={fx} off={off} bt={bt} a={alpha} b={beta} rc={rc} "
          f"{dt*1e3:.2f} ms bad={bad.shape[0]}", flush=True)
    if bad.shape[0]:
        rows = sorted(set(bad[:, 0].tolist()))
        cols = sorted(set(bad[:, 1].tolist()))
        print("  rows", rows[:10], "...", len(rows), " cols", cols[:20], "...", len(cols))
        r, c = bad[0].tolist()
        print("  sample", r, c, "C0", C0[r, c].item(), "got", C[r, c].item(), "want", want[r, c].item(),
              "ab", ref[r, c].item())


def main():
    ctx = Context(0)
    for off in (0, 1):
        for a, b in ((1, 0), (-1, 1), (1, 1), (-1, 0)):
            run(ctx, 200, 136, 33, 200, 68, off, 0, a, b)
    run(ctx, 200, 136, 33, 200, 68, 0, 1, -1, 1)
    run(ctx, 128, 128, 16, 128, 128, 0, 0, -1, 1)
    run(ctx, 200, 136, 33, 100, 68, 0, 0, -1, 1)
    run(ctx, 200, 136, 33, 200, 34, 0, 0, -1, 1)
    for M, N, K in ((37, 45, 29), (257, 129, 47)):
        for fy, fx in ((1, 1), (37 if M == 37 else 257, 45 if N == 45 else 129)):
            run(ctx, M, N, K, fy, fx, 0, 0, -1, 1)


if __name__ == "__main__":
    main()
