"""Row-sharded scaled 3mm across G GPUs with an NCCL exchange of F.

G = (A*B)*(C*D) with n = l = m = o = p = N.  Rank r owns rows
[r*N/G, (r+1)*N/G) of A, C, E, F, G; B and D are replicated.  Each rank
computes E_r = A_r*B and F_r = C_r*D with the knob-driven DMMA GEMM, then
G_r = E_r * F is accumulated over KB fixed K-blocks of F in ASCENDING block
order: block b (rows of F owned by rank b // (KB/G)) is broadcast by its
owner over NCCL on the collective stream while the GEMM of block b-1 runs on
the compute stream.  Because the K-blocking (KB) does not depend on G, every
element of G sees the same sequence of fp64 DMMA accumulations through
memory for any G, so the result is bitwise identical for G in {1, 2, 4, 8}.

Inputs are generated on the device (counter-based U[0,1), shard-invariant,
tt_dev_fill_uniform): there is no CPU oracle at N = 32768 (2.1e14 flop).
Correctness: the Freivalds check G*x == A*(B*(C*(D*x))) (relative 1e-10) and
the 1-vs-G bitwise equality.

Plumbing (device buffers, NCCL, streams) is torch; the math is the C ABI.
`gemm_fn` can be swapped for a deterministic CPU stand-in so the sharding
and ordering logic is testable with the gloo backend (tests/test_sharded.py).
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass


@dataclass
class ScaledConfig:
    n: int = 32768
    kblocks: int = 8          # K-split of G = E*F; fixed so results are G-invariant
    seed: int = 20230913
    cfg: tuple = (128, 128, 128, 128, 128, 128)  # CTA regions (P0..P5) of the three products


def _tt_gemm(ctx, stream_ptr):
    lib = ctx.lib

    def gemm(a, b, c, beta: int):
        M, K = a.shape
        N = b.shape[1]
        fy = _fit(M, 128)
        fx = _fit(N, 128)
        rc = lib.tt_dev_gemm(ctx.handle, ctypes.c_void_p(a.data_ptr()), a.stride(0),
                             ctypes.c_void_p(b.data_ptr()), b.stride(0), 0,
                             ctypes.c_void_p(c.data_ptr()), c.stride(0), M, N, K, fy, fx, 1, beta,
                             stream_ptr)
        ctx.check(rc)
    return gemm


def _fit(extent: int, f: int) -> int:
    f = min(f, extent)
    while extent % f:
        f -= 1
    return f


def fill_inputs(ctx, stream_ptr, mats: dict, row0: int, seed: int):
    """Fills the rank's shards: A_r, C_r (rows row0..), B, D (replicated)."""
    ids = {"a": 0, "b": 1, "c": 2, "d": 3}
    for name, t in mats.items():
        r0 = row0 if name in ("a", "c") else 0
        rc = ctx.lib.tt_dev_fill_uniform(ctx.handle, ctypes.c_void_p(t.data_ptr()), t.shape[0],
                                         t.shape[1], t.stride(0), r0, seed, ids[name], stream_ptr)
        ctx.check(rc)


def sharded_mm3(A_r, B, C_r, D, rank: int, world: int, kblocks: int, gemm_fn, dist=None,
                comm_wait=None):
    """The sharded product.  Returns (G_r, F_full, E_r).

    gemm_fn(a, b, c, beta): c (+)= a @ b, deterministic per call.
    dist: torch.distributed (None for world == 1).
    """
    import torch
    N = B.shape[0]
    rows = A_r.shape[0]
    E_r = torch.empty((rows, B.shape[1]), dtype=torch.float64, device=A_r.device)
    F_r_view = None
    F = torch.empty((N, D.shape[1]), dtype=torch.float64, device=A_r.device)
    # my shard of F lives inside the gathered F (no extra copy)
    F_r_view = F[rank * rows:(rank + 1) * rows]
    gemm_fn(A_r, B, E_r, 0)
    gemm_fn(C_r, D, F_r_view, 0)
    G_r = torch.empty((rows, D.shape[1]), dtype=torch.float64, device=A_r.device)
    kb = N // kblocks
    per_rank = kblocks // world
    works = []
    if world > 1:
        # ascending broadcasts of every F block from its owner (async, NCCL stream)
        for b in range(kblocks):
            owner = b // per_rank
            works.append(dist.broadcast(F[b * kb:(b + 1) * kb], src=owner, async_op=True))
    for b in range(kblocks):
        if works:
            works[b].wait()  # the compute stream waits for block b only
        gemm_fn(E_r[:, b * kb:(b + 1) * kb], F[b * kb:(b + 1) * kb], G_r, 0 if b == 0 else 1)
    return G_r, F, E_r


def run_scaled(n: int = 32768, steps: int = 1, warmup: int = 1, kblocks: int = 8,
               seed: int = 20230913, check: bool = True):
    """torchrun entry: one rank per GPU.  Returns rank 0's result dict."""
    import os

    import torch
    import torch.distributed as dist

    from .kernels import Context
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl")
    if n % (world * kblocks) or kblocks % world:
        raise ValueError("n must divide into world*kblocks blocks and kblocks % world == 0")
    torch.cuda.set_device(local)
    ctx = Context(local)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    rows = n // world
    dev = f"cuda:{local}"
    mats = {"a": torch.empty((rows, n), dtype=torch.float64, device=dev),
            "b": torch.empty((n, n), dtype=torch.float64, device=dev),
            "c": torch.empty((rows, n), dtype=torch.float64, device=dev),
            "d": torch.empty((n, n), dtype=torch.float64, device=dev)}
    fill_inputs(ctx, sptr, mats, rank * rows, seed)
    gemm = _tt_gemm(ctx, sptr)
    d = dist if world > 1 else None
    for _ in range(warmup):
        sharded_mm3(mats["a"], mats["b"], mats["c"], mats["d"], rank, world, kblocks, gemm, d)
    torch.cuda.synchronize()
    if d:
        d.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        G_r, F, E_r = sharded_mm3(mats["a"], mats["b"], mats["c"], mats["d"], rank, world,
                                  kblocks, gemm, d)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if d:
        d.all_reduce(t, op=d.ReduceOp.MAX)
    ms_max = float(t.item())
    flops = 6.0 * n ** 3
    out = {"n": n, "world": world, "kblocks": kblocks, "ms": ms_max,
           "tflops": flops / (ms_max * 1e-3) / 1e12}
    if check:
        # Freivalds: G x vs A (B (C (D x))), x ~ U[0,1) (fixed generator)
        g = torch.Generator(device=dev).manual_seed(7)
        x = torch.rand((n, 1), dtype=torch.float64, device=dev, generator=g)
        dx = mats["d"] @ x
        cdx_r = mats["c"] @ dx
        cdx = torch.empty((n, 1), dtype=torch.float64, device=dev)
        if d:
            d.all_gather_into_tensor(cdx, cdx_r)
        else:
            cdx = cdx_r
        rhs_r = mats["a"] @ (mats["b"] @ cdx)
        lhs_r = G_r @ x
        rel = ((lhs_r - rhs_r).abs().max() / rhs_r.abs().max()).reshape(1)
        if d:
            d.all_reduce(rel, op=d.ReduceOp.MAX)
        out["freivalds_rel"] = float(rel.item())
        # order-independent checksum of G (sum of per-rank fp64 sums, rank order)
        s = G_r.sum().reshape(1)
        sums = [torch.zeros_like(s) for _ in range(world)] if d else [s]
        if d:
            d.all_gather(sums, s)
        out["checksum_rank_sums"] = [float(v.item()) for v in sums]
        out["g_hash_rank0_rows"] = float(G_r[:8].sum().item())
    if d:
        d.barrier()
    return out if rank == 0 else None
