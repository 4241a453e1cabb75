"""Host-side checks of the persistent tile-DAG schedule (dag_factor.cu), no GPU.

The queue's task list is built by the C++ library (tt_dag_tasks); the walker
CTA's per-step work (update + DIAG of tile (k,k), L(k+1,k), U(k,k+1)) is
modelled here exactly as the kernel runs it.  These tests prove, for LU and
Cholesky over ragged knob combinations, that
  * running walker step k before the first queue task of step k is a valid
    execution order under the kernel's counter protocol (every wait
    condition already holds when it is reached; the queue is taken in list
    order and only waits on earlier tasks or earlier walker steps, so the
    persistent kernel cannot deadlock);
  * every tile receives each of its stages exactly once and ends complete;
  * executing the tasks in list order with plain numpy arithmetic reproduces
    the reference factorisation (oracle), i.e. the task decomposition
    (regions anchored at the panel end, Cholesky lower clipping) is the
    reference's operation set (kernels.cpp:178-218, :264-308).
"""
import numpy as np
import pytest

import oracle
from paper_2309_07235_b200 import _lib

DIAG, TRSM_L, TRSM_U, GEMM = 0, 1, 2, 3

CASES = [("lu", 64, 8, 8), ("lu", 64, 16, 8), ("lu", 96, 3, 12), ("lu", 120, 40, 24),
         ("lu", 100, 25, 50), ("lu", 2000, 400, 50), ("lu", 160, 160, 16), ("lu", 64, 1, 32),
         ("cholesky", 64, 8, 8), ("cholesky", 96, 32, 12), ("cholesky", 120, 5, 20),
         ("cholesky", 100, 50, 25), ("cholesky", 4000, 160, 50), ("cholesky", 64, 64, 64)]


def decode(t):
    return int(t[0]) & 3, int(t[0]) >> 2, int(t[1]), int(t[2]), int(t[3])


def tiles(r0, r1, T):
    return range(r0 // T, (r1 - 1) // T + 1)


def needs(kind, j, k, r0, r1, T, chol):
    kT = k * T
    if kind == DIAG:
        return [((k, k), kT)]
    if kind == TRSM_L:
        return [((i, k), kT) for i in tiles(r0, r1, T)] + [((k, k), kT + T)]
    if kind == TRSM_U:
        return [((k, j), kT), ((k, k), kT + T)]
    out = []
    for i in tiles(r0, r1, T):
        out += [((i, j), kT), ((i, k), kT + T)]
    return out + [((j, k) if chol else (k, j), kT + T)]


def signals(kind, j, k, r0, r1, T):
    if kind == DIAG:
        return {(k, k): T}
    if kind == TRSM_U:
        return {(k, j): T}
    col = k if kind == TRSM_L else j
    return {(i, col): min(r1, (i + 1) * T) - max(r0, i * T) for i in tiles(r0, r1, T)}


def walker_needs(k, T, nt, chol):
    out = []
    if k >= 2:
        out.append(((k, k), (k - 1) * T))
    if k + 1 < nt:
        out.append(((k + 1, k), k * T))
        if not chol:
            out.append(((k, k + 1), k * T))
    return out


def walker_signals(k, T, nt, chol):
    sig = {(k, k): 2 * T if k >= 1 else T}
    if k + 1 < nt:
        sig[(k + 1, k)] = T
        if not chol:
            sig[(k, k + 1)] = T
    return sig


def interleaved(tasks, nt, T, chol, nurg):
    """A sequential execution the kernel's queues admit: per step k the walker,
    then step k of the urgent queue, then step k of the bulk queue, each queue
    in its own order.  Every wait condition must hold when its task is
    reached; together with the per-queue step order this is the kernel's
    deadlock-freedom argument (see build_tasks)."""
    urg, bulk = tasks[:nurg], tasks[nurg:]
    for q in (urg, bulk):
        assert np.all(np.diff(q[:, 1]) >= 0), "queue not in step order"
    cnt = np.zeros((nt, nt), dtype=np.int64)
    out = []
    iu = ib = 0
    for k in range(nt):
        for tile, nd in walker_needs(k, T, nt, chol):
            assert cnt[tile] >= nd, ("walker", k, tile, nd, cnt[tile])
        out.append(("W", k))
        for tile, rows in walker_signals(k, T, nt, chol).items():
            cnt[tile] += rows
        for q, idx in ((urg, "u"), (bulk, "b")):
            i = iu if idx == "u" else ib
            while i < len(q) and q[i][1] == k:
                t = q[i]
                kind, j, kk, r0, r1 = decode(t)
                for tile, nd in needs(kind, j, kk, r0, r1, T, chol):
                    assert cnt[tile] >= nd, (idx, t, tile, nd, cnt[tile])
                out.append(("Q", t))
                for tile, rows in signals(kind, j, kk, r0, r1, T).items():
                    cnt[tile] += rows
                i += 1
            if idx == "u":
                iu = i
            else:
                ib = i
    assert iu == len(urg) and ib == len(bulk)
    return out


@pytest.mark.parametrize("kernel,n,by,bx", CASES)
def test_task_order_and_coverage(kernel, n, by, bx):
    tasks = _lib.dag_tasks(kernel, n, by, bx)
    assert tasks is not None
    chol = kernel == "cholesky"
    T, nt = bx, n // bx
    assert not np.any((tasks[:, 0] & 3) == DIAG)  # DIAG belongs to the walker
    cnt = np.zeros((nt, nt), dtype=np.int64)
    nurg = _lib.load().tt_dag_urgent(_lib.KERNEL_IDS[kernel], n, by, bx)
    for what, t in interleaved(tasks, nt, T, chol, nurg):
        if what == "W":
            need, sig = walker_needs(t, T, nt, chol), walker_signals(t, T, nt, chol)
        else:
            kind, j, k, r0, r1 = decode(t)
            need, sig = needs(kind, j, k, r0, r1, T, chol), signals(kind, j, k, r0, r1, T)
        for (tile, nd) in need:
            assert cnt[tile] >= nd, (what, t, tile, nd, cnt[tile])
        for tile, rows in sig.items():
            i, jj = tile
            if chol:
                assert i >= jj, t
            cnt[tile] += rows
            assert cnt[tile] <= (min(i, jj) + 1) * T, (what, t, tile)
    for i in range(nt):
        for jj in range(nt):
            if chol and jj > i:
                assert cnt[i, jj] == 0
            else:
                assert cnt[i, jj] == (min(i, jj) + 1) * T, (i, jj)


def run_tasks_numpy(a, tasks, bx, chol, nurg):
    a = a.copy()
    T = bx
    nt = a.shape[0] // T

    def trsm_l(k, r0, r1):
        kT = k * T
        d = a[kT:kT + T, kT:kT + T]
        m = np.tril(d).T if chol else np.triu(d)
        a[r0:r1, kT:kT + T] = np.linalg.solve(m.T, a[r0:r1, kT:kT + T].T).T

    def trsm_u(k, j):
        kT, jT = k * T, j * T
        lo = np.tril(a[kT:kT + T, kT:kT + T], -1) + np.eye(T)
        a[kT:kT + T, jT:jT + T] = np.linalg.solve(lo, a[kT:kT + T, jT:jT + T])

    def gemm(k, r0, r1, j):
        kT, jT = k * T, j * T
        b = a[jT:jT + T, kT:kT + T].T if chol else a[kT:kT + T, jT:jT + T]
        upd = a[r0:r1, jT:jT + T] - a[r0:r1, kT:kT + T] @ b
        if chol:
            rows = np.arange(r0, r1)[:, None]
            cols = np.arange(jT, jT + T)[None, :]
            upd = np.where(rows >= cols, upd, a[r0:r1, jT:jT + T])
        a[r0:r1, jT:jT + T] = upd

    for what, t in interleaved(tasks, nt, T, chol, nurg):
        if what == "W":  # walker step k
            k = t
            kT = k * T
            if k >= 1:
                gemm(k - 1, kT, kT + T, k)
            blk = a[kT:kT + T, kT:kT + T].copy()
            if chol:
                oracle.cholesky_factor_inplace(blk, T, T)
                a[kT:kT + T, kT:kT + T][np.tril_indices(T)] = blk[np.tril_indices(T)]
            else:
                oracle.lu_factor_inplace(blk, T, T)
                a[kT:kT + T, kT:kT + T] = blk
            if k + 1 < nt:
                trsm_l(k, kT + T, kT + 2 * T)
                if not chol:
                    trsm_u(k, k + 1)
            continue
        kind, j, k, r0, r1 = decode(t)
        if kind == TRSM_L:
            trsm_l(k, r0, r1)
        elif kind == TRSM_U:
            trsm_u(k, j)
        else:
            gemm(k, r0, r1, j)
    return a


@pytest.mark.parametrize("kernel,n,by,bx", [c for c in CASES if c[1] <= 160])
def test_task_semantics_reproduce_reference(kernel, n, by, bx):
    chol = kernel == "cholesky"
    a0 = oracle.gen_spd(n, 5)
    nurg = _lib.load().tt_dag_urgent(_lib.KERNEL_IDS[kernel], n, by, bx)
    out = run_tasks_numpy(a0, _lib.dag_tasks(kernel, n, by, bx), bx, chol, nurg)
    ref = a0.copy()
    if chol:
        oracle.cholesky_factor_inplace(ref, by, bx)
        assert np.array_equal(np.triu(out, 1), np.triu(a0, 1))  # upper triangle never written
        assert oracle.cholesky_residual(a0, np.tril(out)) <= 1e-13
        assert np.abs(np.tril(out) - np.tril(ref)).max() <= 1e-10 * np.abs(ref).max()
    else:
        oracle.lu_factor_inplace(ref, by, bx)
        assert oracle.lu_residual_packed(a0, out) <= 1e-13
        assert np.abs(out - ref).max() <= 1e-10 * np.abs(ref).max()


def test_ineligible_configs_use_graph_schedule():
    assert _lib.dag_tasks("lu", 2000, 400, 5) is None     # tile below the DMMA atom
    assert _lib.dag_tasks("lu", 2000, 400, 80) is None    # tile above 64 (graph schedule)
    assert _lib.dag_tasks("cholesky", 4000, 4000, 4000) is None
