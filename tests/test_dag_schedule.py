"""Host-side checks of the persistent tile-DAG schedule (dag_factor.cu), no GPU.

The task list is built by the C++ library (tt_dag_tasks).  These tests prove,
for LU and Cholesky over ragged knob combinations, that
  * list order is a valid execution order under the kernel's counter protocol
    (every task's wait condition already holds when it is reached, so the
    persistent kernel, which takes tasks in list order, cannot deadlock);
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


@pytest.mark.parametrize("kernel,n,by,bx", CASES)
def test_task_order_and_coverage(kernel, n, by, bx):
    tasks = _lib.dag_tasks(kernel, n, by, bx)
    assert tasks is not None
    chol = kernel == "cholesky"
    T, nt = bx, n // bx
    cnt = np.zeros((nt, nt), dtype=np.int64)
    for t in tasks:
        kind, j, k, r0, r1 = decode(t)
        for (tile, need) in needs(kind, j, k, r0, r1, T, chol):
            assert cnt[tile] >= need, (t, tile, need, cnt[tile])
        for tile, rows in signals(kind, j, k, r0, r1, T).items():
            i, jj = tile
            if chol:
                assert i >= jj, t
            stage = k if kind == GEMM else min(i, jj)
            # the rows land in this tile's current stage
            assert stage * T <= cnt[tile] and cnt[tile] + rows <= (stage + 1) * T, (t, tile)
            cnt[tile] += rows
    for i in range(nt):
        for jj in range(nt):
            if chol and jj > i:
                assert cnt[i, jj] == 0
            else:
                assert cnt[i, jj] == (min(i, jj) + 1) * T, (i, jj)


def run_tasks_numpy(a, tasks, bx, chol):
    a = a.copy()
    T = bx
    for t in tasks:
        kind, j, k, r0, r1 = decode(t)
        kT, jT = k * T, j * T
        d = a[kT:kT + T, kT:kT + T]
        if kind == DIAG:
            blk = d.copy()
            if chol:
                oracle.cholesky_factor_inplace(blk, T, T)
                a[kT:kT + T, kT:kT + T][np.tril_indices(T)] = blk[np.tril_indices(T)]
            else:
                oracle.lu_factor_inplace(blk, T, T)
                a[kT:kT + T, kT:kT + T] = blk
        elif kind == TRSM_L:
            m = np.tril(d).T if chol else np.triu(d)
            a[r0:r1, kT:kT + T] = np.linalg.solve(m.T, a[r0:r1, kT:kT + T].T).T
        elif kind == TRSM_U:
            lo = np.tril(d, -1) + np.eye(T)
            a[kT:kT + T, jT:jT + T] = np.linalg.solve(lo, a[kT:kT + T, jT:jT + T])
        else:
            b = a[jT:jT + T, kT:kT + T].T if chol else a[kT:kT + T, jT:jT + T]
            upd = a[r0:r1, jT:jT + T] - a[r0:r1, kT:kT + T] @ b
            if chol:
                rows = np.arange(r0, r1)[:, None]
                cols = np.arange(jT, jT + T)[None, :]
                upd = np.where(rows >= cols, upd, a[r0:r1, jT:jT + T])
            a[r0:r1, jT:jT + T] = upd
    return a


@pytest.mark.parametrize("kernel,n,by,bx", [c for c in CASES if c[1] <= 160])
def test_task_semantics_reproduce_reference(kernel, n, by, bx):
    chol = kernel == "cholesky"
    a0 = oracle.gen_spd(n, 5)
    out = run_tasks_numpy(a0, _lib.dag_tasks(kernel, n, by, bx), bx, chol)
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
