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
    """{kind | j << 2, k0 | q << 16, r0, r1}: a GEMM applies steps [k0, k0+q)."""
    return int(t[0]) & 3, int(t[0]) >> 2, int(t[1]) & 0xFFFF, max(1, int(t[1]) >> 16), \
        int(t[2]), int(t[3])


def tiles(r0, r1, T):
    return range(r0 // T, (r1 - 1) // T + 1)


def nchunks(m, d, o):
    """dag_factor.cuh: chunks of a tile with m updates in a column of phase o
    (boundaries o, o+d, o+2d, ... ending at or before step m-1)."""
    if m < 1 or d <= 1:
        return 0
    if o == 0:
        return (m - 1) // d
    return 1 + (m - 1 - o) // d if o <= m - 1 else 0


def chunk_end(m, d, o):
    nc = nchunks(m, d, o)
    if o == 0:
        return nc * d
    return 0 if nc == 0 else o + (nc - 1) * d


def stages_before(m, s, d, col):
    """Stages of tile column `col` (phase col % d) with m updates covering steps < s."""
    o = col % d
    e = chunk_end(m, d, o)
    if s > e:
        return nchunks(m, d, o) + (s - e)
    if s == 0:
        return 0
    return s // d if o == 0 else 1 + (s - o) // d


def fin(m, d, col):
    return stages_before(m, m, d, col) + 1


def ready(t):
    kind, _, k0, q, _, _ = decode(t)
    return k0 + q - 1 if kind == GEMM else k0


def needs(kind, j, k0, q, r0, r1, T, chol, d, full=False):
    """What the kernel waits on (dep_at / strip_deps).  A GEMM over [k0, kl] waits
    only for the operands of step kl; full=True lists every step's operands,
    which the chain argument (dag_factor.cu, dep_at) says are then final too."""
    if kind == DIAG:
        return [((k0, k0), stages_before(k0, k0 - 1, d, k0) * T)]
    if kind == TRSM_L:
        return [((i, k0), stages_before(k0, k0, d, k0) * T) for i in tiles(r0, r1, T)] + \
            [((k0, k0), fin(k0, d, k0) * T)]
    if kind == TRSM_U:
        return [((k0, j), stages_before(k0, k0, d, j) * T), ((k0, k0), fin(k0, d, k0) * T)]
    kl = k0 + q - 1
    ks = range(k0, kl + 1) if full else [kl]
    out = []
    for i in tiles(r0, r1, T):
        out.append(((i, j), stages_before(min(i, j), k0, d, j) * T))
        out += [((i, k), fin(k, d, k) * T) for k in ks]
    return out + [(((j, k) if chol else (k, j)), fin(k, d, k if chol else j) * T) for k in ks]


def signals(kind, j, k0, r0, r1, T):
    if kind == DIAG:
        return {(k0, k0): T}
    if kind == TRSM_U:
        return {(k0, j): T}
    col = k0 if kind == TRSM_L else j
    return {(i, col): min(r1, (i + 1) * T) - max(r0, i * T) for i in tiles(r0, r1, T)}


def walker_needs(k, T, nt, chol, d):
    out = []
    if k >= 1:
        out.append(((k, k), stages_before(k, k - 1, d, k) * T))
    if k + 1 < nt:
        out.append(((k + 1, k), stages_before(k, k, d, k) * T))
        if not chol:
            out.append(((k, k + 1), stages_before(k, k, d, k + 1) * T))
    return out


def walker_signals(k, T, nt, chol):
    sig = {(k, k): 2 * T if k >= 1 else T}
    if k + 1 < nt:
        sig[(k + 1, k)] = T
        if not chol:
            sig[(k, k + 1)] = T
    return sig


def key(t, T, d):
    """(deadline, ready step, TRSM before GEMM): the queue order of build_tasks."""
    kind, j, k0, q, r0, r1 = decode(t)
    if kind != GEMM:
        return (k0, k0, 0)
    dls = []
    for i in tiles(r0, r1, T):
        e = chunk_end(min(i, j), d, j % d)
        if k0 + q <= e:  # a chunk: the next chunk's ready step, or the first single
            dls.append(k0 + q + d - 1 if k0 + q < e else e)
        else:
            dls.append(k0 + 1)
    return (min(dls), k0 + q - 1, 1)


def interleaved(tasks, nt, T, chol, nurg, d):
    """A sequential execution the kernel's in-order queues admit: repeatedly run
    the walker's next step, else the urgent queue's head, else the bulk queue's
    head — whichever has every wait condition (and every operand of a chunked
    GEMM) satisfied.  Getting stuck would mean the persistent kernel can
    deadlock; each queue must also be sorted by the (deadline, ready step,
    kind) key that makes the order topological (see build_tasks)."""
    urg, bulk = tasks[:nurg], tasks[nurg:]
    for q in (urg, bulk):
        ks = [key(t, T, d) for t in q]
        assert all(x <= y for x, y in zip(ks, ks[1:])), "queue not in key order"
    cnt = np.zeros((nt, nt), dtype=np.int64)
    out = []
    iu = ib = wk = 0

    def ok(need):
        return all(cnt[tile] >= nd for tile, nd in need)

    while wk < nt or iu < len(urg) or ib < len(bulk):
        if wk < nt and ok(walker_needs(wk, T, nt, chol, d)):
            out.append(("W", wk))
            for tile, rows in walker_signals(wk, T, nt, chol).items():
                cnt[tile] += rows
            wk += 1
            continue
        ran = False
        for qn in ("u", "b"):
            q, i = (urg, iu) if qn == "u" else (bulk, ib)
            if i >= len(q):
                continue
            t = q[i]
            kind, j, k0, qq, r0, r1 = decode(t)
            if not ok(needs(kind, j, k0, qq, r0, r1, T, chol, d, full=True)):
                continue
            out.append(("Q", t))
            for tile, rows in signals(kind, j, k0, r0, r1, T).items():
                cnt[tile] += rows
            if qn == "u":
                iu += 1
            else:
                ib += 1
            ran = True
            break
        assert ran, ("stuck", wk, iu, ib)
    return out


@pytest.mark.parametrize("kernel,n,by,bx", CASES)
def test_task_order_and_coverage(kernel, n, by, bx):
    tasks = _lib.dag_tasks(kernel, n, by, bx)
    assert tasks is not None
    chol = kernel == "cholesky"
    T = _lib.dag_tile(n, by, bx)
    nt = n // T
    d = _lib.dag_chunk_depth(n, by, bx)
    assert not np.any((tasks[:, 0] & 3) == DIAG)  # DIAG belongs to the walker
    cnt = np.zeros((nt, nt), dtype=np.int64)
    nurg = _lib.load().tt_dag_urgent(_lib.KERNEL_IDS[kernel], n, by, bx)
    for what, t in interleaved(tasks, nt, T, chol, nurg, d):
        if what == "W":
            need, sig = walker_needs(t, T, nt, chol, d), walker_signals(t, T, nt, chol)
        else:
            kind, j, k0, q, r0, r1 = decode(t)
            need, sig = needs(kind, j, k0, q, r0, r1, T, chol, d), signals(kind, j, k0, r0, r1, T)
        for (tile, nd) in need:
            assert cnt[tile] >= nd, (what, t, tile, nd, cnt[tile])
        for tile, rows in sig.items():
            i, jj = tile
            if chol:
                assert i >= jj, t
            cnt[tile] += rows
            assert cnt[tile] <= fin(min(i, jj), d, jj) * T, (what, t, tile)
    for i in range(nt):
        for jj in range(nt):
            if chol and jj > i:
                assert cnt[i, jj] == 0
            else:
                assert cnt[i, jj] == fin(min(i, jj), d, jj) * T, (i, jj)


def test_chunked_updates_present():
    """Bulk tiles get their updates d steps at a time (K = d * bx)."""
    for kernel, n, by, bx in (("cholesky", 4000, 250, 50), ("lu", 4000, 160, 50), ("lu", 2000, 200, 40)):
        tasks = _lib.dag_tasks(kernel, n, by, bx)
        d = _lib.dag_chunk_depth(n, by, bx)
        assert d >= 4
        qs = tasks[:, 1] >> 16
        gem = (tasks[:, 0] & 3) == GEMM
        assert np.any(qs[gem] == d) and np.all(qs[gem] <= d)


def run_tasks_numpy(a, tasks, bx, chol, nurg, d):
    a = a.copy()
    T = bx
    nt = a.shape[0] // T

    def trsm_l(k, r0, r1):
        kT = k * T
        dd = a[kT:kT + T, kT:kT + T]
        m = np.tril(dd).T if chol else np.triu(dd)
        a[r0:r1, kT:kT + T] = np.linalg.solve(m.T, a[r0:r1, kT:kT + T].T).T

    def trsm_u(k, j):
        kT, jT = k * T, j * T
        lo = np.tril(a[kT:kT + T, kT:kT + T], -1) + np.eye(T)
        a[kT:kT + T, jT:jT + T] = np.linalg.solve(lo, a[kT:kT + T, jT:jT + T])

    def gemm(k0, q, r0, r1, j):
        jT = j * T
        c = a[r0:r1, jT:jT + T].copy()
        for k in range(k0, k0 + q):  # ascending steps, as the kernel accumulates them
            kT = k * T
            b = a[jT:jT + T, kT:kT + T].T if chol else a[kT:kT + T, jT:jT + T]
            c = c - a[r0:r1, kT:kT + T] @ b
        if chol:
            rows = np.arange(r0, r1)[:, None]
            cols = np.arange(jT, jT + T)[None, :]
            c = np.where(rows >= cols, c, a[r0:r1, jT:jT + T])
        a[r0:r1, jT:jT + T] = c

    for what, t in interleaved(tasks, nt, T, chol, nurg, d):
        if what == "W":  # walker step k
            k = t
            kT = k * T
            if k >= 1:
                gemm(k - 1, 1, kT, kT + T, k)
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
        kind, j, k0, q, r0, r1 = decode(t)
        if kind == TRSM_L:
            trsm_l(k0, r0, r1)
        elif kind == TRSM_U:
            trsm_u(k0, j)
        else:
            gemm(k0, q, r0, r1, j)
    return a


# forced chunk depths (TT_DAG_CHUNK): many tiles per chunk at small n
CHUNKED = [("lu", 120, 40, 8, 3), ("lu", 160, 32, 16, 2), ("lu", 96, 3, 8, 4), ("lu", 200, 50, 10, 5),
           ("cholesky", 128, 16, 8, 4), ("cholesky", 160, 40, 10, 3), ("cholesky", 96, 96, 8, 2),
           ("cholesky", 200, 5, 8, 6), ("lu", 64, 64, 8, 1), ("cholesky", 64, 8, 8, 1)]


@pytest.mark.parametrize("kernel,n,by,bx,d", CHUNKED)
def test_chunked_order_coverage_and_semantics(monkeypatch, kernel, n, by, bx, d):
    monkeypatch.setenv("TT_DAG_CHUNK", str(d))
    assert _lib.dag_chunk_depth(n, by, bx) == d
    test_task_order_and_coverage(kernel, n, by, bx)
    test_task_semantics_reproduce_reference(kernel, n, by, bx)
    tasks = _lib.dag_tasks(kernel, n, by, bx)
    gem = (tasks[:, 0] & 3) == GEMM
    if d > 1 and n // bx > d + 1:
        assert np.any((tasks[gem, 1] >> 16) == d)


@pytest.mark.parametrize("kernel,n,by,bx", [c for c in CASES if c[1] <= 160])
def test_task_semantics_reproduce_reference(kernel, n, by, bx):
    chol = kernel == "cholesky"
    a0 = oracle.gen_spd(n, 5)
    nurg = _lib.load().tt_dag_urgent(_lib.KERNEL_IDS[kernel], n, by, bx)
    out = run_tasks_numpy(a0, _lib.dag_tasks(kernel, n, by, bx), _lib.dag_tile(n, by, bx), chol, nurg,
                          _lib.dag_chunk_depth(n, by, bx))
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


def test_knob_mapping():
    """bx -> tile T and chunk depth, by -> task rows (dag_factor.cu tile_for / region_rows)."""
    assert _lib.dag_tile(2000, 400, 40) == 40                  # 8 <= bx <= 64: T = bx
    assert _lib.dag_tile(2000, 400, 80) == 40                  # wider panels: divisor <= 64 ...
    assert _lib.dag_chunk_depth(2000, 400, 80) == 2            # ... and rank-bx bulk updates
    assert _lib.dag_tile(4000, 250, 250) == 50
    assert 4 <= _lib.dag_chunk_depth(4000, 250, 250) <= 5   # bx/T = 5, capped by shared memory
    assert _lib.dag_tile(4000, 4000, 4000) == 50
    assert _lib.dag_tile(2000, 400, 5) == 10                   # sub-atom panels packed
    assert _lib.dag_tile(4000, 250, 1) == 8
    assert _lib.dag_region_rows(2000, 16, 40) == 128           # small row tiles packed
    assert _lib.dag_region_rows(2000, 50, 40) == 150
    assert _lib.dag_region_rows(2000, 400, 40) == 400
    assert _lib.dag_region_rows(4000, 1, 8) == 640              # narrow tiles: >= 5120 elements
    assert _lib.dag_tasks("cholesky", 4000, 1, 1) is not None
    assert _lib.dag_tasks("lu", 67 * 3, 3, 67) is None         # prime panel > 64: graph schedule
    assert _lib.dag_tile(67 * 3, 3, 67) is None


@pytest.mark.parametrize("kernel,n,by,bx", [("lu", 160, 16, 80), ("cholesky", 160, 5, 160),
                                            ("lu", 96, 96, 4), ("cholesky", 120, 10, 2),
                                            ("lu", 200, 8, 100), ("cholesky", 100, 100, 1)])
def test_mapped_knobs_order_and_semantics(kernel, n, by, bx):
    """Knob settings outside 8..64 run the persistent schedule with the mapped tile."""
    assert _lib.dag_tasks(kernel, n, by, bx) is not None
    test_task_order_and_coverage(kernel, n, by, bx)
    test_task_semantics_reproduce_reference(kernel, n, by, bx)
