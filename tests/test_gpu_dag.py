"""GPU parity of the persistent tile-DAG schedule (dag_factor.cu: walker CTA +
urgent/bulk queues) against the oracle.

Covers what the reference's kernel tests pin (kernels_test.cpp:159-316), on
every knob setting (all run the persistent kernel; panel widths outside 8..64
through the mapped tile, dag_factor.cu tile_for): parity over a
knob sweep, failure predicates at chosen columns (vanishing pivot, non-positive
diagonal — NaN passes), bitwise determinism under the dynamic task schedule,
the upper triangle of Cholesky never written, the walker-only (n = bx) and
two-step cases, and agreement with the launch-graph schedule.
"""
import itertools

import numpy as np
import pytest

import oracle
from paper_2309_07235_b200 import NumericalError, _lib, cholesky_factor_inplace, cholesky_tiled, lu_factor_inplace

pytestmark = pytest.mark.gpu


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


def on_dag(kernel, n, by, bx):
    return _lib.dag_tasks(kernel, n, by, bx) is not None


def rel(x, ref):
    return np.abs(x - ref).max() / np.abs(ref).max()


N = 200
BXS = divisors(N)  # every panel width runs the persistent kernel (mapped tile outside 8..64)
BYS = [1, 5, 8, 25, 40, 100, 200]


@pytest.fixture(scope="module")
def spd():
    return oracle.gen_spd(N, 21)


@pytest.fixture(scope="module")
def lu_ref(spd):
    r = spd.copy()
    oracle.lu_factor_inplace(r, N, N)
    return r


@pytest.fixture(scope="module")
def chol_ref(spd):
    r = spd.copy()
    oracle.cholesky_factor_inplace(r, N, N)
    return np.tril(r)


def test_lu_knob_sweep(gpu_ctx, spd, lu_ref):
    for by, bx in itertools.product(BYS, BXS):
        assert on_dag("lu", N, by, bx), (by, bx)
        w = spd.copy()
        lu_factor_inplace(w, by, bx, ctx=gpu_ctx)
        assert oracle.lu_residual_packed(spd, w) <= 1e-12, (by, bx)
        assert rel(w, lu_ref) <= 1e-10, (by, bx)


def test_cholesky_knob_sweep(gpu_ctx, spd, chol_ref):
    iu = np.triu_indices(N, 1)
    for by, bx in itertools.product(BYS, BXS):
        w = spd.copy()
        cholesky_factor_inplace(w, by, bx, ctx=gpu_ctx)
        assert np.array_equal(w[iu], spd[iu]), (by, bx)  # upper triangle never written
        assert oracle.cholesky_residual(spd, w) <= 1e-12, (by, bx)
        assert rel(np.tril(w), chol_ref) <= 1e-10, (by, bx)


@pytest.mark.parametrize("n,bx", [(64, 64), (40, 40), (80, 40), (16, 8)])
def test_walker_edge_shapes(gpu_ctx, n, bx):
    a = oracle.gen_spd(n, 3)
    for by in (1, bx, n):
        w = a.copy()
        lu_factor_inplace(w, by, bx, ctx=gpu_ctx)
        assert oracle.lu_residual_packed(a, w) <= 1e-12, (n, by, bx)
        c = a.copy()
        cholesky_factor_inplace(c, by, bx, ctx=gpu_ctx)
        assert oracle.cholesky_residual(a, c) <= 1e-12, (n, by, bx)


def _singular_at(n, c, chol):
    """SPD matrix whose step-c pivot is exactly 0 (LU) / -1 (Cholesky): row and
    column c decoupled from the leading block."""
    a = oracle.gen_spd(n, 7)
    a[c, :] = 0.0
    a[:, c] = 0.0
    a[c, c] = -1.0 if chol else 0.0
    if not chol:
        a[c, c + 1:] = 1.0  # keep U's row non-trivial after the failing pivot
    return a


@pytest.mark.parametrize("c", [0, 37, 40, 93, 199])
@pytest.mark.parametrize("by,bx", [(40, 40), (8, 8), (200, 25), (100, 50)])
def test_failure_column_matches_oracle(gpu_ctx, c, by, bx):
    for chol in (False, True):
        a = _singular_at(N, c, chol)
        ref = a.copy()
        with pytest.raises(oracle.OracleNumericalError) as oe:
            (oracle.cholesky_factor_inplace if chol else oracle.lu_factor_inplace)(ref, by, bx)
        want = int(str(oe.value).rsplit(" ", 1)[1])
        assert want == c
        with pytest.raises(NumericalError) as ge:
            (cholesky_factor_inplace if chol else lu_factor_inplace)(a.copy(), by, bx, ctx=gpu_ctx)
        assert ge.value.index == want, (chol, c, by, bx)
    # the context stays usable after an aborted schedule
    w = oracle.gen_spd(N, 1)
    lu_factor_inplace(w, by, bx, ctx=gpu_ctx)


def test_nan_passes_failure_checks(gpu_ctx):
    # comparisons with NaN are false: the reference raises nothing
    a = oracle.gen_spd(N, 2)
    a[50, 50] = np.nan
    w = a.copy()
    lu_factor_inplace(w, 40, 40, ctx=gpu_ctx)
    assert np.isnan(w).any()
    c = a.copy()
    cholesky_factor_inplace(c, 40, 40, ctx=gpu_ctx)
    assert np.isnan(np.tril(c)).any()


def test_bitwise_determinism_dynamic_schedule(gpu_ctx):
    # kernels_test.cpp:284-296 under the dynamic task queue: the arithmetic per
    # element is fixed by the task list, not by which CTA ran a task or when
    a = oracle.gen_spd(400, 4)
    for by, bx in ((40, 40), (100, 25), (400, 50), (8, 8)):
        outs = []
        for _ in range(3):
            w = a.copy()
            lu_factor_inplace(w, by, bx, ctx=gpu_ctx)
            outs.append(w)
        assert all(np.array_equal(outs[0], o) for o in outs[1:]), (by, bx)
        outs = []
        for _ in range(3):
            w = a.copy()
            cholesky_factor_inplace(w, by, bx, ctx=gpu_ctx)
            outs.append(w)
        assert all(np.array_equal(outs[0], o) for o in outs[1:]), (by, bx)


@pytest.mark.parametrize("by,bx", [(40, 40), (40, 100), (8, 200), (50, 4)])
def test_graph_and_dag_schedules_agree(gpu_ctx, monkeypatch, by, bx):
    """The same knob setting through both schedules (TT_FACTOR_SCHEDULE=graph
    forces the launch-per-kernel graph), both against the oracle; panel widths
    outside 8..64 run the persistent schedule with the mapped tile."""
    a = oracle.gen_spd(N, 5)
    ref = a.copy()
    oracle.lu_factor_inplace(ref, N, N)
    assert on_dag("lu", N, by, bx)
    w_dag = a.copy()
    lu_factor_inplace(w_dag, by, bx, ctx=gpu_ctx)
    monkeypatch.setenv("TT_FACTOR_SCHEDULE", "graph")
    w_graph = a.copy()
    lu_factor_inplace(w_graph, by, bx, ctx=gpu_ctx)
    l_graph = cholesky_tiled(a, by, bx, ctx=gpu_ctx)
    monkeypatch.delenv("TT_FACTOR_SCHEDULE")
    l_dag = cholesky_tiled(a, by, bx, ctx=gpu_ctx)
    assert rel(w_dag, ref) <= 1e-10 and rel(w_graph, ref) <= 1e-10
    assert rel(w_dag, w_graph) <= 1e-10
    assert oracle.cholesky_residual(a, l_dag) <= 1e-12
    assert oracle.cholesky_residual(a, l_graph) <= 1e-12
