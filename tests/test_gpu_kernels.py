"""GPU parity tests: the sm_100a path (through the C ABI) against the oracle.

Tolerances (north_star): 3mm max relative error <= 1e-10; LU / Cholesky
max-norm residual ||A - LU|| / ||A||, ||A - LL^T|| / ||A|| <= 1e-12.  Factor
agreement with the reference's own factors: <= 1e-10 relative (acceptance
criterion 3, acceptance_main.cpp:119-168).  Bit-exact where the GPU path is
bit-exact by construction: the device input generators and run-to-run
determinism (kernels_test.cpp:284-296).
"""
import hashlib
import itertools
import random

import numpy as np
import pytest

import oracle
from paper_2309_07235_b200 import (GpuKernelRunner, KernelCase, MeasureProtocol, NumericalError,
                                   cholesky_factor_batch, cholesky_factor_inplace, cholesky_tiled,
                                   lu_factor_batch, lu_factor_inplace, lu_tiled, mm3_tiled)

pytestmark = pytest.mark.gpu

MINI = (16, 18, 20, 22, 24)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


def rel(x, ref):
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300))


# ------------------------------------------------------------------ GEMM core

@pytest.mark.parametrize("bt", [False, True])
def test_gemm_tile_family_vs_torch(gpu_ctx, bt):
    """Every (BM, BN) variant, NN and NT, odd extents, odd (8-byte aligned) origins,
    K tails, and the C = A*B / C -= A*B modes, against torch fp64."""
    import ctypes
    import torch
    torch.manual_seed(0)
    lib = gpu_ctx.lib
    side = torch.cuda.Stream()  # a real (non-legacy) stream shared with the library
    torch.cuda.set_stream(side)
    stream = ctypes.c_void_p(side.cuda_stream)
    cases = [(37, 45, 29), (128, 128, 16), (200, 136, 33), (8, 8, 4), (1, 1, 1), (130, 70, 100),
             (257, 129, 47)]
    regions = [1, 8, 16, 32, 64, 128, 200]
    for (M, N, K), (fy, fx), off in itertools.product(cases, itertools.product(regions, regions),
                                                      (0, 1)):
        if off and (fy, fx) not in ((8, 8), (64, 64), (128, 128), (1, 200)):
            continue
        fy_ = [d for d in divisors(M) if d <= fy][-1]
        fx_ = [d for d in divisors(N) if d <= fx][-1]
        lda = (K + off + 1) // 2 * 2 + 2
        A = torch.rand(M, lda, dtype=torch.float64, device="cuda")[:, off:off + K]
        if bt:
            ldb = (K + off + 1) // 2 * 2
            B = torch.rand(N, ldb, dtype=torch.float64, device="cuda")[:, off:off + K]
            ref_ab = A @ B.T
        else:
            ldb = (N + off + 1) // 2 * 2 + 4
            B = torch.rand(K, ldb, dtype=torch.float64, device="cuda")[:, off:off + N]
            ref_ab = A @ B
        # even ldc -> TMA-prefetched C (beta=1); odd ldc -> plain C loads
        ldc = N + (3 if off else (2 if N % 2 == 0 else 3))
        Cfull = torch.rand(M, ldc, dtype=torch.float64, device="cuda")
        C0 = Cfull[:, :N].clone()
        for alpha, beta in ((1, 0), (-1, 1)):
            Cfull[:, :N] = C0
            rc = lib.tt_dev_gemm(gpu_ctx.handle, ctypes.c_void_p(A.data_ptr()), lda,
                                 ctypes.c_void_p(B.data_ptr()), ldb, int(bt),
                                 ctypes.c_void_p(Cfull.data_ptr()), ldc, M, N, K, fy_, fx_, alpha,
                                 beta, stream)
            gpu_ctx.check(rc)
            want = alpha * ref_ab + (C0 if beta else 0)
            err = (Cfull[:, :N] - want).abs().max().item() / max(want.abs().max().item(), 1e-300)
            assert err <= 1e-13, (M, N, K, fy_, fx_, alpha, beta, off, err)
        assert torch.all(Cfull[:, N:] != 0)  # columns outside the view untouched (rand > 0)
    torch.cuda.set_stream(torch.cuda.default_stream())


# ------------------------------------------------------------------------ 3mm

def test_mm3_mini_random_configs(gpu_ctx, garrays):
    # kernels_test.cpp:128-157 with the north_star tolerance
    mats = [garrays[f"mm3mini_1_{x}"] for x in "abcd"]
    ref = garrays["mm3mini_1_g"]
    rng = random.Random(21)
    ext = (16, 20, 20, 24, 16, 24)
    cfgs = [(1, 1, 1, 1, 1, 1), (16, 20, 20, 24, 16, 24), (4, 5, 1, 1, 1, 1)]
    cfgs += [tuple(rng.choice(divisors(e)) for e in ext) for _ in range(30)]
    for cfg in cfgs:
        g = mm3_tiled(*mats, cfg, ctx=gpu_ctx)
        assert rel(g, ref) <= 1e-10, cfg
        assert oracle.mm3_residual(ref, g) <= 1e-12, cfg
    with pytest.raises(ValueError):
        mm3_tiled(*mats, (3, 1, 1, 1, 1, 1), ctx=gpu_ctx)
    with pytest.raises(ValueError):
        mm3_tiled(*mats, (1, 1), ctx=gpu_ctx)


def test_mm3_hand_examples(gpu_ctx):
    a = np.array([[1.0, 2.0]]); b = np.array([[3.0], [4.0]])
    c = np.array([[5.0]]); d = np.array([[6.0]])
    assert mm3_tiled(a, b, c, d, (1, 1, 1, 1, 1, 1), ctx=gpu_ctx)[0, 0] == 330.0
    i4 = np.eye(4)
    assert np.array_equal(mm3_tiled(i4, i4, i4, i4, (2, 4, 1, 2, 4, 1), ctx=gpu_ctx), i4)
    with pytest.raises(ValueError):
        mm3_tiled(np.zeros((2, 3)), np.zeros((4, 2)), np.zeros((2, 2)), np.zeros((2, 2)),
                  (1, 1, 1, 1, 1, 1), ctx=gpu_ctx)


def test_mm3_determinism(gpu_ctx, garrays):
    mats = [garrays[f"mm3mini_4_{x}"] for x in "abcd"]
    c = (4, 10, 5, 8, 16, 12)
    assert np.array_equal(mm3_tiled(*mats, c, ctx=gpu_ctx), mm3_tiled(*mats, c, ctx=gpu_ctx))
    assert rel(mm3_tiled(*mats, c, ctx=gpu_ctx), garrays["mm3mini_4_g"]) <= 1e-10


@pytest.mark.slow
def test_mm3_large_vs_oracle(gpu_ctx, golden):
    dims = (800, 900, 1000, 1100, 1200)
    runner = GpuKernelRunner(KernelCase("3mm", *dims), gpu_ctx)
    mats = runner.inputs()
    assert [sha(x) for x in mats] == [sha(x) for x in oracle.gen_3mm(dims, 1)]
    ref = oracle.mm3_reference(*mats)
    for cfg in ((25, 25, 25, 30, 25, 30), (80, 200, 200, 240, 80, 240), (800, 1000, 1000, 1200, 800, 1200),
                (16, 125, 125, 120, 32, 120), (1, 2, 5, 3, 4, 8)):
        g = runner.run(cfg)
        assert rel(g, ref) <= 1e-10, cfg
        assert runner.residual(ref) <= 1e-10


# ------------------------------------------------------------------------ LU

def test_lu_sweep_n64(gpu_ctx, garrays):
    # kernels_test.cpp:194-210 / acceptance criterion 3, all 49 configs
    a = garrays["spd_64_3"]
    ref = garrays["lu_64_3"]
    lref, uref = np.tril(ref, -1) + np.eye(64), np.triu(ref)
    scale = max(np.abs(lref).max(), np.abs(uref).max())
    for by, bx in itertools.product(divisors(64), divisors(64)):
        l, u = lu_tiled(a, by, bx, ctx=gpu_ctx)
        packed = np.tril(l, -1) + u
        assert oracle.lu_residual_packed(a, packed) <= 1e-12, (by, bx)
        assert np.abs(l - lref).max() <= 1e-10 * scale and np.abs(u - uref).max() <= 1e-10 * scale


@pytest.mark.parametrize("n,seed", [(100, 9), (48, 13)])
def test_lu_panel_widths(gpu_ctx, garrays, n, seed):
    a = garrays[f"spd_{n}_{seed}"]
    ref = garrays[f"lu_{n}_{seed}"]
    for bx in divisors(n):
        by = divisors(n)[len(divisors(n)) // 2]
        w = a.copy()
        lu_factor_inplace(w, by, bx, ctx=gpu_ctx)
        assert oracle.lu_residual_packed(a, w) <= 1e-12
        assert rel(w, ref) <= 1e-10, (by, bx)


def test_lu_contracts(gpu_ctx):
    a = oracle.gen_spd(32, 5)
    l, u = lu_tiled(a, 8, 4, ctx=gpu_ctx)
    assert (np.diag(l) == 1.0).all()
    assert (np.triu(l, 1) == 0.0).all() and (np.tril(u, -1) == 0.0).all()
    for by, bx in ((3, 4), (8, 0), (64, 4)):
        with pytest.raises(ValueError):
            lu_tiled(a, by, bx, ctx=gpu_ctx)
    with pytest.raises(ValueError):
        lu_factor_inplace(np.zeros((3, 4)), 1, 1, ctx=gpu_ctx)
    # hand example kernels_test.cpp:166-181
    m = np.array([[4.0, 3.0], [6.0, 3.0]])
    lu_factor_inplace(m, 1, 1, ctx=gpu_ctx)
    assert m[1, 0] == 1.5 and m[1, 1] == -1.5 and m[0, 0] == 4.0 and m[0, 1] == 3.0
    # vanishing pivot :186-191 (and one found deeper in the matrix)
    with pytest.raises(NumericalError) as ei:
        lu_factor_inplace(np.array([[0.0, 1.0], [1.0, 0.0]]), 1, 1, ctx=gpu_ctx)
    assert ei.value.index == 0
    z = np.eye(40)
    z[17, 17] = 0.0
    with pytest.raises(NumericalError) as ei:
        lu_factor_inplace(z, 40, 8, ctx=gpu_ctx)
    assert ei.value.index == 17
    i3 = np.eye(3)
    l, u = lu_tiled(i3, 1, 3, ctx=gpu_ctx)
    assert np.array_equal(l, i3) and np.array_equal(u, i3)


@pytest.mark.slow
def test_lu_large_vs_oracle(gpu_ctx):
    n = 2000
    runner = GpuKernelRunner(KernelCase("lu", n), gpu_ctx)
    (a,) = runner.inputs()
    ref = a.copy()
    oracle.lu_factor_inplace(ref, 400, 50)
    for cfg in ((400, 50), (40, 40), (2000, 2000), (125, 125), (200, 16), (1000, 8)):
        w = runner.run(cfg)
        assert runner.residual() <= 1e-12, cfg
        assert rel(w, ref) <= 1e-10, cfg


# ------------------------------------------------------------------ Cholesky

def test_cholesky_sweep_n64(gpu_ctx, garrays):
    a = garrays["spd_64_3"]
    ref = np.tril(garrays["chol_64_3"])
    scale = np.abs(ref).max()
    for by, bx in itertools.product(divisors(64), divisors(64)):
        w = a.copy()
        cholesky_factor_inplace(w, by, bx, ctx=gpu_ctx)
        iu = np.triu_indices(64, 1)
        assert np.array_equal(w[iu], a[iu]), (by, bx)  # upper triangle never written
        l = np.tril(w)
        assert oracle.cholesky_residual(a, w) <= 1e-12, (by, bx)
        assert np.abs(l - ref).max() <= 1e-10 * scale, (by, bx)


@pytest.mark.parametrize("n,seed", [(100, 9), (48, 13)])
def test_cholesky_panel_widths(gpu_ctx, garrays, n, seed):
    a = garrays[f"spd_{n}_{seed}"]
    ref = np.tril(garrays[f"chol_{n}_{seed}"])
    for bx in divisors(n):
        by = divisors(n)[len(divisors(n)) // 3]
        l = cholesky_tiled(a, by, bx, ctx=gpu_ctx)
        assert rel(l, ref) <= 1e-10, (by, bx)
        assert oracle.cholesky_residual(a, l) <= 1e-12


def test_cholesky_contracts(gpu_ctx):
    a = oracle.gen_spd(32, 5)
    l = cholesky_tiled(a, 4, 8, ctx=gpu_ctx)
    assert (np.diag(l) > 0).all() and (np.triu(l, 1) == 0).all()
    for by, bx in ((5, 8), (4, -1)):
        with pytest.raises(ValueError):
            cholesky_tiled(a, by, bx, ctx=gpu_ctx)
    m = np.array([[4.0, 2.0], [2.0, 3.0]])
    cholesky_factor_inplace(m, 1, 1, ctx=gpu_ctx)
    assert m[0, 0] == 2.0 and m[1, 0] == 1.0 and m[1, 1] == np.sqrt(2.0) and m[0, 1] == 2.0
    with pytest.raises(NumericalError) as ei:
        cholesky_factor_inplace(np.array([[1.0, 2.0], [2.0, 1.0]]), 1, 1, ctx=gpu_ctx)
    assert ei.value.index == 1


def test_determinism(gpu_ctx):
    # kernels_test.cpp:284-296
    a = oracle.gen_spd(48, 13)
    l1, u1 = lu_tiled(a, 8, 6, ctx=gpu_ctx)
    l2, u2 = lu_tiled(a, 8, 6, ctx=gpu_ctx)
    assert np.array_equal(l1, l2) and np.array_equal(u1, u2)
    assert np.array_equal(cholesky_tiled(a, 8, 6, ctx=gpu_ctx), cholesky_tiled(a, 8, 6, ctx=gpu_ctx))


def test_batch_api_matches_one_shot(gpu_ctx):
    """The pipelined batch entry points give, per matrix, exactly the one-shot
    drop-in's result (same schedule), on pinned and pageable buffers, and report
    the first failing matrix / column like lu_factor_inplace."""
    import torch
    for n, by, bx in ((200, 40, 20), (96, 96, 8), (60, 12, 5)):
        mats = [oracle.gen_spd(n, s) for s in range(5)]
        one = [m.copy() for m in mats]
        for m in one:
            lu_factor_inplace(m, by, bx, ctx=gpu_ctx)
        pinned = [torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy() for _ in mats]
        for p, m in zip(pinned, mats):
            p[...] = m
        lu_factor_batch(pinned, by, bx, ctx=gpu_ctx)
        for p, o in zip(pinned, one):
            assert np.array_equal(p, o), (n, by, bx)
        ch = [m.copy() for m in mats]
        cholesky_factor_batch(ch, by, bx, ctx=gpu_ctx)
        for c, m in zip(ch, mats):
            ref = m.copy()
            cholesky_factor_inplace(ref, by, bx, ctx=gpu_ctx)
            assert np.array_equal(c, ref)
    lu_factor_batch([], 1, 1, ctx=gpu_ctx)
    bad = [oracle.gen_spd(40, 1), np.eye(40), oracle.gen_spd(40, 2)]
    bad[1][17, 17] = 0.0
    with pytest.raises(NumericalError) as ei:
        lu_factor_batch(bad, 40, 8, ctx=gpu_ctx)
    assert ei.value.index == 17
    with pytest.raises(ValueError):
        lu_factor_batch([np.eye(8), np.eye(9)], 1, 1, ctx=gpu_ctx)


@pytest.mark.slow
def test_cholesky_xl_device_residual(gpu_ctx, golden):
    n = 4000
    runner = GpuKernelRunner(KernelCase("cholesky", n), gpu_ctx)
    full = golden.get("hashes", {})
    (a,) = runner.inputs()
    if "spd_4000_1" in full:
        assert sha(a) == full["spd_4000_1"]
    for cfg in ((80, 32), (250, 125), (160, 160)):
        w = runner.run(cfg)
        assert runner.residual() <= 1e-12, cfg
        iu = np.triu_indices(n, 1)
        assert np.array_equal(w[iu], a[iu])


# ------------------------------------------------------- generators + harness

def test_device_generators_bitwise(gpu_ctx, garrays, golden):
    for n, seed in ((64, 3), (100, 9), (1, 3)):
        r = GpuKernelRunner(KernelCase("lu", n, seed=seed), gpu_ctx)
        assert np.array_equal(r.inputs()[0], garrays[f"spd_{n}_{seed}"])
    r = GpuKernelRunner(KernelCase("cholesky", 400, seed=1), gpu_ctx)
    assert sha(r.inputs()[0]) == golden["hashes"]["spd_400_1"]
    r = GpuKernelRunner(KernelCase("3mm", *MINI, seed=1), gpu_ctx)
    for x, name in zip(r.inputs(), "abcd"):
        assert np.array_equal(x, garrays[f"mm3mini_1_{name}"])
    r = GpuKernelRunner(KernelCase("3mm", 80, 90, 100, 110, 120, seed=1), gpu_ctx)
    assert [sha(x) for x in r.inputs()] == golden["hashes"]["mm3_small_inputs_1"]


def test_spot_check_probes(gpu_ctx):
    # harness.cpp:147-156: mini case at config_at(space, size/2), residual <= 1e-10
    r = GpuKernelRunner(KernelCase("lu", 64), gpu_ctx)
    r.run((8, 8))
    assert r.residual() <= 1e-12
    r = GpuKernelRunner(KernelCase("cholesky", 64), gpu_ctx)
    r.run((8, 8))
    assert r.residual() <= 1e-12
    r = GpuKernelRunner(KernelCase("3mm", *MINI), gpu_ctx)
    g = r.run((4, 5, 1, 1, 1, 1))
    ref = oracle.mm3_reference(*oracle.gen_3mm(MINI, 1))
    assert oracle.mm3_residual(ref, g) <= 1e-10


def test_measure_semantics(gpu_ctx):
    # harness_test.cpp:91-107
    r = GpuKernelRunner(KernelCase("lu", 64), gpu_ctx)
    t1 = r.measure((1, 1), MeasureProtocol(0, 1))
    t8 = r.measure((8, 8), MeasureProtocol(0, 1))
    assert t1 > 0 and t8 > 0
    with pytest.raises(ValueError):
        r.measure((1, 1), MeasureProtocol(0, 0))
    with pytest.raises(ValueError):
        r.measure((3, 3))
    s = r.samples((8, 8), 1, 5)
    assert len(s) == 5 and min(s) > 0
    med = r.measure((8, 8), MeasureProtocol(1, 3, "median"))
    assert med > 0
    # the knobs change the schedule: 1x1 panels are far slower than 64x64
    big = GpuKernelRunner(KernelCase("lu", 400), gpu_ctx)
    slow = big.measure((1, 1), MeasureProtocol(1, 3, "min"))
    fast = big.measure((400, 50), MeasureProtocol(1, 3, "min"))
    assert slow > 2 * fast
    assert gpu_ctx.cache_size >= 3


# ------------------------------------------------- scaled 3mm + measured tuning

def test_scaled_mm3_single_gpu_freivalds():
    from paper_2309_07235_b200.sharded import run_scaled
    out = run_scaled(n=2048, steps=1, warmup=0, kblocks=8)
    assert out["freivalds_rel"] <= 1e-10
    assert out["tflops"] > 0


def test_measured_tuning_loop(gpu_ctx):
    """run_tuning with the GPU objective (spot check, device inputs, BO) on cuda:0."""
    from paper_2309_07235_b200 import tuning
    recs, total = tuning.run_tuning_measured("bayesopt", "lu", "small", 5, 14, devices=(0,),
                                             warmups=1, reps=3)
    assert len(recs) == 14 and len({r.flat for r in recs}) == 14
    assert all(r.runtime_s and r.runtime_s > 0 for r in recs)
    best = float("inf")
    for r in recs:
        best = min(best, r.runtime_s)
        assert r.best_so_far_s == best
    assert [r.elapsed_s for r in recs] == sorted(r.elapsed_s for r in recs)
    # two evaluator slots on the same device exercise the asynchronous dispatcher
    recs2, _ = tuning.run_tuning_measured("bayesopt", "3mm", "small", 5, 16, devices=(0, 0),
                                          warmups=0, reps=1)
    assert len(recs2) == 16 and {r.worker for r in recs2} == {0, 1}
