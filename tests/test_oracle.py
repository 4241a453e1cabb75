"""CPU tests: the oracle (oracle/tt_oracle.c) pinned against the reference.

Pins come from tests/golden/ (generated from the unmodified reference by
tests/golden/make_golden.py) and from the literal known-answer tests of
/root/reference/proj/tests/kernels_test.cpp.  These run without a GPU.
"""
import hashlib
import itertools
import random

import numpy as np
import pytest

import oracle


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def divisors(n):
    return [d for d in range(1, n + 1) if n % d == 0]


MINI = (16, 18, 20, 22, 24)


def test_gen_3mm_golden_checksum(golden):
    # kernels_test.cpp:74-97
    a, b, c, d = oracle.gen_3mm(MINI, 1)
    assert a.shape == (16, 18) and b.shape == (18, 20) and c.shape == (20, 22) and d.shape == (22, 24)
    assert a[0, 0] == golden["pins"]["kernels_test_gen3mm_mini_seed1_a00"] == 0.13387664401253263
    assert abs(a.sum() - 141.35364217401869) <= 1e-15 * 141.35364217401869 * 10
    a2, _, _, d2 = oracle.gen_3mm(MINI, 1)
    assert np.array_equal(a, a2) and np.array_equal(d, d2)
    with pytest.raises(ValueError):
        oracle.gen_3mm((16, 18, 20, 0, 24), 1)


@pytest.mark.parametrize("n,seed", [(1, 3), (32, 5), (48, 13), (64, 3), (64, 7), (100, 9)])
def test_gen_spd_bitwise(garrays, n, seed):
    a = oracle.gen_spd(n, seed)
    assert np.array_equal(a, garrays[f"spd_{n}_{seed}"])
    assert np.array_equal(a, a.T)  # kernels.cpp:44-51 bit-exact symmetry
    assert (np.diag(a) >= n).all()


def test_gen_spd_hash_400(golden):
    assert sha(oracle.gen_spd(400, 1)) == golden["hashes"]["spd_400_1"]


@pytest.mark.parametrize("n,seed", [(32, 5), (48, 13), (64, 3), (64, 7), (100, 9)])
def test_lu_config_independent_bitwise(garrays, n, seed):
    """Every tiled config equals the reference's factor bitwise."""
    a = garrays[f"spd_{n}_{seed}"]
    want = garrays[f"lu_{n}_{seed}"]
    divs = divisors(n)
    pairs = list(itertools.product(divs, divs)) if n == 64 else [(divs[len(divs) // 2], d) for d in divs]
    for by, bx in pairs:
        w = a.copy()
        oracle.lu_factor_inplace(w, by, bx)
        assert np.array_equal(w, want), (by, bx)


@pytest.mark.parametrize("n,seed", [(32, 5), (48, 13), (64, 3), (64, 7), (100, 9)])
def test_cholesky_config_independent_bitwise(garrays, n, seed):
    a = garrays[f"spd_{n}_{seed}"]
    want = garrays[f"chol_{n}_{seed}"]
    divs = divisors(n)
    pairs = list(itertools.product(divs, divs)) if n == 64 else [(divs[len(divs) // 2], d) for d in divs]
    for by, bx in pairs:
        w = a.copy()
        oracle.cholesky_factor_inplace(w, by, bx)
        assert np.array_equal(w, want), (by, bx)
        iu = np.triu_indices(n, 1)
        assert np.array_equal(w[iu], a[iu])  # upper triangle never written


def test_mm3_tiled_random_configs_bitwise(garrays):
    # kernels_test.cpp:128-157: every tiled config equals the reference
    mats = [garrays[f"mm3mini_1_{x}"] for x in "abcd"]
    want = garrays["mm3mini_1_g"]
    assert np.array_equal(oracle.mm3_reference(*mats), want)
    rng = random.Random(21)
    ext = (16, 20, 20, 24, 16, 24)
    cfgs = [(1, 1, 1, 1, 1, 1), (16, 20, 20, 24, 16, 24)]
    cfgs += [tuple(rng.choice(divisors(e)) for e in ext) for _ in range(30)]
    for cfg in cfgs:
        assert np.array_equal(oracle.mm3_tiled(*mats, list(cfg)), want), cfg
    with pytest.raises(ValueError):
        oracle.mm3_tiled(*mats, [3, 1, 1, 1, 1, 1])
    with pytest.raises(ValueError):
        oracle.mm3_tiled(*mats, [1, 1])


def test_hand_examples():
    # kernels_test.cpp:99-121
    a = np.array([[1.0, 2.0]]); b = np.array([[3.0], [4.0]])
    c = np.array([[5.0]]); d = np.array([[6.0]])
    assert oracle.mm3_reference(a, b, c, d)[0, 0] == 330.0
    i4 = np.eye(4)
    assert np.array_equal(oracle.mm3_reference(i4, i4, i4, i4), i4)
    # :166-181 hand-eliminated 2x2
    m = np.array([[4.0, 3.0], [6.0, 3.0]])
    oracle.lu_factor_inplace(m, 1, 1)
    assert m[1, 0] == 1.5 and m[0, 0] == 4.0 and m[0, 1] == 3.0 and m[1, 1] == -1.5
    # :232-243 closed-form 2x2
    m = np.array([[4.0, 2.0], [2.0, 3.0]])
    oracle.cholesky_factor_inplace(m, 1, 1)
    assert m[0, 0] == 2.0 and m[1, 0] == 1.0 and m[1, 1] == np.sqrt(2.0) and m[0, 1] == 2.0
    # :186-191 vanishing pivot, :248-255 non-SPD
    with pytest.raises(oracle.OracleNumericalError):
        oracle.lu_factor_inplace(np.array([[0.0, 1.0], [1.0, 0.0]]), 1, 1)
    with pytest.raises(oracle.OracleNumericalError):
        oracle.cholesky_factor_inplace(np.array([[1.0, 2.0], [2.0, 1.0]]), 1, 1)


def test_error_contracts():
    # kernels_test.cpp:212-225, 273-282
    a = oracle.gen_spd(32, 5)
    for by, bx in ((3, 4), (8, 0), (64, 4)):
        with pytest.raises(ValueError):
            oracle.lu_factor_inplace(a.copy(), by, bx)
    for by, bx in ((5, 8), (4, -1)):
        with pytest.raises(ValueError):
            oracle.cholesky_factor_inplace(a.copy(), by, bx)


def test_residuals(golden, garrays):
    a = garrays["spd_64_3"]
    assert oracle.lu_residual_packed(a, garrays["lu_64_3"]) <= 1e-10
    assert oracle.cholesky_residual(a, garrays["chol_64_3"]) <= 1e-10
    # residual_for(mini, {8,4}) of the reference, recomputed by the oracle
    a1 = oracle.gen_spd(64, 1)
    w = a1.copy()
    oracle.lu_factor_inplace(w, 8, 4)
    assert oracle.lu_residual_packed(a1, w) == golden["residual_for"]["lu_mini_8x4"]
    w = a1.copy()
    oracle.cholesky_factor_inplace(w, 16, 2)
    assert oracle.cholesky_residual(a1, w) == golden["residual_for"]["cholesky_mini_16x2"]
    i5 = np.eye(5)
    w = i5.copy()
    oracle.lu_factor_inplace(w, 1, 1)
    assert oracle.lu_residual_packed(i5, w) == 0.0


def test_small_size_hashes(golden):
    a = oracle.gen_spd(400, 1)
    w = a.copy()
    oracle.lu_factor_inplace(w, 400, 50)
    assert sha(w) == golden["hashes"]["lu_400_1"]
    w = a.copy()
    oracle.cholesky_factor_inplace(w, 80, 40)
    assert sha(w) == golden["hashes"]["chol_400_1"]
    mats = oracle.gen_3mm((80, 90, 100, 110, 120), 1)
    assert [sha(x) for x in mats] == golden["hashes"]["mm3_small_inputs_1"]
    assert sha(oracle.mm3_tiled(*mats, [8, 10, 10, 12, 8, 12])) == golden["hashes"]["mm3_small_g_1"]


@pytest.mark.skipif(oracle.ref_lib() is None, reason="reference library not built here")
def test_oracle_vs_reference_library_random_inputs():
    """Direct cross-check against the compiled reference (build container only)."""
    import ctypes
    R = oracle.ref_lib()
    rng = np.random.default_rng(0)
    for n in (7, 30, 96):
        a = rng.random((n, n)) + n * np.eye(n)
        a = a @ a.T
        for by, bx in ((1, 1), (divisors(n)[1], divisors(n)[-2]), (n, n)):
            w1 = a.copy(); w2 = a.copy()
            oracle.lu_factor_inplace(w1, by, bx)
            assert R.ref_lu_factor_inplace(w2.ctypes.data_as(ctypes.c_void_p), n, n, by, bx) == 0
            assert np.array_equal(w1, w2)
            w1 = a.copy(); w2 = a.copy()
            oracle.cholesky_factor_inplace(w1, by, bx)
            assert R.ref_cholesky_factor_inplace(w2.ctypes.data_as(ctypes.c_void_p), n, n, by, bx) == 0
            assert np.array_equal(w1, w2)
