"""Generates the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (needs /root/reference and `make -C oracle`):

    python tests/golden/make_golden.py [--full]

Every number here comes from oracle/_ref/libtiletuner_ref.so, i.e. the
reference's own core library compiled from its sources; the literal pins of
kernels_test.cpp:89-92 are copied in as the reference states them.  The
outputs are small (mini/N<=64 arrays as .npz, larger cases as sha256 of the
raw row-major bytes) so they can travel to the GPU box, where
/root/reference does not exist.  --full adds the LARGE/EXTRALARGE hashes
(gen_spd(4000) alone takes ~40 s on one core).
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent
KERNELS = {"lu": 0, "cholesky": 1, "3mm": 2}
SIZES = {
    "lu": {"mini": 64, "small": 400, "large": 2000, "extralarge": 4000},
    "cholesky": {"mini": 64, "small": 400, "large": 2000, "extralarge": 4000},
    "3mm": {"mini": (16, 18, 20, 22, 24), "small": (80, 90, 100, 110, 120),
            "large": (800, 900, 1000, 1100, 1200), "extralarge": (1600, 1800, 2000, 2200, 2400)},
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def ref_spd(R, n, seed):
    a = np.empty((n, n))
    assert R.ref_gen_spd(n, seed, a.ctypes.data_as(ctypes.c_void_p)) == 0
    return a


def ref_3mm(R, dims, seed):
    n, l, m, o, p = dims
    mats = [np.empty(s) for s in ((n, l), (l, m), (m, o), (o, p))]
    assert R.ref_gen_3mm(n, l, m, o, p, seed, *(x.ctypes.data_as(ctypes.c_void_p) for x in mats)) == 0
    return mats


def ref_lu(R, a, by, bx):
    w = a.copy()
    rc = R.ref_lu_factor_inplace(w.ctypes.data_as(ctypes.c_void_p), a.shape[0], a.shape[1], by, bx)
    return rc, w


def ref_chol(R, a, by, bx):
    w = a.copy()
    rc = R.ref_cholesky_factor_inplace(w.ctypes.data_as(ctypes.c_void_p), a.shape[0], a.shape[1],
                                       by, bx)
    return rc, w


def ref_mm3(R, mats, cfg):
    a, b, c, d = mats
    g = np.empty((a.shape[0], d.shape[1]))
    arr = (ctypes.c_int * len(cfg))(*cfg)
    rc = R.ref_mm3_tiled(*(x.ctypes.data_as(ctypes.c_void_p) for x in mats), a.shape[0],
                         a.shape[1], b.shape[1], c.shape[1], d.shape[1],
                         ctypes.cast(arr, ctypes.c_void_p), len(cfg),
                         g.ctypes.data_as(ctypes.c_void_p))
    return rc, g


def divisors(R, n):
    buf = (ctypes.c_int * 256)()
    k = R.ref_divisor_candidates(n, ctypes.cast(buf, ctypes.c_void_p), 256)
    return list(buf[:k])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    args = ap.parse_args()
    R = oracle.ref_lib()
    if R is None:
        sys.exit("oracle/_ref/libtiletuner_ref.so missing: run `make -C oracle` here first")

    arrays, pins = {}, {}
    # kernels_test.cpp:89-92 (literal pins from the reference's own test)
    pins["kernels_test_gen3mm_mini_seed1_a00"] = 0.13387664401253263
    pins["kernels_test_gen3mm_mini_seed1_sumA"] = 141.35364217401869

    for n, seed in ((1, 3), (32, 5), (48, 13), (64, 3), (64, 7), (100, 9)):
        a = ref_spd(R, n, seed)
        arrays[f"spd_{n}_{seed}"] = a
        if n > 1:
            rc, lu = ref_lu(R, a, 1, 1)
            assert rc == 0
            arrays[f"lu_{n}_{seed}"] = lu
            rc, ch = ref_chol(R, a, 1, 1)
            assert rc == 0
            arrays[f"chol_{n}_{seed}"] = ch
    for seed in (1, 4):
        mats = ref_3mm(R, SIZES["3mm"]["mini"], seed)
        for nm, x in zip("abcd", mats):
            arrays[f"mm3mini_{seed}_{nm}"] = x
        rc, g = ref_mm3(R, mats, [1, 1, 1, 1, 1, 1])
        assert rc == 0
        arrays[f"mm3mini_{seed}_g"] = g
    # the 30 random mini configurations of kernels_test.cpp:140-149 use
    # random_config(space, Rng(21)); record them via config_at of the reference
    # space so the GPU test replays exactly those (flat indices from Rng(21)
    # are regenerated in tests with the product's own Rng restatement).

    # hashes of larger generator outputs and factors (config-independent on the CPU)
    hashes = {}
    small = ref_spd(R, 400, 1)
    hashes["spd_400_1"] = sha(small)
    rc, lu = ref_lu(R, small, 400, 50)
    hashes["lu_400_1"] = sha(lu)
    rc, ch = ref_chol(R, small, 80, 40)
    hashes["chol_400_1"] = sha(ch)
    mats = ref_3mm(R, SIZES["3mm"]["small"], 1)
    hashes["mm3_small_inputs_1"] = [sha(x) for x in mats]
    rc, g = ref_mm3(R, mats, [8, 10, 10, 12, 8, 12])
    hashes["mm3_small_g_1"] = sha(g)
    if args.full:
        for n in (2000, 4000):
            a = ref_spd(R, n, 1)
            hashes[f"spd_{n}_1"] = sha(a)
            print("spd", n, "done", flush=True)
            if n == 2000:
                rc, lu = ref_lu(R, a, 400, 50)
                hashes["lu_2000_1"] = sha(lu)
        for name in ("large", "extralarge"):
            mats = ref_3mm(R, SIZES["3mm"][name], 1)
            hashes[f"mm3_{name}_inputs_1"] = [sha(x) for x in mats]

    # search-space pins (space.cpp:10-115), bit-exact host interface
    space = {}
    for n in sorted({1, 2, 9, 64, 400, 800, 900, 1000, 1100, 1200, 1600, 1800, 2000, 2200, 2400,
                     4000, 16, 18, 20, 22, 24}):
        space[f"divisors_{n}"] = divisors(R, n)
    for kname, kid in KERNELS.items():
        for size in SIZES[kname]:
            total = ctypes.c_uint64()
            assert R.ref_space_size(kid, size.encode(), ctypes.byref(total)) == 0
            space[f"size_{kname}_{size}"] = total.value
            nparams = 6 if kname == "3mm" else 2
            samples = []
            for flat in sorted({0, 1, total.value // 2, total.value - 1, (total.value * 7) // 13}):
                cfg = (ctypes.c_int * nparams)()
                assert R.ref_config_at(kid, size.encode(), flat, ctypes.cast(cfg, ctypes.c_void_p)) == 0
                enc = (ctypes.c_double * nparams)()
                assert R.ref_encode(kid, size.encode(), ctypes.cast(cfg, ctypes.c_void_p), nparams,
                                    ctypes.cast(enc, ctypes.c_void_p)) == 0
                samples.append({"flat": flat, "config": list(cfg), "encode": [float(x) for x in enc]})
            space[f"samples_{kname}_{size}"] = samples

    # synthetic-objective tuning traces (harness.cpp:199-265, virtual clock)
    traces = {}
    for kname, size, evals in (("lu", "large", 40), ("cholesky", "extralarge", 40),
                               ("3mm", "mini", 30), ("3mm", "extralarge", 30)):
        for tuner_id, tname in enumerate(("random", "grid", "genetic", "boosted", "bayesopt")):
            flat = (ctypes.c_uint64 * evals)()
            rt = (ctypes.c_double * evals)()
            cnt = ctypes.c_int()
            assert R.ref_run_tuning_synthetic(KERNELS[kname], size.encode(), tuner_id, 7, evals,
                                              ctypes.cast(flat, ctypes.c_void_p),
                                              ctypes.cast(rt, ctypes.c_void_p),
                                              ctypes.byref(cnt)) == 0
            traces[f"{kname}_{size}_{tname}_seed7"] = {
                "flat": list(flat[:cnt.value]), "runtime": [float(x) for x in rt[:cnt.value]]}

    # residual_for at mini (kernels_test.cpp:307-316) and the spot-check probes
    resid = {}
    for kname, cfg in (("lu", [8, 4]), ("cholesky", [16, 2]), ("3mm", [2, 4, 10, 3, 8, 6]),
                       ("lu", [8, 8]), ("cholesky", [8, 8]), ("3mm", [4, 5, 1, 1, 1, 1])):
        out = ctypes.c_double()
        arr = (ctypes.c_int * len(cfg))(*cfg)
        assert R.ref_residual_for(KERNELS[kname], b"mini", 1, ctypes.cast(arr, ctypes.c_void_p),
                                  len(cfg), ctypes.byref(out)) == 0
        resid[f"{kname}_mini_{'x'.join(map(str, cfg))}"] = out.value

    np.savez_compressed(OUT / "golden_arrays.npz", **arrays)
    meta = {"generated_by": "tests/golden/make_golden.py from oracle/_ref/libtiletuner_ref.so",
            "pins": pins, "hashes": hashes, "space": space, "traces": traces,
            "residual_for": resid}
    name = "golden_full.json" if args.full else "golden.json"
    (OUT / name).write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", OUT / "golden_arrays.npz", OUT / name)


if __name__ == "__main__":
    main()
