"""tiletuner-gpu CLI: the reference CLI's spaces | verify |
tune front end with device flags, trace format v1 (the reference's, byte for
byte) and v2 (device + schedule variant per record).

CPU tests pin the v1 bytes against the unmodified reference's run_tuning +
render_trace (oracle/_ref, persist.cpp:97-127), the reference parser reading
our traces (persist.cpp:129-222), `spaces` against the reference space, and
the exit-code contract (0 / 1 domain / 2 usage, tools/tiletuner.cpp:276-298).
GPU tests run verify and a measured tune on the B200.
"""
import ctypes
import os
import subprocess
from pathlib import Path

import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2309_07235_b200" / "tiletuner-gpu"
KERNELS = {"lu": 0, "cholesky": 1, "3mm": 2}
TUNERS = {"random": 0, "grid": 1, "bayesopt": 4}


def run(*args, env=None, check_rc=None):
    e = dict(os.environ)
    if env:
        e.update(env)
    p = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, env=e,
                       timeout=600)
    if check_rc is not None:
        assert p.returncode == check_rc, (p.returncode, p.stdout, p.stderr)
    return p


REF_TRACE = ROOT / "oracle" / "_ref" / "ref_trace"


def ref_trace(kernel, size, tuner, seed, evals):
    """The unmodified reference's run_tuning + render_trace (created = 0)."""
    p = subprocess.run([str(REF_TRACE), "render", kernel, size, tuner, str(seed), str(evals)],
                       capture_output=True, text=True, timeout=600, check=True)
    return p.stdout


def ref_parse_best(path):
    """The reference's read_trace + best_of on a file: (records, config string, best)."""
    p = subprocess.run([str(REF_TRACE), "parse", str(path)], capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr
    n, cfg, best = p.stdout.split()
    return int(n), cfg, float(best)


needs_ref = pytest.mark.skipif(oracle.ref_lib() is None or not REF_TRACE.exists(),
                               reason="reference core not built here")


def test_cli_built():
    assert CLI.exists(), "build first: python -c 'import __graft_entry__ as g; g.build()'"


@needs_ref
@pytest.mark.parametrize("kernel,size", [("lu", "large"), ("cholesky", "extralarge"),
                                         ("3mm", "mini"), ("3mm", "large")])
def test_spaces_match_reference(kernel, size):
    out = run("spaces", kernel, size, check_rc=0).stdout.splitlines()
    R = oracle.ref_lib()
    total = ctypes.c_uint64()
    assert R.ref_space_size(KERNELS[kernel], size.encode(), ctypes.byref(total)) == 0
    assert out[-1] == f"total_size: {total.value}"
    for line in out[:-1]:  # "P<i> <extent> <k>_candidates: c0,c1,..."
        name, extent, count, cands = line.split(" ", 3)
        got = [int(x) for x in cands.split(",")]
        buf = (ctypes.c_int * 256)()
        k = R.ref_divisor_candidates(int(extent), buf, 256)
        assert got == list(buf[:k]) and count == f"{k}_candidates:", line


@needs_ref
@pytest.mark.parametrize("kernel,size,tuner,seed,evals", [
    ("lu", "large", "bayesopt", 42, 25), ("cholesky", "extralarge", "random", 7, 20),
    ("3mm", "large", "bayesopt", 3, 24), ("3mm", "mini", "grid", 0, 12), ("lu", "mini", "grid", 5, 30)])
def test_synthetic_v1_trace_equals_reference_bytes(tmp_path, kernel, size, tuner, seed, evals):
    out = tmp_path / "t.trace"
    p = run("tune", kernel, size, "--tuner", tuner, "--seed", seed, "--max-evals", evals,
            "--synthetic", "--reproducible", "--trace-format", "v1", "--out", out, check_rc=0)
    assert out.read_text() == ref_trace(kernel, size, tuner, seed, evals)
    n, cfg, best = ref_parse_best(out)  # the reference parser reads it
    assert n == evals and f"best_config: {cfg}" in p.stdout


@needs_ref
def test_v2_trace_reads_back_and_converts_to_reference_v1(tmp_path):
    out = tmp_path / "t2.trace"
    run("tune", "3mm", "large", "--tuner", "bayesopt", "--seed", 9, "--max-evals", 15, "--synthetic",
        "--reproducible", "--batch", 1, "--out", out, check_rc=0)
    text = out.read_text()
    assert text.startswith("# tiletuner-trace v2\n")
    assert "# columns: eval_index,config,runtime_s,elapsed_s,best_so_far_s,status,device,variant" in text
    show = run("show", out, "--as-v1", check_rc=0).stdout
    v1 = show[show.index("# tiletuner-trace v1"):]
    assert v1 == ref_trace("3mm", "large", "bayesopt", 9, 15)
    assert "version: v2" in show and "evals: 15" in show


def test_v1_reader_accepts_reference_format_and_rejects_bad(tmp_path):
    good = tmp_path / "g.trace"
    run("tune", "lu", "mini", "--synthetic", "--reproducible", "--trace-format", "v1",
        "--max-evals", 6, "--out", good, check_rc=0)
    s = run("show", good, check_rc=0).stdout
    assert "version: v1" in s and "evals: 6" in s
    bad = tmp_path / "b.trace"
    bad.write_text(good.read_text().replace("# seed:", "# sneed:"))
    r = run("show", bad)
    assert r.returncode == 1 and "unknown header key" in r.stderr
    bad.write_text(good.read_text().replace(",ok\n", ",maybe\n", 1))
    assert run("show", bad).returncode == 1
    bad.write_text("# tiletuner-trace v3\n")
    assert run("show", bad).returncode == 1


@pytest.mark.parametrize("name,evals,best", [
    ("tune_lu_large_bo60_r01c.trace", 60, "P0=200|P1=40"),
    ("tune_chol_xl_bo60_r01c.trace", 60, "P0=250|P1=50"),
    ("tune_3mm_xl_bo200_r01c.trace", 200, None)])
def test_reads_measured_v2_traces_from_the_gpu(name, evals, best):
    """The committed traces of measured GPU runs (profiles/) parse back: v2
    header, device and schedule-variant columns, best record."""
    path = ROOT / "profiles" / name
    out = run("show", path, check_rc=0).stdout
    assert "version: v2" in out and f"evals: {evals}" in out and "devices_used: 0" in out
    if best:
        assert f"best_config: {best}" in out
    variants = {l.split(",")[7] for l in path.read_text().splitlines() if not l.startswith("#")}
    assert variants <= {"dag", "graph", "dgemm"} and variants


def test_synthetic_batch_and_reproducible(tmp_path):
    a, b = tmp_path / "a.trace", tmp_path / "b.trace"
    for f in (a, b):
        run("tune", "3mm", "mini", "--synthetic", "--reproducible", "--batch", 4, "--max-evals", 16,
            "--out", f, check_rc=0)
    assert a.read_bytes() == b.read_bytes()  # byte-stable --reproducible
    assert "# batch: 4" in a.read_text()


def test_exit_codes(tmp_path):
    assert run().returncode == 2
    assert run("bogus").returncode == 2
    assert run("spaces", "qr", "large").returncode == 2
    assert run("spaces", "lu", "huge").returncode == 2
    assert run("tune", "lu", "mini", "--max-evals", "x").returncode == 2
    assert run("tune", "lu", "mini", "--frobnicate").returncode == 2
    assert run("tune", "lu", "mini", "--synthetic", "--tuner", "genetic").returncode == 1
    assert run("tune", "lu", "mini", "--synthetic", "--max-evals", 0).returncode == 1
    assert run("--help").returncode == 0


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_verify_on_gpu():
    for kernel, size, samples in (("lu", "mini", 6), ("cholesky", "mini", 6), ("3mm", "mini", 6),
                                  ("lu", "small", 3)):
        p = run("verify", kernel, size, "--samples", samples, check_rc=0)
        lines = p.stdout.splitlines()
        assert len(lines) == samples and all(l.endswith("PASS") for l in lines), p.stdout
    p = run("verify", "lu", "mini", "--samples", 2, env={"TILETUNER_TEST_CORRUPT": "1"})
    assert p.returncode == 1 and "FAIL" in p.stdout


@pytest.mark.gpu
def test_measured_tune_on_gpu(tmp_path):
    out = tmp_path / "m.trace"
    p = run("tune", "lu", "small", "--tuner", "bayesopt", "--max-evals", 8, "--gpus", 1,
            "--out", out, env={"TILETUNER_REPS": "2"}, check_rc=0)
    text = out.read_text()
    assert "# objective: measured" in text and "# devices: 0" in text and "# repetitions: 2" in text
    recs = [l.split(",") for l in text.splitlines() if not l.startswith("#")]
    assert len(recs) == 8 and all(r[6] == "0" and r[7] in ("dag", "graph") for r in recs)
    assert "best_runtime_s:" in p.stdout


@pytest.mark.gpu
def test_measured_tune_two_workers_trace_invariants(tmp_path):
    """--batch 2 on one GPU: two concurrent evaluators (two contexts on device 0);
    records in completion order keep elapsed non-decreasing and best_so_far an
    exact prefix-min (harness_test.cpp:133-153), and both workers report."""
    out = tmp_path / "b2.trace"
    run("tune", "3mm", "small", "--tuner", "random", "--max-evals", 12, "--gpus", 1, "--batch", 2,
        "--seed", 5, "--out", out, env={"TILETUNER_REPS": "1"}, check_rc=0)
    text = out.read_text()
    assert "# batch: 2" in text and "# devices: 0,0" in text
    recs = [l.split(",") for l in text.splitlines() if not l.startswith("#")]
    assert len(recs) == 12 and all(r[7] == "dgemm" for r in recs)
    el = [float(r[3]) for r in recs]
    assert el == sorted(el)
    best, prefix = float("inf"), []
    for r in recs:
        if r[5] == "ok":
            best = min(best, float(r[2]))
        prefix.append(best)
    assert [float(r[4]) for r in recs] == prefix
    assert sorted(int(r[0]) for r in recs) == list(range(12))


@pytest.mark.gpu
def test_two_workers_one_gpu_persistent_factorisations(tmp_path):
    """Two evaluators on one GPU run persistent (spin-waiting) factorisation
    kernels concurrently: cooperative launches keep each grid co-resident, so
    neither waits on CTAs that cannot be scheduled (no watchdog abort)."""
    out = tmp_path / "lu2.trace"
    run("tune", "lu", "small", "--tuner", "random", "--max-evals", 10, "--gpus", 1, "--batch", 2,
        "--seed", 3, "--out", out, env={"TILETUNER_REPS": "2"}, check_rc=0)
    recs = [l.split(",") for l in out.read_text().splitlines() if not l.startswith("#")]
    assert len(recs) == 10 and all(r[5] == "ok" for r in recs)
