"""GPU tests of the batched evaluator's failure semantics and the T1/T8 harness.

* MeasurementError (harness.cpp:252-256): the reference flushes the partial trace
  and rethrows.  Here one failing device retires only its worker — its candidate
  is re-evaluated elsewhere and the run completes; when every worker failed the
  partial trace comes back with the error (tt_tune_measured, the CLI).
* run_tuning_virtual: W evaluators emulated on one device on a virtual clock
  (every evaluation measured for real) — the harness behind T1 / T8.
"""
import pytest

from paper_2309_07235_b200 import tuning

pytestmark = pytest.mark.gpu


def test_fault_on_one_worker_is_requeued(monkeypatch):
    monkeypatch.setenv("TT_FAULT_INJECT", "1:2")
    recs, _ = tuning.run_tuning_measured("bayesopt", "lu", "small", 3, 24, devices=(0, 0))
    assert len(recs) == 24  # the run completes on the surviving worker
    assert len({r.flat for r in recs}) == 24
    assert sum(r.worker == 1 for r in recs) == 2  # worker 1 retired at its 3rd evaluation
    el = [r.elapsed_s for r in recs]
    assert el == sorted(el)


def test_fault_on_only_worker_flushes_partial_trace(monkeypatch):
    monkeypatch.setenv("TT_FAULT_INJECT", "0:5")
    with pytest.raises(tuning.TuningError) as ei:
        tuning.run_tuning_measured("bayesopt", "lu", "small", 3, 24, devices=(0,))
    recs = ei.value.records
    assert len(recs) == 5 and "injected device fault" in str(ei.value)
    best = float("inf")
    for r in recs:
        best = min(best, r.runtime_s)
        assert r.best_so_far_s == best


def test_cli_flushes_partial_trace(tmp_path, monkeypatch):
    import subprocess
    from pathlib import Path
    cli = Path(tuning.__file__).resolve().parent / "tiletuner-gpu"
    out = tmp_path / "t.trace"
    env = dict(__import__("os").environ, TT_FAULT_INJECT="0:4")
    p = subprocess.run([str(cli), "tune", "lu", "small", "--tuner", "bayesopt", "--max-evals", "20",
                        "--gpus", "1", "--out", str(out)], env=env, capture_output=True, text=True)
    assert p.returncode == 1, p.stderr
    assert "partial trace flushed" in p.stderr
    body = [l for l in out.read_text().splitlines() if l and not l.startswith("#")]
    assert len(body) == 4  # the 4 records measured before the fault


def test_virtual_harness_w1_matches_sequential_semantics():
    r1, tot1 = tuning.run_tuning_virtual("bayesopt", "lu", "large", 7, 30, workers=1)
    r8, tot8 = tuning.run_tuning_virtual("bayesopt", "lu", "large", 7, 30, workers=8)
    for recs in (r1, r8):
        assert len(recs) == 30 and len({r.flat for r in recs}) == 30
        el = [r.elapsed_s for r in recs]
        assert el == sorted(el)
        assert all(r.eval_s > 0 for r in recs)
    # one evaluator: elapsed is the running sum of ask + evaluation times
    acc = 0.0
    for r in r1:
        acc += r.ask_s + r.eval_s
        assert abs(r.elapsed_s - acc) <= 1e-9 * max(1.0, acc) + 1e-12
    assert {r.worker for r in r8} == set(range(8))
    assert tot8 < tot1  # same budget on 8 evaluators
