"""The C++ drop-in (paper_2309_07235_b200/csrc/tiletuner_gpu.hpp) on a GPU, in one
program with the unmodified reference core: examples/dropin_harness.cpp, built by
oracle/Makefile into oracle/_ref/dropin_harness (INTEGRATION.md sections 2-3,
reference harness.cpp:99-105, kernels.hpp:29-70)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "oracle" / "_ref" / "dropin_harness"


@pytest.mark.gpu
def test_cpp_dropin_runs_against_reference_on_gpu():
    assert EXE.exists(), "build() builds oracle/_ref/dropin_harness (needs the reference sources)"
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
