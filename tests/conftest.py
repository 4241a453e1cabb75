import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size parity)")


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_full():
    p = GOLDEN / "golden_full.json"
    if not p.exists():
        pytest.skip("golden_full.json not generated")
    return json.loads(p.read_text())


@pytest.fixture(scope="session")
def garrays():
    with np.load(GOLDEN / "golden_arrays.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def gpu_ctx():
    """The product context on cuda:0.  Fails loudly (no CPU fallback)."""
    from paper_2309_07235_b200 import Context
    ctx = Context(0)
    yield ctx
    ctx.close()
