import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def stk():
    import paper_1912_10082_b200 as s
    return s


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    return O


@pytest.fixture(scope="session")
def kats():
    import json
    return json.loads((ROOT / "tests" / "golden" / "spec_kats.json").read_text())


@pytest.fixture(scope="session")
def ref_bands():
    import numpy as np
    return dict(np.load(ROOT / "tests" / "golden" / "wave_bands_ref.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but CUDA is not available")
    return torch.device("cuda:0")
