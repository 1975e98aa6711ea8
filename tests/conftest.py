import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def small_cases():
    return json.loads((GOLDEN / "small_cases.json").read_text())


def small_text(n: int, seed: int) -> np.ndarray:
    """Regenerates the texts of tests/golden/make_golden.py (SMALL)."""
    return np.random.Generator(np.random.PCG64([900, seed])).integers(0, 4, n, dtype=np.uint8)


def codes_to_str(codes) -> str:
    return "".join("ACGT"[int(c)] for c in codes)


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: GPU tests must fail loudly, not skip, when CUDA is absent."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    return torch.device("cuda:0")
