"""Shared fixtures.  GPU tests are marked ``gpu`` (run with ``-m gpu`` on a
B200); everything else runs on CPU.  The seed is the reference's
(pkg/tests/conftest.py:27-29)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "halftile_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU")


@pytest.fixture
def rng():
    return np.random.default_rng(20260810)


@pytest.fixture(scope="session")
def golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


@pytest.fixture(scope="session")
def cuda():
    """GPU tests must not pass silently without a GPU: fail loudly."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("test marked gpu needs a CUDA device (run with -m 'not gpu' on CPU)")
    torch.cuda.set_device(0)
    return torch.device("cuda:0")
