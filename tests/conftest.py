import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
# reproducible keyring for the parity tests (the product default is a per-process secret)
os.environ.setdefault("CGB_KEY_SEED", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import rnsbfv

    rnsbfv.build()
    return rnsbfv


@pytest.fixture
def rng():
    return np.random.default_rng(0)
