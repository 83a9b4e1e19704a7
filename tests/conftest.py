import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

GOLDEN = os.path.join(ROOT, "tests", "golden")

# the paper's 6-point running example: a..f = ids 0..5
FIG_COORDS = np.array([[5, 1], [4, 3], [4, 2], [1, 2], [1, 0], [0, 3]], dtype=np.float32)
A, B, C, D, E, F = range(6)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: larger parity cases")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    return oracle
