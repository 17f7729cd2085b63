import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(ROOT, "tests", "golden", "golden.npz")
    with np.load(path) as g:
        return {k: g[k] for k in g.files}


@pytest.fixture(scope="session")
def golden_r2():
    path = os.path.join(ROOT, "tests", "golden", "golden_r2.npz")
    with np.load(path) as g:
        return {k: g[k] for k in g.files}


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected on a machine without CUDA")
    return torch.device("cuda", 0)
