import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")


@pytest.fixture(scope="session")
def ctx():
    """A product context on cuda:0.  GPU tests fail loudly (no fallback) without a device."""
    import paper_1610_08035_b200 as P
    c = P.Context(0)
    yield c
    c.close()


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(1e-300, float(np.max(np.abs(b)))))
