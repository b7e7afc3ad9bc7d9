import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: larger sizes")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def ops_golden():
    return golden("ops.npz")


@pytest.fixture(scope="session")
def nets():
    from oracle import mg_oracle as mo
    return {v: mo.load_net_json(os.path.join(GOLDEN, f"net_{v}.json"))
            for v in ("conv", "fc", "conv_k2")}


def rel_err(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / den)
