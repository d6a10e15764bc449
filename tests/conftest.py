import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running parity case")


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def sign_align(a, b):
    """Per-row sign alignment (DPSS sign is ambiguous for antisymmetric tapers, eig.cpp:281-289)."""
    s = np.sign(np.sum(a * b, axis=-1, keepdims=True))
    s[s == 0] = 1
    return a * s


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.lib_c()
    return oracle
