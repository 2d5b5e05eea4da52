import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libptg.so")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture(scope="session")
def oracle():
    from oracle import ptgo
    ptgo.lib()
    return ptgo


@pytest.fixture(scope="session")
def reference(oracle):
    if not oracle.has_reference():
        pytest.skip("reference library oracle/_ref/libptycho_ref.so not built (no /root/reference)")
    oracle.ref()
    return oracle


def rand_field(n, seed, scale=1.0):
    """test_support.hpp:34-41 analogue: U[-1,1]^2 entries (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    return scale * (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n)))


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def rel(a, b, floor=0.0):
    return abs(a - b) / max(abs(b), floor, 1e-300)
