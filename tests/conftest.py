import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (run through gpurun)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    try:
        return Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def ctx():
    from paper_1910_13555_b200.store import Context
    c = Context(0)
    yield c
    c.close()


def frob_rel(a, b):
    """frobenius_rel_error (oracles.hpp:49-57)."""
    diff = float(np.sum((a - b) ** 2))
    ref = float(np.sum(b * b))
    return np.sqrt(diff) if ref == 0 else np.sqrt(diff / ref)
