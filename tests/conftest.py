import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libvolpot_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def rel_l2(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="session")
def rest():
    import oracle
    return oracle.restatement()


@pytest.fixture(scope="session")
def ref():
    import oracle
    try:
        return oracle.reference()
    except (FileNotFoundError, OSError) as e:  # pragma: no cover
        pytest.skip(f"reference oracle unavailable: {e}")


@pytest.fixture(scope="session")
def vp():
    import paper_2203_05933_b200 as vp
    if vp.device_count() < 1:
        pytest.fail("gpu test run without a usable sm_100 device")
    return vp
