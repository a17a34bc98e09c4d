import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def P():
    import paper_2605_26580_b200 as P
    return P


@pytest.fixture(scope="session")
def oracle():
    from oracle.binding import Checker
    return Checker("oracle")


@pytest.fixture(scope="session")
def reference():
    from oracle.binding import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref (the reference built from /root/reference) not present")
    return Reference()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1e-30, np.abs(b).max()))
