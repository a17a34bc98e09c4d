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


_REPORT = {}


@pytest.fixture(scope="session")
def parity_report():
    """Measured parity numbers (errors, decision agreement) collected by the GPU tests; written as JSON to
    $CIDER_PARITY_REPORT at session end (the GPU runs copy it into profiles/)."""
    return _REPORT


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("CIDER_PARITY_REPORT")
    if path and _REPORT:
        import json
        with open(path, "w") as f:
            json.dump(_REPORT, f, indent=1, sort_keys=True, default=float)
