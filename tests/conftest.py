import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: large configuration (minutes)")


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated (tests/golden/make_golden.py)")
    return np.load(path)


@pytest.fixture(scope="session")
def small():
    return golden("small_cases.npz")


@pytest.fixture(scope="session")
def ref_arm():
    import oracle

    if not oracle.have_ref():
        pytest.skip("reference build oracle/_ref absent")
    return oracle.ref()


@pytest.fixture(scope="session")
def port_arm():
    import oracle

    return oracle.port()
