import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the sm_100a C-ABI)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import bindings as B
    B.ensure_built()
    return B.Oracle()


@pytest.fixture(scope="session")
def refimpl():
    from oracle import bindings as B
    if not os.path.exists(B.REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return B.Ref()


@pytest.fixture(scope="session")
def ctx():
    from paper_1310_3435_b200 import sdd
    return sdd.default_context(0)
