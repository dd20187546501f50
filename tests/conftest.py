import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size (BASELINE config) property tests")


@pytest.fixture(scope="session")
def orc():
    from oracle_ctypes import oracle
    return oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_ctypes import reference
    r = reference()
    if r is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return r
