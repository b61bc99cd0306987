import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def yb():
    import paper_1301_4539_b200 as Y
    if not os.path.exists(Y.LIB_PATH):
        Y.build()
    return Y
