import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ctx():
    from paper_2604_07980_b200.ranger import Context
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def orc():
    import oracle_lib
    return oracle_lib.oracle()


@pytest.fixture(scope="session")
def chk():
    """GPU parity checker: the reference itself (oracle/_ref) when present,
    the C restatement otherwise and for the 9x7 extension."""
    import oracle_lib
    return oracle_lib.checker()
