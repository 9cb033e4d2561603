import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libtersoff_b200.so)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref (the compiled reference) is not present")
    return Reference()


@pytest.fixture(scope="session")
def tb():
    import paper_1607_02904_b200 as tb
    return tb


@pytest.fixture(scope="session")
def si(tb):
    return tb.builtin_silicon()


@pytest.fixture(scope="session")
def sic_text():
    with open(os.path.join(GOLDEN, "SiC.tersoff")) as fh:
        return fh.read()
