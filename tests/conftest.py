import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def dev():
    import paper_2508_08343_b200 as lt

    return lt.device(0)


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle

    if not pyoracle.available("ref"):
        pytest.skip("oracle/_ref/libloratwin_ref.so not built (needs /root/reference at build time)")
    return pyoracle.RefOracle(threads=os.cpu_count() or 1)


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle

    if not os.path.exists(os.path.join(ROOT, "oracle", "restate.c")):
        pytest.skip("restatement not present")
    return pyoracle.PortOracle(threads=os.cpu_count() or 1)
