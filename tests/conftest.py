import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
ORACLE = os.path.join(ROOT, "oracle")
if ORACLE not in sys.path:
    sys.path.insert(0, ORACLE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long CPU-side oracle runs")


@pytest.fixture(scope="session")
def port():
    import pyoracle

    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    import pyoracle

    if not pyoracle.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent here)")
    return pyoracle.Ref()
