import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.Ref.available():
        pytest.skip("reference library oracle/_ref not built")
    return oracle.ref()


@pytest.fixture(scope="session")
def gpu():
    """The product library on a real device (fails loudly if unusable)."""
    from paper_1510_08982_b200 import _lib
    L = _lib.lib()
    assert L.heat_device_count() > 0, "no CUDA device visible to the gpu tests"
    return L
