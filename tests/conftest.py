import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return Reference()


@pytest.fixture(scope="session")
def cuda():
    if not _has_gpu():
        pytest.fail("GPU test collected on a host without a CUDA device")
    from paper_2512_07350_b200 import _lib

    _lib.check(_lib.lib().lp_device_check(0))
    return True
