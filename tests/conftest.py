import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# A protocol bug must fail a test quickly rather than sit out the 20 s default per rank.
os.environ.setdefault("ZC_COMM_TIMEOUT_MS", "8000")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.ref()
    if r is None:
        pytest.skip("reference library oracle/_ref was not built (no /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def zc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_12396_b200 import zcomm
    zcomm.lib()
    return zcomm
