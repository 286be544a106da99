import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built librsw.so")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def rsw_gpu():
    """The CUDA path.  Fails loudly (no fallback) when the library or the GPU is missing."""
    import torch
    import paper_1303_6615_b200 as rsw
    from paper_1303_6615_b200 import build
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    build.build()
    rsw.load()
    return rsw
