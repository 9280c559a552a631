import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmoa.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()


@pytest.fixture(scope="module")
def moa():
    """The product package (libmoa.so through ctypes); GPU tests only."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_14909_b200 as m
    return m
