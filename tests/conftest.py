import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libggb.so")
    config.addinivalue_line("markers", "slow: larger graphs")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def ggb():
    import paper_2104_10039_b200 as m
    return m


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    return o
