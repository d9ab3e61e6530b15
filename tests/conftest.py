import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built liblfsr.so")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def lfsr_mod():
    """The CUDA path (fails loudly if liblfsr.so is missing or no GPU is visible)."""
    import torch
    assert torch.cuda.is_available(), "gpu test needs a CUDA device"
    import paper_2206_05047_b200 as m
    m.load_library()
    return m
