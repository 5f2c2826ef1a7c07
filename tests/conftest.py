import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_sessionstart(session):
    """Build the in-tree CUDA library when it is missing or older than its sources (a no-op
    otherwise), so the ABI and GPU tests always load the current code."""
    from paper_2507_14869_b200 import build as B

    B.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("-m gpu test run without a CUDA device")
    return torch.device("cuda:0")
