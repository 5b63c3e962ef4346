import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def cuda():
    """The GPU tests run on the B200 box; there, a missing GPU is a failure, not a skip."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test needs a CUDA device"
    return torch
