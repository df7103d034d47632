import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def pytest_sessionstart(session):
    """Build libhfb200.so in-tree if it is missing or stale (nvcc cross-compiles
    sm_100a without a GPU); the package refuses to import without it."""
    try:
        from paper_1811_07717_b200 import build as B

        B.build(force=False)
    except Exception as exc:  # surfaced by the import error in the tests themselves
        print(f"warning: could not build libhfb200.so: {exc}")
