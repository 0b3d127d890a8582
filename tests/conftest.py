import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libfk_cuda.so; run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from paper_2508_07071_b200.opfuse import Library
    return Library("oracle")


@pytest.fixture(scope="session")
def reference():
    from paper_2508_07071_b200.opfuse import Library
    return Library("reference")


@pytest.fixture(scope="session")
def cuda():
    """The product library on cuda:0. Fails (never skips) when it cannot run."""
    import torch
    from paper_2508_07071_b200.opfuse import Library
    assert torch.cuda.is_available(), "gpu test on a host without a CUDA device"
    torch.cuda.set_device(0)
    return Library("cuda")
