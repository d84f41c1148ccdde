import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(scope="session")
def cuda_lib():
    """The product C-ABI library, loaded through the Python binding.  GPU
    tests fail loudly (never skip to a CPU path) when it is missing."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but torch.cuda.is_available() is False")
    from paper_1909_00562_b200 import binding, build
    build.build()
    return binding.lib()


@pytest.fixture(scope="session")
def built_lib():
    """Build libattnsm.so in-tree if needed (nvcc cross-compiles without a
    GPU) and load it."""
    from paper_1909_00562_b200 import binding, build
    build.build()
    return binding.lib()
