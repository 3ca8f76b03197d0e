import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: full-size inputs (tens of seconds)")


@pytest.fixture(scope="session")
def gpu_lib():
    """The CUDA path through the C-ABI; fails loudly when unavailable."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    import paper_1903_01665_b200 as fb
    fb.load()  # raises if libfalcon.so is missing: no fallback
    return fb
