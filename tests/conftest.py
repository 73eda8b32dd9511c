import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libspecmoe.so")
    config.addinivalue_line("markers", "sanitizer: compute-sanitizer tier (also gpu)")


@pytest.fixture(scope="session")
def oracle():
    import oracle_py
    oracle_py.build()
    return oracle_py


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test requires CUDA")  # never silently skip on the GPU tier
    from paper_2508_21706_b200 import build
    build.build()
    return torch.device("cuda:0")
