import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, TESTS):  # TESTS: shared helpers of the GPU parity modules (test_gpu_parity.build_net, ...)
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity of the CUDA path vs the oracle")
    config.addinivalue_line("markers", "slow: long-running (full-size sampled parity)")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o
    o.lib()
    return o


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_00209_b200 as b
    b.lib()  # raises if libbnn.so is missing -- never a silent fallback
    return b
