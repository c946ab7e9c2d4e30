import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(autouse=True)
def _gpu_tests_need_a_gpu(request):
    """A selected `gpu` test fails loudly (never skips or silently passes) when no CUDA
    device is visible: there is no CPU fallback of the path to test instead."""
    if request.node.get_closest_marker("gpu") is not None:
        import torch
        if not torch.cuda.is_available():
            pytest.fail("gpu test selected but no CUDA device is visible (run with -m 'not gpu' on a CPU box)")
