import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# AUTO sends tiny jobs to the per-reference direct kernel (gbm3d_api.cu, small_direct); the
# parity tests' small edge-case images must keep exercising the tile kernels they were written
# for, so the rule is off here and tested on its own (test_auto_small_jobs_direct, subprocess).
os.environ.setdefault("GBM3D_NO_SMALL_DIRECT", "1")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: larger CPU cases")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run under gpurun)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
