import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgnnv.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _guard_check(request):
    """With GNNV_GUARD_ALLOC=1: after every GPU test, no library allocation's
    guard region may have changed (out-of-bounds writes; the pool's
    compute-sanitizer is closed)."""
    yield
    if os.environ.get("GNNV_GUARD_ALLOC") == "1" and "gpu" in request.keywords:
        from paper_2404_09544_b200 import gnnv

        report = gnnv.check_guards()
        assert report == "", report
