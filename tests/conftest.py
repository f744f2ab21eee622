import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built CUDA library")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(params=["cluster", "wide"])
def sparse_kernel(request):
    """Run a sparse-decode test on both fused kernels: one thread-block cluster
    per unit (the default) and the wide decode (P CTAs per unit)."""
    from paper_2505_19586_b200 import _lib

    _lib.set_sparse_kernel(0 if request.param == "cluster" else 1)
    yield request.param
    _lib.set_sparse_kernel(-1)
