import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(params=["1", "2"], ids=["ks1", "ks2"])
def walk_ks(request, monkeypatch):
    """Runs a GPU parity test once per K1 walk variant: one scenario per
    thread and two per thread (the variant every benchmark launch takes).
    LUMOS_WALK_KS pins the choice inside ts_replay_batch (capi.cpp); batches
    starting at an odd global id always take one scenario per thread."""
    monkeypatch.setenv("LUMOS_WALK_KS", request.param)
    return int(request.param)
