import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
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
def _device_error_flags(request):
    """After every GPU test: no workspace the binding cached may carry a device error bit
    (larosa_error_flags: keep-all fallback of an inconsistent Top-K histogram, fixed-point
    overflow).  Tests that provoke one on purpose clear it themselves."""
    yield
    if "gpu" not in request.keywords:
        return
    import torch
    if not torch.cuda.is_available():
        return
    from paper_2507_01299_b200 import larosa as LZ
    bad = [(i, f) for i, ws in enumerate(LZ.workspaces()) for f in [LZ.error_flags(ws)] if f]
    assert not bad, f"device error flags set in cached workspaces: {bad}"
