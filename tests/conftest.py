"""Shared test configuration.

Markers: ``gpu`` tests need a B200 (they run through libhmx.so); everything
else runs on the CPU-only build container.  The reference package is never
imported here: parity is pinned by the committed fixtures in tests/golden/
(made by tests/golden/make_golden.py) and by the CPU oracle in oracle/.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhmx.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _release_device_plans(request):
    """Cached plans hold per-CTA scratch arenas (GBs at c2 size): free them
    after every GPU test so one module's plans cannot starve the next."""
    yield
    if "gpu" not in request.keywords:
        return
    import gc

    from paper_1911_07531_b200 import arith

    arith.clear_plans()
    gc.collect()
    try:
        import torch

        torch.cuda.empty_cache()
    except Exception:
        pass
