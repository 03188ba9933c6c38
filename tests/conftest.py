import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtidepool_gpu.so")


def _install_fake_native() -> bool:
    """TPG_FAKE_NATIVE=1 (test runs only): drive the standalone host layer
    through the CPU test double of the C ABI (tests/fake_native.py, kernels
    by the C oracle) so its pipeline can be exercised without a GPU."""
    import os
    if os.environ.get("TPG_FAKE_NATIVE") != "1":
        return False
    from fake_native import FakeNative
    from oracle import oracle
    from paper_1810_08723_b200 import _native
    if not isinstance(_native._lib, FakeNative):
        _native._lib = FakeNative(oracle.lib())
    return True


def _has_gpu() -> bool:
    if _install_fake_native():
        return True
    try:
        from paper_1810_08723_b200 import _native
        return _native.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if not any("gpu" in item.keywords for item in items):
        return
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
