"""The C-ABI library loads on a CPU-only host and exports every symbol
include/tidepool_gpu.h declares (no compute calls without a GPU)."""

import re
from pathlib import Path

import pytest

from paper_1810_08723_b200 import _native, abi

HEADER = Path(__file__).resolve().parents[1] / "include" / "tidepool_gpu.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tpg_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(abi.PROTOTYPES)


@pytest.mark.skipif(not _native.LIB_PATH.exists(), reason="library not built")
def test_library_exports_every_header_symbol():
    L = _native.load_only()
    for name in header_functions():
        assert hasattr(L, name), name
    assert L.tpg_version().decode().startswith("tidepool_gpu")


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(abi.Plan) == 4 + 4 + 8 * 8 + 3 * 8 * 8
    assert C.sizeof(abi.Operand) == 8 + 8 + 4 + 4 + 16


def test_ops_fail_loudly_without_a_device(monkeypatch):
    """No CPU fallback: with the library missing every op raises."""
    from paper_1810_08723_b200 import errors
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", Path("/nonexistent/libtidepool_gpu.so"))
    with pytest.raises(errors.NativeLibraryMissing):
        _native.lib()
