"""Loader for the in-tree C-ABI library libtidepool_gpu.so.

There is no fallback: if the library is missing or no CUDA device is
visible, every gpu operation raises NativeLibraryMissing / DeviceError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import abi
from .errors import AllocationError, DeviceError, NativeLibraryMissing

LIB_PATH = Path(os.environ.get("TIDEPOOL_GPU_LIB",
                               Path(__file__).resolve().parent / "libtidepool_gpu.so"))

_lib = None
_lock = threading.Lock()

E_ALLOC = -2


def lib():
    """The loaded library (initialised); raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is not built; run `python -m paper_1810_08723_b200.build`")
            try:
                L = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
            except OSError as exc:
                raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
            abi.declare(L)
            rc = L.tpg_init()
            if rc != 0:
                raise DeviceError(f"tpg_init failed: {L.tpg_last_error().decode()}")
            _lib = L
    return _lib


def load_only():
    """dlopen + declare without initialising CUDA (CPU-side symbol checks)."""
    L = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    return abi.declare(L)


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = _lib.tpg_last_error().decode() if _lib is not None else "library not loaded"
    if rc == E_ALLOC:
        raise AllocationError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg}" if what else msg)


def device_count() -> int:
    n = C.c_int(0)
    try:
        L = lib()
    except (NativeLibraryMissing, DeviceError):
        return 0
    L.tpg_device_count(C.byref(n))
    return n.value
