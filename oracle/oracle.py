"""ctypes front of the C oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.  The functions take the same plan / operand
descriptors as the product C ABI (include/tidepool_gpu.h) but operate on
HOST buffers, following the reference loops one element at a time.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import build as _build

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.build()
        L = C.CDLL(str(path))
        from paper_1810_08723_b200 import abi  # struct layouts only
        P, PL, OP = C.POINTER, C.POINTER(abi.Plan), C.POINTER(abi.Operand)
        u32p = P(C.c_uint32)
        sig = {
            "tpo_binary": [C.c_int, PL, OP, OP, OP, C.c_int, C.c_int, u32p],
            "tpo_unary": [C.c_int, PL, OP, OP, C.c_int, C.c_int, C.c_int, u32p],
            "tpo_reduce": [C.c_int, C.c_double, PL, PL, OP, OP, C.c_int, C.c_int, u32p],
            "tpo_matmul": [OP, P(C.c_int64), OP, P(C.c_int64), OP, P(C.c_int64), C.c_int64,
                           C.c_int64, C.c_int64, C.c_int, C.c_int, u32p],
            "tpo_fill": [PL, OP, C.c_void_p, C.c_int32],
            "tpo_arange": [PL, OP],
            "tpo_byteswap": [PL, OP],
            "tpo_threads": [],
            "tpo_set_threads": [C.c_int],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        _lib = L
    return _lib


def ptr(buf) -> int:
    """Address of a writable bytearray / numpy array."""
    import numpy as np
    if isinstance(buf, np.ndarray):
        return buf.ctypes.data
    return C.addressof(C.c_char.from_buffer(buf))


def threads() -> int:
    return lib().tpo_threads()


def set_threads(n: int) -> int:
    lib().tpo_set_threads(int(n))
    return threads()
