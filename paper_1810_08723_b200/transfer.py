"""Asynchronous host <-> device transfers for pipelined end-to-end use.

The reference moves data between host and device synchronously through the
destination's copy entry (ops.py:110-118).  For host-to-host pipelines
(upload a slab, run ops on it, download the result while the next slab
uploads) the module exposes:

    buf = pinned((4096, 512), np.float32)       # page-locked numpy array
    upload(buf, t, stream)                      # async H2D into a tensor
    download(t, buf, stream)                    # async D2H from a tensor
    with use_stream(stream): tp.add(...)        # ops launch on `stream`

`upload`/`download` take tensors whose bytes form a contiguous run or a
2-D pitched slab (unit-stride axis 0, any axis-1 stride), i.e. column
slabs and row slabs of column-major tensors.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native
from .errors import ShapeError
from .table import use_stream  # noqa: F401  (public: ops launch on a given stream)


class _PinnedOwner:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            _native.lib().tpg_host_free(self.ptr)
        except Exception:
            pass


def pinned(shape, dtype, order: str = "F") -> np.ndarray:
    """A numpy array in page-locked host memory (freed with the array)."""
    dtype = np.dtype(dtype)
    n = int(math.prod(shape)) * dtype.itemsize
    p = C.c_void_p()
    _native.check(_native.lib().tpg_host_alloc(max(n, 16), C.byref(p)), "pinned alloc")
    raw = (C.c_ubyte * max(n, 16)).from_address(p.value)
    raw._tpg_owner = _PinnedOwner(p.value)
    arr = np.frombuffer(raw, dtype=np.uint8, count=n).view(dtype)
    return arr.reshape(shape, order=order)


def _layout(t):
    """(first byte offset, rows bytes, ncols, pitch) of a tensor whose
    bytes are a contiguous run or a 2-D pitched slab."""
    es = t.dtype.size
    keep = [(d, st) for d, st in zip(t.dims, t.strides) if d != 1]  # extent-1 strides are free
    dims, strides = [d for d, _ in keep], [st for _, st in keep]
    if not dims or t.nelem == 1:
        return t.offset, es, 1, es
    if t.nelem == 0:
        return t.offset, 0, 1, 0
    if len(dims) == 1:
        if strides[0] != es:
            raise ShapeError("transfer needs a unit-stride view")
        return t.offset, dims[0] * es, 1, dims[0] * es
    if len(dims) == 2 and strides[0] == es and strides[1] >= dims[0] * es:
        if strides[1] == dims[0] * es:
            n = dims[0] * dims[1] * es
            return t.offset, n, 1, n
        return t.offset, dims[0] * es, dims[1], strides[1]
    raise ShapeError("transfer needs a contiguous run or a 2-D pitched slab")


def _host_layout(arr, width, height):
    """(pointer, pitch) of a host array holding `height` runs of `width`
    bytes: contiguous, or a 2-D column-major slab view (unit-stride axis 0)
    of a larger array, e.g. out[r0:r1, :] of a Fortran-ordered matrix."""
    if arr.flags.c_contiguous or arr.flags.f_contiguous:
        if arr.nbytes < width * height:
            raise ShapeError("host buffer too small")
        return arr.ctypes.data, width
    if (arr.ndim == 2 and arr.strides[0] == arr.itemsize and arr.shape[0] * arr.itemsize == width
            and arr.shape[1] == height and arr.strides[1] >= width):
        return arr.ctypes.data, arr.strides[1]
    raise ShapeError("host buffer must be contiguous or a column-major 2-D slab")


def upload(src: np.ndarray, t, stream=None) -> None:
    """Async copy of a (pinned) host array's bytes into tensor `t`."""
    off, width, height, pitch = _layout(t)
    hp, hpitch = _host_layout(src, width, height)
    st = stream or t.storage.stream
    t.storage.order(st)
    t.storage.note_use(st)
    s = st.handle
    L = _native.lib()
    dst = t.storage.ptr + off
    if height == 1:
        _native.check(L.tpg_memcpy_h2d(dst, hp, width, s), "upload")
    else:
        _native.check(L.tpg_memcpy2d(dst, pitch, hp, hpitch, width, height, s), "upload")


def download(t, dst: np.ndarray, stream=None) -> None:
    """Async copy of tensor `t`'s bytes into a (pinned) host array."""
    off, width, height, pitch = _layout(t)
    hp, hpitch = _host_layout(dst, width, height)
    st = stream or t.storage.stream
    t.storage.order(st)
    t.storage.note_use(st)
    s = st.handle
    L = _native.lib()
    src = t.storage.ptr + off
    if height == 1:
        _native.check(L.tpg_memcpy_d2h(hp, src, width, s), "download")
    else:
        _native.check(L.tpg_memcpy2d(hp, hpitch, src, pitch, width, height, s), "download")
