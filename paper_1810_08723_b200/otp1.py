"""OTP1 tensor files read and written directly from / to the GPU
(SURVEY.md §8f item 4).

Format (reference interop.py:29-30, 94-167): a 8-byte header
`<4sBBBB` = magic b"OTP\\x01", dtype wire code, byte order (0 little, 1
big), ndim, reserved 0; then ndim little-endian uint64 extents; then the
elements in contiguous column-major order, each in the tensor's own byte
order (bit-exact, no conversion).

The reference stages a gpu-like tensor through host memory with a Python
pair-list gather and packs the payload element by element
(interop.py:105-121).  Here:
  save: a strided tensor is first packed on the device by the descriptor
        gather (byte-exact, byte order kept), then streamed to the sink
        through two pinned staging buffers: the device-to-host copy of
        chunk i+1 overlaps the host write of chunk i;
  load: header parsed and validated with the reference's checks and
        messages, the payload streamed through two pinned buffers into a
        contiguous gpu tensor (host read of chunk i+1 overlaps the
        host-to-device copy of chunk i); `native=True` additionally
        byte-swaps a big-endian file on the device (values kept).
"""

from __future__ import annotations

import ctypes as C
import io
import math
import struct

from . import _native, dtypes, tensors as tz
from .errors import FormatError

MAGIC = b"OTP\x01"
_HEADER = struct.Struct("<4sBBBB")
CHUNK = 32 << 20


def pack_header(dtype, byteorder: str, dims) -> bytes:
    head = _HEADER.pack(MAGIC, dtype.code, 0 if byteorder == "little" else 1, len(dims), 0)
    return head + b"".join(struct.pack("<Q", d) for d in dims)


def parse_header(source):
    """(dtype, byteorder, dims) from a binary stream, with the reference's
    validation order and messages (interop.py:135-160)."""
    head = source.read(_HEADER.size)
    if len(head) < _HEADER.size:
        raise FormatError("truncated OTP1 header")
    magic, dtype_code, order_code, ndim, reserved = _HEADER.unpack(head)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic.hex()} (expected {MAGIC.hex()})")
    if reserved != 0:
        raise FormatError(f"reserved header byte is {reserved}, must be 0")
    if ndim > tz.MAX_DIMS:
        raise FormatError(f"{ndim} dimensions exceed the limit of {tz.MAX_DIMS}")
    if order_code not in (0, 1):
        raise FormatError(f"bad byte-order code {order_code}")
    try:
        dtype = dtypes.by_wire_code(dtype_code)
    except Exception:
        raise FormatError(f"bad dtype code {dtype_code}") from None
    dims = []
    for _ in range(ndim):
        raw = source.read(8)
        if len(raw) < 8:
            raise FormatError("truncated OTP1 dimension list")
        dims.append(struct.unpack("<Q", raw)[0])
    return dtype, ("little" if order_code == 0 else "big"), tuple(dims)


def _is_packed(t) -> bool:
    return t.strides == tz.column_major_strides(t.dims, t.dtype.size)


class _Pinned:
    """Two pinned host buffers + events for double-buffered streaming."""

    def __init__(self, nbytes: int):
        L = _native.lib()
        self.n = nbytes
        self.buf, self.ev = [], []
        for _ in range(2):
            p = C.c_void_p()
            _native.check(L.tpg_host_alloc(max(nbytes, 16), C.byref(p)), "pinned alloc")
            self.buf.append(p.value)
            e = C.c_void_p()
            _native.check(L.tpg_event_create(C.byref(e)), "event")
            self.ev.append(e.value)

    def view(self, i: int, n: int) -> memoryview:
        return memoryview((C.c_char * n).from_address(self.buf[i])).cast("B")

    def close(self):
        L = _native.lib()
        for p in self.buf:
            L.tpg_host_free(p)
        for e in self.ev:
            L.tpg_event_destroy(e)


def save_otp1(t, sink, chunk: int = CHUNK) -> None:
    """Write a gpu tensor to a path or binary file object (reference
    interop.save_otp1 semantics: contiguous column-major payload, dtype and
    byte order preserved bit-exactly)."""
    if isinstance(sink, (str, bytes)):
        with open(sink, "wb") as fh:
            save_otp1(t, fh, chunk)
        return
    sink.write(pack_header(t.dtype, t.byteorder, t.dims))
    nbytes = t.nelem * t.dtype.size
    if nbytes == 0:
        return
    src = t if _is_packed(t) else tz.contiguous_clone(t)  # device descriptor gather
    stream = src.storage.stream
    src.storage.order(stream)
    L = _native.lib()
    pin = _Pinned(min(chunk, nbytes))
    try:
        base = src.storage.ptr + src.offset
        offs = list(range(0, nbytes, pin.n))

        def issue(k):
            n = min(pin.n, nbytes - offs[k])
            _native.check(L.tpg_memcpy_d2h(pin.buf[k % 2], base + offs[k], n, stream.handle),
                          "d2h")
            _native.check(L.tpg_event_record(pin.ev[k % 2], stream.handle), "event")

        issue(0)
        for k in range(len(offs)):
            if k + 1 < len(offs):
                issue(k + 1)  # next chunk's copy runs while this one is written
            _native.check(L.tpg_event_sync(pin.ev[k % 2]), "event sync")
            n = min(pin.n, nbytes - offs[k])
            sink.write(pin.view(k % 2, n))
    finally:
        stream.sync()
        pin.close()


def save_otp1_bytes(t) -> bytes:
    sink = io.BytesIO()
    save_otp1(t, sink)
    return sink.getvalue()


def load_otp1(source, device=None, native: bool = False, chunk: int = CHUNK):
    """Read an OTP1 stream into a contiguous column-major gpu tensor.
    The file's byte order is kept (bit-exact) unless native=True, which
    byte-swaps big-endian data on the device."""
    if isinstance(source, str):
        with open(source, "rb") as fh:
            return load_otp1(fh, device, native, chunk)
    if isinstance(source, (bytes, bytearray, memoryview)):
        return load_otp1(io.BytesIO(bytes(source)), device, native, chunk)
    dtype, order, dims = parse_header(source)
    device = device or tz.default_device()
    t = tz.tensor_create(dims, dtype, device)
    t.byteorder = order
    expect = math.prod(dims) * dtype.size
    if expect:
        L = _native.lib()
        stream = t.storage.stream
        pin = _Pinned(min(chunk, expect))
        try:
            base = t.storage.ptr + t.offset
            done = 0
            k = 0
            while done < expect:
                n = min(pin.n, expect - done)
                if k >= 2:  # buffer k%2 was handed to the copy two chunks ago
                    _native.check(L.tpg_event_sync(pin.ev[k % 2]), "event sync")
                got = source.readinto(pin.view(k % 2, n)) if hasattr(source, "readinto") else None
                if got is None:
                    raw = source.read(n)
                    got = len(raw)
                    pin.view(k % 2, got)[:] = raw
                if got < n:
                    raise FormatError(
                        f"truncated OTP1 payload: {done + got} of {expect} bytes")
                _native.check(L.tpg_memcpy_h2d(base + done, pin.buf[k % 2], n, stream.handle),
                              "h2d")
                _native.check(L.tpg_event_record(pin.ev[k % 2], stream.handle), "event")
                done += n
                k += 1
        finally:
            stream.sync()
            pin.close()
    if native and order == "big" and expect:
        from . import ops
        ops.byteswap(t)
    return t
