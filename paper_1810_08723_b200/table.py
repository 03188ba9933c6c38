"""The ("core", "gpu") function table: 31 entries with the reference's
table-entry signatures, each a thin shim onto one C-ABI call.

Reference table: backend_cpu.build_core_table (pkg/src/tidepool/
backend_cpu.py:10-27) and the per-key call signatures listed in SURVEY.md
§8b, e.g. binary entries are called as
``h(plan, d_buf, store, a_buf, a_unpack, b_buf, b_unpack, fn, bases)``
(ops.py:282-283 -> kernels.py:213-214).  Where the reference passes Python
closures (store / unpack / fn / init-step-fin), this table receives small
descriptor objects carrying the same information (dtype, byte order, mode,
op, compute dtype); the closure-decoding adapter for the unmodified
reference lives in tidepool_plugin.py and produces the same descriptors.
Every entry enqueues asynchronously on the current stream; there is no
host fallback.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native, abi, dtypes
from .errors import DomainError

_tls = threading.local()


def current_stream():
    return getattr(_tls, "stream", None)


class use_stream:
    """Context manager: launches inside go to `stream` (a GpuStream)."""

    def __init__(self, stream):
        self.stream = stream

    def __enter__(self):
        self.prev = getattr(_tls, "stream", None)
        _tls.stream = self.stream
        return self.stream

    def __exit__(self, *exc):
        _tls.stream = self.prev


def _sh():
    s = current_stream()
    return s.handle if s is not None else None


# ---------------------------------------------------------------------------
# descriptors (what the reference's closures carry)
# ---------------------------------------------------------------------------
class Codec:
    """dtypes.codec(d, byteorder) stand-in; `imm` holds packed bytes when the
    operand is a by-value scalar (buffer None)."""
    __slots__ = ("dtype", "byteorder", "imm")

    def __init__(self, dtype, byteorder="little", imm: bytes | None = None):
        self.dtype = dtype
        self.byteorder = byteorder
        self.imm = imm


class Store:
    """ops._make_store stand-in: destination dtype, byte order, mode."""
    __slots__ = ("dtype", "byteorder", "mode", "loss")

    def __init__(self, dtype, byteorder, mode="standard"):
        self.dtype = dtype
        self.byteorder = byteorder
        self.mode = mode
        self.loss = False  # set when a warning-mode cast lost information


class BinaryFn:
    __slots__ = ("op", "compute", "mode")

    def __init__(self, op, compute, mode="standard"):
        self.op, self.compute, self.mode = op, compute, mode


class UnaryFn:
    __slots__ = ("op", "compute", "mode", "force_complex")

    def __init__(self, op, compute, mode="standard", force_complex=False):
        self.op, self.compute, self.mode, self.force_complex = op, compute, mode, force_complex


class ReduceAcc:
    """Stands in for (init, step, fin) of ops._reduction_acc."""
    __slots__ = ("op", "compute", "p")

    def __init__(self, op, compute, p=2.0):
        self.op, self.compute, self.p = op, compute, p


class MatmulFn:
    __slots__ = ("compute",)

    def __init__(self, compute):
        self.compute = compute


def operand(buf, base, codec: Codec) -> abi.Operand:
    if buf is None:
        return abi.make_operand(None, 0, codec.dtype.code, codec.byteorder == "big", codec.imm)
    return abi.make_operand(buf.ptr, base, codec.dtype.code, codec.byteorder == "big")


def dest(buf, base, store: Store) -> abi.Operand:
    return abi.make_operand(buf.ptr, base, store.dtype.code, store.byteorder == "big")


# ---------------------------------------------------------------------------
# status flags (ops._status) and error/warning-mode handling
# ---------------------------------------------------------------------------
_host_status: set = set()
_FLAG_NAMES = {abi.FLAG_DOMAIN: "domain-violation", abi.FLAG_INT_DIV0: "integer-division-by-zero"}


def _drain_flags(dev: int) -> int:
    f = C.c_uint32(0)
    L = _native.lib()
    _native.check(L.tpg_flags_get(dev, C.byref(f)), "flags")
    if f.value:
        _native.check(L.tpg_flags_clear(dev), "flags clear")
    for bit, name in _FLAG_NAMES.items():
        if f.value & bit:
            _host_status.add(name)
    return f.value


def get_status(devices_to_sync) -> frozenset:
    for d in devices_to_sync:
        d.synchronize()
        _drain_flags(d.index)
    return frozenset(_host_status)


def clear_status(devices_to_sync) -> None:
    for d in devices_to_sync:
        d.synchronize()
        _drain_flags(d.index)
    _host_status.clear()


def _guarded(mode: str, run, check, dev: int):
    """Launch under the reference's mode rules (dtypes.CastContext,
    dtypes.py:233-255).  standard / complex: run.  error: drain pending
    flags, then either a dry-run `check` (no writes; raise before anything
    is stored) or, for entries without one (reductions, products), the real
    launch followed by the flag read; raise DomainError on cast loss.
    warning: run, then one diagnostic per call on cast loss.  The flag reads
    (tpg_flags_get) wait for every stream of `dev`."""
    if mode in ("standard", "complex"):
        _native.check(run(), "kernel")
        return
    _drain_flags(dev)
    if mode == "error" and check is not None:
        _native.check(check(), "kernel check")
        _raise_on(_drain_flags(dev))
        _native.check(run(), "kernel")
        return
    _native.check(run(), "kernel")
    f = _drain_flags(dev)
    if mode == "error":
        _raise_on(f)
    elif f & abi.FLAG_CAST_LOSS:
        dtypes.emit_warning("cast lost information (value out of range or not representable)")


def _raise_on(flags: int) -> None:
    if flags & abi.FLAG_CAST_LOSS:
        raise DomainError("value cannot be represented in the destination dtype")
    if flags & abi.FLAG_INT_DIV0:
        raise DomainError("integer division by zero")
    if flags & abi.FLAG_DOMAIN:
        raise DomainError("input outside the real domain in error mode")


def _dev(buf) -> int:
    """Device index of a table-entry buffer (a Storage)."""
    return buf.device.index


# ---------------------------------------------------------------------------
# entries
# ---------------------------------------------------------------------------
def binary_entry(op_name):
    code = abi.BINARY_CODE[op_name]

    def entry(plan, d_buf, store, a_buf, a_unpack, b_buf, b_unpack, fn, bases):
        L = _native.lib()
        p = plan.to_c()
        d = dest(d_buf, bases[0], store)
        a = operand(a_buf, bases[1], a_unpack)
        b = operand(b_buf, bases[2], b_unpack)
        mode = dtypes.MODE_CODE[store.mode]
        comp = fn.compute.code
        args = (_sh(), code, C.byref(p), C.byref(d), C.byref(a), C.byref(b), comp, mode)
        _guarded(store.mode, lambda: L.tpg_binary(*args), lambda: L.tpg_binary_check(*args),
                 _dev(d_buf))

    entry.__name__ = f"gpu_{op_name}"
    return entry


def unary_entry(op_name):
    code = abi.UNARY_CODE[op_name]

    def entry(plan, d_buf, store, a_buf, a_unpack, fn, bases):
        L = _native.lib()
        p = plan.to_c()
        d = dest(d_buf, bases[0], store)
        a = operand(a_buf, bases[1], a_unpack)
        mode = dtypes.MODE_CODE[store.mode]
        if op_name == "identity":
            comp, fc = a_unpack.dtype.code, 0
        else:
            comp, fc = fn.compute.code, int(bool(fn.force_complex))
        args = (_sh(), code, C.byref(p), C.byref(d), C.byref(a), comp, mode, fc)
        _guarded(store.mode, lambda: L.tpg_unary(*args), lambda: L.tpg_unary_check(*args),
                 _dev(d_buf))

    entry.__name__ = f"gpu_{op_name}"
    return entry


def reduce_entry(op_name):
    code = abi.REDUCE_CODE[op_name]

    def entry(outer, inner, d_buf, store, a_buf, a_unpack, init, step, fin, bases):
        L = _native.lib()
        po, pi = outer.to_c(), inner.to_c()
        d = dest(d_buf, bases[0], store)
        a = operand(a_buf, bases[1], a_unpack)
        mode = dtypes.MODE_CODE[store.mode]
        acc = init
        args = (_sh(), code, float(acc.p), C.byref(po), C.byref(pi), C.byref(d), C.byref(a),
                acc.compute.code, mode)
        _guarded(store.mode, lambda: L.tpg_reduce(*args), None, _dev(d_buf))

    entry.__name__ = f"gpu_reduce_{op_name}"
    return entry


def matmul_entry(d_buf, d_base, d_strides, store, a_buf, a_base, a_strides, a_unpack,
                 b_buf, b_base, b_strides, b_unpack, m, n, k, mul, init, step, fin):
    L = _native.lib()
    d = dest(d_buf, d_base, store)
    a = operand(a_buf, a_base, a_unpack)
    b = operand(b_buf, b_base, b_unpack)
    ds = (C.c_int64 * 2)(*d_strides)
    as_ = (C.c_int64 * 2)(*a_strides)
    bs = (C.c_int64 * 2)(*b_strides)
    _guarded(store.mode, lambda: L.tpg_matmul(_sh(), C.byref(d), ds, C.byref(a), as_, C.byref(b),
                                              bs, m, n, k, mul.compute.code,
                                              dtypes.MODE_CODE[store.mode]), None, _dev(d_buf))


def matmul_batched_entry(batch, d_buf, d_base, d_strides, store, a_buf, a_base, a_strides,
                         a_unpack, b_buf, b_base, b_strides, b_unpack, m, n, k, mul):
    """Extension entry (no reference op): strides are (row, col, batch)."""
    L = _native.lib()
    d = dest(d_buf, d_base, store)
    a = operand(a_buf, a_base, a_unpack)
    b = operand(b_buf, b_base, b_unpack)
    ds = (C.c_int64 * 3)(*d_strides)
    as_ = (C.c_int64 * 3)(*a_strides)
    bs = (C.c_int64 * 3)(*b_strides)
    _guarded(store.mode, lambda: L.tpg_matmul_batched(_sh(), batch, C.byref(d), ds, C.byref(a),
                                                      as_, C.byref(b), bs, m, n, k,
                                                      mul.compute.code,
                                                      dtypes.MODE_CODE[store.mode]),
             None, _dev(d_buf))


class ChainFn:
    """Descriptor of a fused chain: per step (op, result dtype, compute
    dtype, scalar Codec, scalar_first)."""
    __slots__ = ("steps", "mode")

    def __init__(self, steps, mode="standard"):
        self.steps, self.mode = steps, mode


def chain_entry(plan, d_buf, store, a_buf, a_unpack, fn, bases):
    """Extension entry: one pass for a chain of binary
    ops with by-value scalars, bit-identical to the ops run one by one."""
    L = _native.lib()
    p = plan.to_c()
    d = dest(d_buf, bases[0], store)
    a = operand(a_buf, bases[1], a_unpack)
    n = len(fn.steps)
    arr = (abi.ChainStep * n)()
    for i, (op, rdt, comp, codec, sfirst) in enumerate(fn.steps):
        arr[i].op = abi.BINARY_CODE[op]
        arr[i].dtype = rdt.code
        arr[i].compute = comp.code
        arr[i].scalar_first = 1 if sfirst else 0
        arr[i].scalar_dtype = codec.dtype.code
        raw = bytes(codec.imm).ljust(16, b"\0")
        for j in range(16):
            arr[i].scalar[j] = raw[j]
    mode = dtypes.MODE_CODE[store.mode]
    args = (_sh(), C.byref(p), C.byref(d), C.byref(a), n, arr, mode)
    _guarded(store.mode, lambda: L.tpg_chain(*args), lambda: L.tpg_chain_check(*args),
             _dev(d_buf))


def fill_entry(plan, buf, pack, value, base):
    L = _native.lib()
    raw = dtypes.pack_value(pack.dtype, value, pack.byteorder)
    d = abi.make_operand(buf.ptr, base, pack.dtype.code, pack.byteorder == "big")
    cbuf = C.create_string_buffer(raw, len(raw))
    _native.check(L.tpg_fill(_sh(), C.byref(plan.to_c()), C.byref(d), cbuf, len(raw)), "fill")


def arange_entry(plan, buf, pack, cast_fn, base):
    L = _native.lib()
    d = abi.make_operand(buf.ptr, base, pack.dtype.code, pack.byteorder == "big")
    _native.check(L.tpg_arange(_sh(), C.byref(plan.to_c()), C.byref(d)), "arange")


def byteswap_entry(buf, base, plan, dtype, byteorder="little"):
    L = _native.lib()
    d = abi.make_operand(buf.ptr, base, dtype.code, False)
    _native.check(L.tpg_byteswap(_sh(), C.byref(plan.to_c()), C.byref(d)), "byteswap")


def gather_entry(dst_buf, src_buf, pairs, size):
    L = _native.lib()
    arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1))
    n = arr.size // 2
    _native.check(L.tpg_gather(_sh(), dst_buf.ptr, src_buf.ptr,
                               arr.ctypes.data_as(C.POINTER(C.c_int64)), n, size), "gather")


def scatter_entry(pairs, d_buf, store, s_buf, s_unpack):
    L = _native.lib()
    arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1))
    d = dest(d_buf, 0, store)
    s = operand(s_buf, 0, s_unpack)
    _guarded(store.mode, lambda: L.tpg_scatter(_sh(), arr.ctypes.data_as(C.POINTER(C.c_int64)),
                                               arr.size // 2, C.byref(d), C.byref(s),
                                               dtypes.MODE_CODE[store.mode]), None, _dev(d_buf))


def scatter_fill_entry(offsets, d_buf, pack, value):
    L = _native.lib()
    arr = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64).reshape(-1))
    raw = dtypes.pack_value(pack.dtype, value, pack.byteorder)
    cbuf = C.create_string_buffer(raw, len(raw))
    _native.check(L.tpg_scatter_fill(_sh(), arr.ctypes.data_as(C.POINTER(C.c_int64)), arr.size,
                                     d_buf.ptr, cbuf, len(raw)), "scatter_fill")


BINARY_OPS = ("add", "subtract", "multiply", "divide", "minimum", "maximum")
UNARY_OPS = ("negate", "absolute", "square_root", "exponential", "logarithm", "sine", "cosine",
             "arcsine", "arccosine", "conjugate")
REDUCE_OPS = ("sum", "product", "minimum", "maximum", "any", "all", "norm")


def build_core_table() -> dict:
    """Same 31 keys as backend_cpu.build_core_table (backend_cpu.py:10-27)."""
    t = {}
    for op in BINARY_OPS:
        t[op] = binary_entry(op)
    for op in UNARY_OPS:
        t[op] = unary_entry(op)
    t["copy"] = unary_entry("identity")
    for op in REDUCE_OPS:
        t[f"reduce_{op}" if op in ("minimum", "maximum") else op] = reduce_entry(op)
    t["matmul"] = matmul_entry
    t["fill"] = fill_entry
    t["arange"] = arange_entry
    t["byteswap"] = byteswap_entry
    t["gather"] = gather_entry
    t["scatter"] = scatter_entry
    t["scatter_fill"] = scatter_fill_entry
    return t
