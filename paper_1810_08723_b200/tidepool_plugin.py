"""Drop-in adapter: the ("core", "gpu") table for an UNMODIFIED reference
`tidepool` (the north_star boundary).

    import tidepool
    from paper_1810_08723_b200 import tidepool_plugin
    tidepool_plugin.register(tidepool)      # adds device type "gpu"
    g = tidepool.devices.by_name("gpu0")
    x = tidepool.cast(t, device=g)          # H2D through the gpu `copy` entry
    y = tidepool.add(x, 1.5)                # the reference pipeline, B200 kernels

What the reference hands across its function table are Python closures
(`store` = ops._make_store, ops.py:145-152; codec `unpack`/`pack`,
dtypes.py:357-391; scalar `fn`s, kernels.py:50-158; reduction (init, step,
fin) triples, ops.py:522-556).  This module recovers the descriptors those
closures encode (dtype, byte order, mode, CastContext, status set, norm
order) by introspection and makes one C-ABI call per entry.

All arithmetic, cast and status semantics stay the reference's:

* status: the device's sticky flag word is drained, in stream order, into
  the `status` set the reference's scalar functions close over
  (kernels.py:72-78, 151-156 -> ops._status, ops.py:27-38) whenever a gpu
  stream synchronises; `tidepool.get_status()` drains every gpu stream first,
  so flags are visible exactly as on the synchronous cpu device;
* cast loss (error / warning mode): reported through the store's own
  `CastContext.domain_loss` (dtypes.py:233-255), so error mode raises the
  reference's `tidepool.errors.DomainError` before anything is written and
  warning mode warns once through the reference's handler (`ctx.flush()` in
  ops.py:284-285);
* native failures raise the reference's `DeviceError` / `AllocationError`.

B200 mechanics:

* storage = CUDA managed memory (the reference reads and writes storage bytes
  on the host through memoryviews), preferred on the GPU, recycled through a
  bounded per-device cache; a recycled block is handed out only after the
  GPU work that last used it has completed;
* entries enqueue asynchronously on the storage's gpu stream (a
  `devices.Stream` subclass whose `sync()` synchronises the CUDA stream);
  nothing synchronises per entry in standard mode;
* lazy casts: a lossless dtype-converting gpu->gpu `copy`
  (the reference's `_dtype_convert`, ops.py:121-124) is recorded instead of
  launched; a binary entry reading its result converts on load from the
  original source (cfg2: one 6 B/element pass instead of 14 B/element), any
  other consumer, writer or synchronisation materialises it first;
* descriptor transfers: `tensors._raw_gather` (gpu->gpu,
  cpu->gpu, gpu->cpu) and the cpu `copy` entry for gpu sources run as one
  plan-driven kernel plus one bulk PCIe copy instead of the reference's
  per-element Python pair list (tensors.py:686-699).

The closure decoders are also used by tests/golden/make_golden.py to turn
captured reference table calls into golden vectors.
"""

from __future__ import annotations

import collections
import collections.abc
import ctypes as C
import threading

MODE_CODE = {"standard": 0, "warning": 1, "error": 2, "complex": 3}
FLAG_DOMAIN, FLAG_INT_DIV0, FLAG_CAST_LOSS = 1, 2, 4


# ---------------------------------------------------------------------------
# closure decoding
# ---------------------------------------------------------------------------
def _cells(fn) -> dict:
    code = getattr(fn, "__code__", None)
    if code is None or fn.__closure__ is None:
        return {}
    return {n: c.cell_contents for n, c in zip(code.co_freevars, fn.__closure__)}


_CELL_INDEX: dict = {}  # (code object, free variable names) -> closure indices (-1: absent)


def _cells_at(fn, names):
    """Contents of the named closure cells of `fn` (None when absent); the
    name -> index mapping is computed once per code object (the reference
    creates a new store / scalar closure per call, over a handful of code
    objects)."""
    try:
        code, cl = fn.__code__, fn.__closure__
    except AttributeError:
        return (None,) * len(names)
    if cl is None:
        return (None,) * len(names)
    idx = _CELL_INDEX.get((code, names))
    if idx is None:
        fv = code.co_freevars
        idx = _CELL_INDEX[(code, names)] = tuple(fv.index(n) if n in fv else -1 for n in names)
    if len(idx) == 1:
        i = idx[0]
        return (cl[i].cell_contents if i >= 0 else None,)
    return [cl[i].cell_contents if i >= 0 else None for i in idx]


def decode_codec(ref_dtypes, fn):
    """(dtype name, byteorder) of a reference codec unpack/pack function."""
    for (d, order), pair in ref_dtypes._CODEC_CACHE.items():
        if fn is pair[0] or fn is pair[1]:
            return d.name, order
    raise LookupError("function is not a reference codec")


def prime_codecs(ref_dtypes) -> None:
    """Populate every (dtype, byteorder) codec so reverse lookups succeed
    (the cache never evicts, dtypes.py:354-391)."""
    for d in ref_dtypes.ALL_DTYPES:
        for order in ("little", "big"):
            ref_dtypes.codec(d, order)


def decode_store(ref_dtypes, store):
    """(dtype name, byteorder, mode) of an ops._make_store closure (or the
    assign_index store, indexing.py:459-460: same free variables)."""
    cells = _cells(store)
    if set(cells) >= {"pack", "to", "mode"}:
        name, order = decode_codec(ref_dtypes, cells["pack"])
        return cells["to"].name, order, cells["mode"]
    if "pack" in cells:  # a bare pack wrapper (tests wrap pack in a lambda)
        name, order = decode_codec(ref_dtypes, cells["pack"])
        return name, order, "standard"
    raise LookupError("unrecognised store closure")


def unary_forces_complex(fn) -> bool:
    """unary_scalar_fn returns `lambda v: complex_fn(complex(v))` for the
    complex branch (kernels.py:145-146)."""
    code = getattr(fn, "__code__", None)
    return code is not None and code.co_freevars == ("complex_fn",)


def norm_order(step) -> float:
    return float(_cells(step).get("p", 2.0))


# ---------------------------------------------------------------------------
# plan helpers (reference IterPlan: .extents, .strides, .total)
# ---------------------------------------------------------------------------
def _span(extents, strides, base, size):
    """[lo, hi) byte range one plan view touches."""
    lo = hi = base
    for e, s in zip(extents, strides):
        if e > 1:
            if s < 0:
                lo += (e - 1) * s
            else:
                hi += (e - 1) * s
    return lo, hi + size


def _is_dense(extents, strides, size):
    """True when the view enumerates [0, total*size) exactly once in
    column-major order (a fresh tensor_create layout)."""
    step = size
    for e, s in zip(extents, strides):
        if e == 1:
            continue
        if s != step:
            return False
        step *= e
    return True


_FUSE_MEMO: dict = {}


def _fuse_strides(copy_plan, bin_ext, bin_str, a_base, size):
    """Memoised _fuse_strides_impl (the same copy / binary layouts recur
    call after call)."""
    key = (tuple(copy_plan.extents), tuple(map(tuple, copy_plan.strides)), tuple(bin_ext),
           tuple(bin_str), a_base, size)
    r = _FUSE_MEMO.get(key, _FUSE_MEMO)
    if r is _FUSE_MEMO:
        if len(_FUSE_MEMO) > 4096:
            _FUSE_MEMO.clear()
        r = _FUSE_MEMO[key] = _fuse_strides_impl(copy_plan, bin_ext, bin_str, a_base, size)
    return r


def _fuse_strides_impl(copy_plan, bin_ext, bin_str, a_base, size):
    """Re-express a binary operand that reads the (dense) destination of a
    recorded copy as a view of the copy's SOURCE.  Returns (src strides per
    binary axis, src byte offset relative to the copy's source offset) or
    None when the binary view does not map axis-for-axis onto the copy plan
    (the caller then materialises the copy)."""
    E = copy_plan.extents
    T, S = copy_plan.strides[0], copy_plan.strides[1]
    if a_base % size:
        return None
    # the operand's base offset as copy-plan digits (mixed radix E)
    lin, digits = a_base // size, []
    for e in E:
        lin, d = divmod(lin, e) if e else (lin, 0)
        digits.append(d)
    if lin:
        return None
    out, used = [], set()
    for f, b in zip(bin_ext, bin_str):
        if f == 1 or b == 0:
            out.append(0)
            continue
        for j, (e, t) in enumerate(zip(E, T)):
            if t == b and e == f and digits[j] == 0 and j not in used:
                used.add(j)
                out.append(S[j])
                break
        else:
            return None
    return out, sum(d * s for d, s in zip(digits, S))


# ---------------------------------------------------------------------------
# registration into the reference
# ---------------------------------------------------------------------------
def _fast_module():
    """The plugin's C host fast path (hostsrc/tpg_pyfast.c, built in-tree by
    build.py): managed block cache + storage buffer type."""
    try:
        from . import _tpg_pyfast
    except ImportError as exc:  # built by __graft_entry__.build() / build.py
        raise ImportError("paper_1810_08723_b200._tpg_pyfast is not built "
                          "(python -m paper_1810_08723_b200.build)") from exc
    return _tpg_pyfast


_DEVBUF = None  # _tpg_pyfast.DevBuf once the first registration loaded it


def _binary_function(L, abi):
    """Address of tpg_binary for the C entry (a ctypes callback into a
    duck-typed test double)."""
    if isinstance(L, C.CDLL):
        return C.cast(L.tpg_binary, C.c_void_p).value
    PP, PO = C.POINTER(abi.Plan), C.POINTER(abi.Operand)
    cb = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, PP, PO, PO, PO, C.c_int, C.c_int)(
        lambda st, op, p, d, a, b, comp, mode: L.tpg_binary(st, op, p.contents, d.contents,
                                                            a.contents, b.contents, comp, mode))
    _CALLBACKS.append(cb)
    return C.cast(cb, C.c_void_p).value


def _unary_function(L, abi):
    """Address of tpg_unary for the C entry (a ctypes callback into a
    duck-typed test double)."""
    if isinstance(L, C.CDLL):
        return C.cast(L.tpg_unary, C.c_void_p).value
    PP, PO = C.POINTER(abi.Plan), C.POINTER(abi.Operand)
    cb = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, PP, PO, PO, C.c_int, C.c_int, C.c_int)(
        lambda st, op, p, d, a, comp, mode, fc: L.tpg_unary(st, op, p.contents, d.contents,
                                                            a.contents, comp, mode, fc))
    _CALLBACKS.append(cb)
    return C.cast(cb, C.c_void_p).value


def _reduce_function(L, abi):
    """Address of tpg_reduce for the C entry (a ctypes callback into a
    duck-typed test double)."""
    if isinstance(L, C.CDLL):
        return C.cast(L.tpg_reduce, C.c_void_p).value
    PP, PO = C.POINTER(abi.Plan), C.POINTER(abi.Operand)
    cb = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_double, PP, PP, PO, PO, C.c_int, C.c_int)(
        lambda st, op, pn, po, pi, d, a, comp, mode: L.tpg_reduce(
            st, op, pn, po.contents, pi.contents, d.contents, a.contents, comp, mode))
    _CALLBACKS.append(cb)
    return C.cast(cb, C.c_void_p).value


_CALLBACKS: list = []  # ctypes callbacks handed to C (kept alive)


def _pool_functions(L):
    """Addresses of the six C-ABI functions the block pool calls.  For a
    ctypes library they are the exported symbols; for a duck-typed test
    double (tests/fake_native.py) they are ctypes callbacks into it."""
    if isinstance(L, C.CDLL):
        names = ("tpg_malloc_managed", "tpg_free_managed", "tpg_event_create_untimed",
                 "tpg_event_record", "tpg_event_query", "tpg_event_sync",
                 "tpg_mark_word_create", "tpg_stream_mark")
        return tuple(C.cast(getattr(L, n), C.c_void_p).value for n in names), ()
    I, P, PP = C.c_int, C.c_void_p, C.POINTER(C.c_void_p)

    def malloc_managed(dev, n, out):
        v = P()
        rc = L.tpg_malloc_managed(dev, n, C.byref(v))
        out[0] = v.value
        return rc

    def ev_create(out):
        v = P()
        rc = L.tpg_event_create_untimed(C.byref(v))
        out[0] = v.value
        return rc
    words = []  # the test double's "device" is synchronous: a mark is set at once

    def mark_create(out):
        w = C.c_uint64(0)
        words.append(w)
        out[0] = C.addressof(w)
        return 0

    def mark(st, word, value):
        if getattr(L, "fail_marks", False):  # test hook: no stream memory ops -> events
            return -4
        C.c_uint64.from_address(word).value = value
        return 0
    cbs = (C.CFUNCTYPE(I, I, C.c_size_t, PP)(malloc_managed),
           C.CFUNCTYPE(I, P)(lambda p: L.tpg_free_managed(p)),
           C.CFUNCTYPE(I, PP)(ev_create),
           C.CFUNCTYPE(I, P, P)(lambda e, st: L.tpg_event_record(e, st)),
           C.CFUNCTYPE(I, P)(lambda e: L.tpg_event_query(e)),
           C.CFUNCTYPE(I, P)(lambda e: L.tpg_event_sync(e)),
           C.CFUNCTYPE(I, PP)(mark_create),
           C.CFUNCTYPE(I, P, P, C.c_uint64)(mark),
           words)
    return tuple(C.cast(f, C.c_void_p).value for f in cbs[:8]), cbs


class _Stats(collections.abc.Mapping):
    """Path counters (lazy / fused / materialized / staged / ...): the Python
    entries bump them here, the C entries count in C (Entries.counts());
    reads add both."""

    def __init__(self):
        self.py = collections.Counter()
        self.entries = None

    def bump(self, key, n=1):
        self.py[key] += n

    def _c(self):
        if self.entries is None:
            return {}
        c = self.entries.counts()
        return {"lazy": c["lazy"], "fused": c["fused"]}

    def __getitem__(self, key):
        return self.py[key] + self._c().get(key, 0)

    def __iter__(self):
        return iter(set(self.py) | set(self._c()))

    def __len__(self):
        return len(set(self.py) | set(self._c()))


class _Runtime:
    """Per-registration state: devices, streams, block cache, lazy casts."""

    CACHE_BYTES = 8 << 30  # per device; beyond this released blocks are freed

    def __init__(self, tp, L):
        self.tp, self.L = tp, L
        self.errors = tp.errors
        self.lock = threading.RLock()
        self.tls = threading.local()
        self.blocks: dict = {}        # ptr -> (device, cap) of live managed blocks
        self.streams: dict = {}       # device -> [GpuStream] (for free tracking)
        self.lazy: dict = {}          # dst ptr -> _Lazy
        self.lazy_by_src: dict = {}   # src ptr -> {dst ptr}
        self.status_sink = tp.ops._status
        fast = _fast_module()
        global _DEVBUF
        _DEVBUF = fast.DevBuf
        fast.set_allocation_error(tp.errors.AllocationError)
        fns, self._pool_callbacks = _pool_functions(L)
        self.pool = fast.BlockPool(fns, self.blocks, self.lazy, self.lazy_by_src,
                                   self.CACHE_BYTES, self.MAX_PENDING)
        self.DevBuf = fast.DevBuf
        self.defaults: dict = {}     # device -> its default GpuStream (rt.current)
        self.event_pool: list = []   # timing events (profile hook)
        self.plans: dict = {}    # (extents, strides) -> abi.Plan (entries rebuild plans per call)
        self.stats = _Stats()  # lazy / fused / materialised / transfer paths
        self.profile = None  # [] -> (start, stop) timing events around each standard-mode launch

    # -- errors --------------------------------------------------------------
    def check(self, rc, what):
        if rc == 0:
            return
        msg = f"{what}: {self.L.tpg_last_error().decode()}"
        if rc == -2:
            raise self.errors.AllocationError(msg)
        raise self.errors.DeviceError(msg)

    # -- memory --------------------------------------------------------------
    MAX_PENDING = 8  # per size class: beyond this many in-flight blocks, wait for the oldest

    def allocate(self, device, nbytes):
        """A storage buffer over a managed block (tpg_pyfast.c BlockPool:
        recycled blocks are handed out only once the GPU work that last
        used them has completed -- host code may write a fresh storage
        without synchronising, e.g. tensor_from_nested / scalar_tensor,
        tensors.py:221-243, 269-280)."""
        return self.pool.allocate(device, nbytes)

    def _new_timing_event(self):
        ev = C.c_void_p()
        self.check(self.L.tpg_event_create(C.byref(ev)), "event create")
        return ev.value

    def _new_event(self):
        ev = C.c_void_p()
        self.check(self.L.tpg_event_create_untimed(C.byref(ev)), "event create")
        return ev.value

    def trim(self, device, keep_bytes):
        """Free cached blocks of `device` until at most keep_bytes remain."""
        self.pool.trim(device, keep_bytes)

    # -- pointers --------------------------------------------------------------
    @staticmethod
    def address(mv):
        """Raw address of a storage memoryview (read-only views included)."""
        obj = mv.obj
        if type(obj) is _DEVBUF:
            return obj.ptr
        if len(mv) == 0:
            return 0
        import numpy as np
        return int(np.frombuffer(mv, dtype=np.uint8).ctypes.data)

    def is_gpu(self, ptr) -> bool:
        return ptr in self.blocks

    # -- streams ----------------------------------------------------------------
    def current(self, device):
        self.pool.bump()  # a new launch epoch for the blocks' completion markers
        st = getattr(self.tls, "stream", None)
        if st is not None and st.device.index == device:
            return st
        st = self.defaults.get(device)
        if st is None:
            st = self.defaults[device] = self.devices[device].default_stream()
        return st

    def drain(self, st):
        """Stream-ordered read-and-clear of the device's status word; status
        bits go to the reference's status set."""
        f = C.c_uint32(0)
        self.check(self.L.tpg_flags_take(st.handle, C.byref(f)), "status flags")
        bits = f.value
        kernels = self.tp.kernels
        if bits & FLAG_DOMAIN:
            self.status_sink.add(kernels.STATUS_DOMAIN)
        if bits & FLAG_INT_DIV0:
            self.status_sink.add(kernels.STATUS_INT_DIV_ZERO)
        return bits

    # -- lazy casts -------------------------------------------------------------
    def _drop_lazy_locked(self, dst_ptr):
        lz = self.lazy.pop(dst_ptr, None)
        if lz is not None:
            srcs = self.lazy_by_src.get(lz.src_ptr)
            if srcs is not None:
                srcs.discard(dst_ptr)
                if not srcs:
                    del self.lazy_by_src[lz.src_ptr]
        return lz

    def materialize(self, dst_ptr):
        with self.lock:
            lz = self._drop_lazy_locked(dst_ptr)
        if lz is not None:
            self.stats.bump("materialized")
            lz.launch(self)

    def before_read(self, ptr):
        if ptr in self.lazy:
            self.materialize(ptr)

    def before_write(self, ptr):
        if ptr in self.lazy:
            self.materialize(ptr)
        srcs = self.lazy_by_src.get(ptr)
        if srcs:
            for d in list(srcs):
                self.materialize(d)

    def materialize_device(self, device, stream=None):
        """Launch the pending copies of `device` (recorded on `stream`, or
        on any stream when None)."""
        with self.lock:
            todo = [p for p, lz in self.lazy.items()
                    if lz.device == device and (stream is None or lz.stream is stream)]
        for p in todo:
            self.materialize(p)


try:  # the C host fast path (built in-tree; register() requires it)
    from . import _tpg_pyfast as _fastmod
except ImportError:
    _fastmod = None


class _Lazy(_fastmod.LazyRecord if _fastmod is not None else object):
    """A recorded dtype-converting gpu->gpu copy (ops._dtype_convert).  The
    fields live in the C base (tpg_pyfast.c LazyRecord), which the C copy
    entry fills and the C binary entry reads directly."""
    __slots__ = () if _fastmod is not None else (
        "device", "plan", "dst_ptr", "ddt", "dbig", "src_ptr", "keep", "src_dtype", "dst_dtype",
        "src_order", "stream", "cext", "cdst", "csrc", "sbase", "soff", "sdt", "sbig")

    def launch(self, rt):
        """Launch on the stream the copy entry ran on (the destination
        storage's stream, where the reference orders its consumers); a
        consumer on another stream of this thread waits for it."""
        st = self.stream
        p = rt.abi.make_plan(self.plan.extents, self.plan.strides)
        d = rt.abi.make_operand(self.dst_ptr, 0, self.ddt, self.dbig)
        a = rt.abi.make_operand(self.sbase, self.soff, self.sdt, self.sbig)
        rt.check(rt.L.tpg_unary(st.handle, 10, C.byref(p), C.byref(d), C.byref(a), self.sdt, 0,
                                0), "copy")
        cur = getattr(rt.tls, "stream", None)
        if cur is not None and cur is not st and cur.device.index == self.device:
            rt.check(rt.L.tpg_stream_wait(cur.handle, st.handle), "stream wait")


def register(tidepool_module, count: int | None = None, lib=None):
    """Attach B200 gpu devices and the ("core", "gpu") table to `tidepool`.

    Returns the registered devices (gpu0, gpu1, ...).  `lib` is a test hook
    (tests/fake_native.py); the product always uses libtidepool_gpu.so."""
    import numpy as np

    from . import _native, abi

    tp = tidepool_module
    ref_devices, ref_dispatch, ref_dtypes = tp.devices, tp.dispatch, tp.dtypes
    ref_tensors, ref_ops = tp.tensors, tp.ops
    errors = tp.errors
    prime_codecs(ref_dtypes)
    try:
        L = lib if lib is not None else _native.lib()
    except Exception as exc:  # no library / no device: the reference's own error class
        raise errors.DeviceError(f"gpu device module unavailable: {exc}") from exc
    rt = _Runtime(tp, L)
    rt.abi = abi
    gpu_type = ref_devices.DeviceType("gpu", supports_byteswapped=True, async_capable=False)
    codec_of = {}
    for (d, order), pair in ref_dtypes._CODEC_CACHE.items():
        codec_of[pair[0]] = codec_of[pair[1]] = (d, order)
    fast_codecs = {f: (d.wire_code, d.size, int(order == "big"),
                       ref_dtypes.widen_for_compute(d).wire_code)
                   for f, (d, order) in codec_of.items()}
    rt.entries = _fast_module().Entries(rt.pool, _binary_function(L, abi), rt, rt.tls, rt.lazy,
                                        rt.lazy_by_src, fast_codecs, rt.stats.py)
    rt.stats.entries = rt.entries
    lossless_table = bytearray(32 * 32)
    for a_ in ref_dtypes.ALL_DTYPES:
        for b_ in ref_dtypes.ALL_DTYPES:
            lossless_table[a_.wire_code * 32 + b_.wire_code] = \
                int(bool(ref_dtypes.lossless_castable(a_, b_)))
    rt.entries.set_copy_support(_Lazy, dict(codec_of), bytes(lossless_table))
    rt.entries.set_unary(_unary_function(L, abi))
    rt.entries.set_reduce(_reduce_function(L, abi))

    # -- devices and streams ------------------------------------------------------
    class GpuStream(ref_devices.Stream):
        """A reference Stream bound to one CUDA stream.  Work is enqueued by
        the calling thread (submit runs the task inline, which only launches
        kernels); sync() waits for the CUDA stream and drains its status."""

        def __init__(self, device, handle=None):
            super().__init__(device)
            if handle is None:
                h = C.c_void_p()
                rt.check(L.tpg_stream_create(device.index, C.byref(h)), "stream create")
                handle = h.value
            self.handle = handle
            rt.streams.setdefault(device.index, []).append(self)
            rt.pool.add_stream(device.index, handle)

        is_default = False  # set on the device's default stream

        def submit(self, task) -> None:
            prev = getattr(rt.tls, "stream", None)
            if prev is None and self.is_default:
                task()  # rt.current() resolves to this stream anyway
                return
            rt.tls.stream = self
            try:
                task()
            finally:
                rt.tls.stream = prev

        def sync(self) -> None:
            rt.materialize_device(self.device.index, self)
            rt.drain(self)
            super().sync()

    class GpuDevice(ref_devices.Device):
        def __init__(self, index):
            super().__init__(gpu_type, index)
            # Device.allocate in C (tpg_pyfast.c Allocator: the same checks
            # and alloc_count accounting as allocate() below)
            self.allocate = rt.pool.allocator(index, self)

        def default_stream(self):
            st = self._default_stream  # set once; read without the lock afterwards
            if st is not None:
                return st
            with self._lock:
                if self._default_stream is None:
                    h = C.c_void_p()
                    rt.check(L.tpg_default_stream(self.index, C.byref(h)), "default stream")
                    self._default_stream = GpuStream(self, h.value)
                    rt.entries.set_default_stream(self.index, h.value, self._default_stream)
                    rt.defaults[self.index] = self._default_stream
                    self._default_stream.is_default = True
                return self._default_stream

        def allocate(self, nbytes):
            if nbytes < 0:
                raise errors.AllocationError("negative allocation size")
            with self._lock:
                self.alloc_count += 1
            return rt.allocate(self.index, nbytes)

        @property
        def properties(self):
            props = super().properties
            p = abi.DeviceProps()
            rt.check(L.tpg_device_props_get(self.index, C.byref(p)), "device properties")
            props.update({"name": p.name.decode(), "processor-count": str(p.sm_count),
                          "free-memory": str(p.free_mem), "total-memory": str(p.total_mem)})
            return props

        def synchronize(self):
            for st in list(rt.streams.get(self.index, ())):
                st.sync()

    # -- operands ---------------------------------------------------------------------
    class _Temps:
        """Device staging for host-resident operands of one entry; freed in
        stream order after the entry's kernel."""

        def __init__(self, st):
            self.st, self.ptrs = st, []

        def stage(self, host_ptr, lo, hi):
            n = hi - lo
            p = C.c_void_p()
            rt.check(L.tpg_malloc_on(self.st.handle, n, C.byref(p)), "staging")
            self.ptrs.append(p.value)
            rt.stats.bump("staged")
            # pageable source: returns once the bytes are consumed
            rt.check(L.tpg_memcpy_h2d(p.value, host_ptr + lo, n, self.st.handle), "H2D")
            return p.value - lo

        def done(self):
            for p in self.ptrs:
                L.tpg_free(self.st.device.index, p, self.st.handle)

    def _codec(fn):
        try:
            return codec_of[fn]
        except KeyError:
            d, order = decode_codec(ref_dtypes, fn)
            return ref_dtypes.by_name(d), order

    _STORE_CELLS = ("pack", "mode", "ctx")

    def _store(store):
        pack, mode, ctx = _cells_at(store, _STORE_CELLS)
        if pack is None:
            raise errors.DeviceError("gpu table: unrecognised store closure")
        d, order = _codec(pack)
        return d, order, mode if mode is not None else "standard", ctx

    def _operand(ptr, base, d, order, temps, extents=None, strides=None):
        """tpg_operand for a storage pointer; host memory is staged."""
        if ptr and not rt.is_gpu(ptr):
            if extents is None:
                raise errors.DeviceError("gpu table: host operand without a plan")
            lo, hi = _span(extents, strides, base, d.size)
            if hi > lo:
                ptr = temps.stage(ptr, lo, hi)
        return abi.make_operand(ptr, base, d.wire_code, order == "big")

    def _plan(pl, strides=None):
        ext = tuple(pl.extents)
        strd = tuple(map(tuple, strides if strides is not None else pl.strides))
        key = (ext, strd)
        p = rt.plans.get(key)
        if p is None:
            if len(rt.plans) > 4096:
                rt.plans.clear()
            p = rt.plans[key] = abi.make_plan(ext, strd)
        return p

    def _loss_message(d):
        return f"value cannot be represented as {d.name}"

    def _timed(st, launch):
        """Launch, bracketed by an event pair when profiling is on
        (rt.profile = []: collects (start, stop) events per launch)."""
        if rt.profile is None:
            return launch()
        a, b = rt._new_timing_event(), rt._new_timing_event()
        L.tpg_event_record(a, st.handle)
        rc = launch()
        L.tpg_event_record(b, st.handle)
        rt.profile.append((a, b))
        return rc

    def _run(st, mode, ctx, to, launch, check=None):
        """Launch with the reference's mode semantics (cast loss -> ctx)."""
        if mode in ("standard", "complex"):
            rt.check(_timed(st, launch), "kernel")
            return
        rt.drain(st)
        if mode == "error" and check is not None:
            rt.check(check(), "kernel check")
            bits = rt.drain(st)
            if bits & FLAG_INT_DIV0:
                raise errors.DomainError("integer division by zero")
            if bits & FLAG_CAST_LOSS:
                if ctx is not None:
                    ctx.domain_loss(_loss_message(to))
                raise errors.DomainError(_loss_message(to))
            rt.check(launch(), "kernel")
            return
        rt.check(launch(), "kernel")
        bits = rt.drain(st)
        if bits & FLAG_CAST_LOSS:
            if ctx is not None:
                ctx.domain_loss(_loss_message(to))   # error: raises; warning: recorded
            elif mode == "error":
                raise errors.DomainError(_loss_message(to))

    _STATUS_CELL = ("status",)

    def _sink(fn):
        s = _cells_at(fn, _STATUS_CELL)[0]
        if isinstance(s, set):
            rt.status_sink = s

    compute_code = {}

    def _compute(d):
        """wire code of widen_for_compute(d) (memoised per dtype)."""
        c = compute_code.get(d)
        if c is None:
            c = compute_code[d] = ref_dtypes.widen_for_compute(d).wire_code
        return c

    # -- entries (SURVEY §8b signatures) -------------------------------------------
    def binary(op):
        code = abi.BINARY_CODE[op]

        def h(plan, d_buf, store, a_buf, a_unpack, b_buf, b_unpack, fn, bases):
            dd, dord, mode, ctx = _store(store)
            da, aord = _codec(a_unpack)
            db, bord = _codec(b_unpack)
            dptr, aptr, bptr = rt.address(d_buf), rt.address(a_buf), rt.address(b_buf)
            dev = rt.blocks[dptr][0]
            st = rt.current(dev)
            _sink(fn)
            compute = _compute(da)
            temps = _Temps(st)
            ops, strides = [], [list(plan.strides[0])]
            for ptr, d, order, base, v in ((aptr, da, aord, bases[1], 1),
                                           (bptr, db, bord, bases[2], 2)):
                fused = None
                lz = rt.lazy.get(ptr)
                if lz is not None and lz.src_ptr != dptr:
                    fused = _fuse_strides(lz.plan, plan.extents, plan.strides[v], base, d.size)
                if fused is not None:
                    s, off = fused
                    with rt.lock:
                        keep = rt.lazy.get(ptr) is lz
                    if keep:
                        rt.stats.bump("fused")
                        o = abi.make_operand(lz.sbase, lz.soff + off, lz.sdt, lz.sbig)
                        ops.append(o)
                        strides.append(s)
                        continue
                rt.before_read(ptr)
                ops.append(_operand(ptr, base, d, order, temps, plan.extents, plan.strides[v]))
                strides.append(list(plan.strides[v]))
            rt.before_write(dptr)
            p = _plan(plan, strides)
            dop = abi.make_operand(dptr, bases[0], dd.wire_code, dord == "big")
            args = (st.handle, code, C.byref(p), C.byref(dop), C.byref(ops[0]), C.byref(ops[1]),
                    compute, MODE_CODE[mode])
            _run(st, mode, ctx, dd, lambda: L.tpg_binary(*args), lambda: L.tpg_binary_check(*args))
            temps.done()
        h.__name__ = f"gpu_{op}"
        # the table entry: C fast path (standard mode, gpu operands of one
        # device; tpg_pyfast.c FastEntry), this Python entry otherwise
        return rt.entries.entry(0, code, h)

    def unary(op):
        code = abi.UNARY_CODE[op]

        def h(plan, d_buf, store, a_buf, a_unpack, fn, bases):
            dd, dord, mode, ctx = _store(store)
            da, aord = _codec(a_unpack)
            dptr, aptr = rt.address(d_buf), rt.address(a_buf)
            dev = rt.blocks[dptr][0]
            st = rt.current(dev)
            if op != "identity":
                _sink(fn)
            if op == "identity" and _try_lazy(plan, dptr, dd, dord, mode, aptr, da, aord, bases,
                                             a_buf, dev):
                return
            rt.before_read(aptr)
            rt.before_write(dptr)
            temps = _Temps(st)
            a = _operand(aptr, bases[1], da, aord, temps, plan.extents, plan.strides[1])
            dop = abi.make_operand(dptr, bases[0], dd.wire_code, dord == "big")
            p = _plan(plan)
            if op == "identity":
                comp, fc = da.wire_code, 0
            else:
                comp = _compute(da)
                fc = int(unary_forces_complex(fn) and not da.is_complex)
            args = (st.handle, code, C.byref(p), C.byref(dop), C.byref(a), comp, MODE_CODE[mode],
                    fc)
            _run(st, mode, ctx, dd, lambda: L.tpg_unary(*args), lambda: L.tpg_unary_check(*args))
            temps.done()
        h.__name__ = f"gpu_{op}"
        if op == "identity":
            return h
        # unary ops: C fast path (standard mode, real gpu operands of one
        # device; tpg_pyfast.c FastEntry kind 2), this Python entry otherwise
        return rt.entries.entry(2, code, h)

    lossless = {}

    def _lossless(a, b):
        r = lossless.get((a, b))
        if r is None:
            r = lossless[(a, b)] = bool(ref_dtypes.lossless_castable(a, b))
        return r

    def _try_lazy(plan, dptr, dd, dord, mode, aptr, da, aord, bases, a_buf, dev):
        """Record a lossless gpu->gpu dtype conversion into a fresh dense
        tensor instead of launching it (ops._dtype_convert, ops.py:121-124)."""
        if (mode != "standard" or da is dd or bases[0] != 0 or not rt.is_gpu(aptr)
                or aptr == dptr or rt.blocks[aptr][0] != dev or aptr in rt.lazy
                or not _lossless(da, dd)
                or not _is_dense(plan.extents, plan.strides[0], dd.size)
                or plan.total == 0):
            return False
        lz = _Lazy()
        lz.device, lz.plan = dev, plan
        lz.stream = rt.current(dev)
        lz.dst_ptr, lz.src_ptr = dptr, aptr
        lz.ddt, lz.dbig = dd.wire_code, int(dord == "big")
        lz.keep = a_buf  # the source storage stays alive while the copy is pending
        lz.src_dtype, lz.dst_dtype, lz.src_order = da, dd, aord
        lz.cext, lz.cdst, lz.csrc = tuple(plan.extents), tuple(plan.strides[0]), tuple(plan.strides[1])
        lz.sbase, lz.soff, lz.sdt, lz.sbig = aptr, bases[1], da.wire_code, int(aord == "big")
        rt.before_write(dptr)
        rt.stats.bump("lazy")
        with rt.lock:
            rt.lazy[dptr] = lz
            rt.lazy_by_src.setdefault(aptr, set()).add(dptr)
        return True

    def reduce_(op):
        code = abi.REDUCE_CODE[op]

        def h(outer, inner, d_buf, store, a_buf, a_unpack, init, step, fin, bases):
            dd, dord, mode, ctx = _store(store)
            da, aord = _codec(a_unpack)
            dptr, aptr = rt.address(d_buf), rt.address(a_buf)
            dev = rt.blocks[dptr][0]
            st = rt.current(dev)
            p = norm_order(step) if op == "norm" else 2.0
            rt.before_read(aptr)
            rt.before_write(dptr)
            temps = _Temps(st)
            if aptr and not rt.is_gpu(aptr):
                ext = tuple(outer.extents) + tuple(inner.extents)
                strd = tuple(outer.strides[1]) + tuple(inner.strides[0])
                a = _operand(aptr, bases[1], da, aord, temps, ext, strd)
            else:
                a = abi.make_operand(aptr, bases[1], da.wire_code, aord == "big")
            dop = abi.make_operand(dptr, bases[0], dd.wire_code, dord == "big")
            po, pi = _plan(outer), _plan(inner)
            comp = _compute(da)
            args = (st.handle, code, float(p), C.byref(po), C.byref(pi), C.byref(dop), C.byref(a),
                    comp, MODE_CODE[mode])
            _run(st, mode, ctx, dd, lambda: L.tpg_reduce(*args))
            temps.done()
        h.__name__ = f"gpu_reduce_{op}"
        # C fast path (standard mode, gpu operands of one device), this
        # Python entry otherwise (kind 4: the norm, whose order is read from
        # the step closure)
        return rt.entries.entry(4 if op == "norm" else 3, code, h)

    def matmul(d_buf, d_base, d_strides, store, a_buf, a_base, a_strides, a_unpack, b_buf,
               b_base, b_strides, b_unpack, m, n, k, mul, init, step, fin):
        dd, dord, mode, ctx = _store(store)
        da, aord = _codec(a_unpack)
        db, bord = _codec(b_unpack)
        dptr, aptr, bptr = rt.address(d_buf), rt.address(a_buf), rt.address(b_buf)
        dev = rt.blocks[dptr][0]
        st = rt.current(dev)
        rt.before_read(aptr)
        rt.before_read(bptr)
        rt.before_write(dptr)
        temps = _Temps(st)
        a = _operand(aptr, a_base, da, aord, temps, (m, k), a_strides)
        b = _operand(bptr, b_base, db, bord, temps, (k, n), b_strides)
        dop = abi.make_operand(dptr, d_base, dd.wire_code, dord == "big")
        ds, as_, bs = ((C.c_int64 * 2)(*s) for s in (d_strides, a_strides, b_strides))
        comp = _compute(da)
        _run(st, mode, ctx, dd, lambda: L.tpg_matmul(st.handle, C.byref(dop), ds, C.byref(a), as_,
                                                     C.byref(b), bs, m, n, k, comp,
                                                     MODE_CODE[mode]))
        temps.done()

    def fill(plan, buf, pack, value, base):
        d, order = _codec(pack)
        ptr = rt.address(buf)
        st = rt.current(rt.blocks[ptr][0])
        rt.before_write(ptr)
        raw = bytearray(d.size)
        pack(raw, 0, value)  # the reference's own packing: exact element bytes
        cbuf = C.create_string_buffer(bytes(raw), d.size)
        dop = abi.make_operand(ptr, base, d.wire_code, order == "big")
        rt.check(L.tpg_fill(st.handle, C.byref(_plan(plan)), C.byref(dop), cbuf, d.size), "fill")

    def arange(plan, buf, pack, cast_fn, base):
        d, order = _codec(pack)
        ptr = rt.address(buf)
        st = rt.current(rt.blocks[ptr][0])
        rt.before_write(ptr)
        dop = abi.make_operand(ptr, base, d.wire_code, order == "big")
        rt.check(L.tpg_arange(st.handle, C.byref(_plan(plan)), C.byref(dop)), "arange")

    def byteswap(buf, base, plan, dtype):
        ptr = rt.address(buf)
        st = rt.current(rt.blocks[ptr][0])
        rt.before_write(ptr)
        dop = abi.make_operand(ptr, base, dtype.wire_code, False)
        rt.check(L.tpg_byteswap(st.handle, C.byref(_plan(plan)), C.byref(dop)), "byteswap")

    def _pairs(pairs):
        arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1))
        return arr, arr.ctypes.data_as(C.POINTER(C.c_int64))

    def _stage_whole(ptr, nbytes, temps):
        if ptr and not rt.is_gpu(ptr) and nbytes:
            return temps.stage(ptr, 0, nbytes)
        return ptr

    def gather(dst_buf, src_buf, pairs, size):
        dptr, sptr = rt.address(dst_buf), rt.address(src_buf)
        st = rt.current(rt.blocks[dptr][0])
        rt.before_read(sptr)
        rt.before_write(dptr)
        arr, pp = _pairs(pairs)
        temps = _Temps(st)
        sptr = _stage_whole(sptr, len(src_buf), temps)
        rt.check(L.tpg_gather(st.handle, dptr, sptr, pp, arr.size // 2, size), "gather")
        temps.done()

    def scatter(pairs, d_buf, store, s_buf, s_unpack):
        dd, dord, mode, ctx = _store(store)
        ds_, sord = _codec(s_unpack)
        dptr, sptr = rt.address(d_buf), rt.address(s_buf)
        st = rt.current(rt.blocks[dptr][0])
        rt.before_read(sptr)
        rt.before_write(dptr)
        arr, pp = _pairs(pairs)
        temps = _Temps(st)
        sptr = _stage_whole(sptr, len(s_buf), temps)
        dop = abi.make_operand(dptr, 0, dd.wire_code, dord == "big")
        sop = abi.make_operand(sptr, 0, ds_.wire_code, sord == "big")
        _run(st, mode, ctx, dd, lambda: L.tpg_scatter(st.handle, pp, arr.size // 2, C.byref(dop),
                                                      C.byref(sop), MODE_CODE[mode]))
        temps.done()

    def scatter_fill(offsets, d_buf, pack, value):
        d, order = _codec(pack)
        dptr = rt.address(d_buf)
        st = rt.current(rt.blocks[dptr][0])
        rt.before_write(dptr)
        arr, pp = _pairs(offsets)
        raw = bytearray(d.size)
        pack(raw, 0, value)
        cbuf = C.create_string_buffer(bytes(raw), d.size)
        rt.check(L.tpg_scatter_fill(st.handle, pp, arr.size, dptr, cbuf, d.size), "scatter_fill")

    # -- extension entries (reference dispatch.add_op, dispatch.py:111-117) ------
    def chain_entry(plan, d_buf, store, a_buf, a_unpack, steps, bases):
        """`ewise_chain`: x <- op_i(x, s_i) for a list of (op, result dtype,
        scalar value, scalar_first) in ONE pass (tpg_chain), bit-identical to
        the binary ops one after another."""
        dd, dord, mode, ctx = _store(store)
        da, aord = _codec(a_unpack)
        dptr, aptr = rt.address(d_buf), rt.address(a_buf)
        st = rt.current(rt.blocks[dptr][0])
        rt.before_read(aptr)
        rt.before_write(dptr)
        n = len(steps)
        arr = (abi.ChainStep * n)()
        for i, (op, rdt, value, sfirst) in enumerate(steps):
            raw = bytearray(16)
            ref_dtypes.codec(rdt, "little")[1](raw, 0, ref_dtypes.cast_scalar(value, rdt))
            arr[i].op = abi.BINARY_CODE[op]
            arr[i].dtype = (dd if i == n - 1 else rdt).wire_code
            arr[i].compute = ref_dtypes.widen_for_compute(rdt).wire_code
            arr[i].scalar_first = int(bool(sfirst))
            arr[i].scalar_dtype = rdt.wire_code
            for j in range(16):
                arr[i].scalar[j] = raw[j]
        temps = _Temps(st)
        a = _operand(aptr, bases[1], da, aord, temps, plan.extents, plan.strides[1])
        dop = abi.make_operand(dptr, bases[0], dd.wire_code, dord == "big")
        p = _plan(plan)
        args = (st.handle, C.byref(p), C.byref(dop), C.byref(a), n, arr, MODE_CODE[mode])
        _run(st, mode, ctx, dd, lambda: L.tpg_chain(*args), lambda: L.tpg_chain_check(*args))
        temps.done()

    def matmul_batched_entry(d_buf, d_base, d_strides, store, a_buf, a_base, a_strides, a_unpack,
                             b_buf, b_base, b_strides, b_unpack, m, n, k, nb):
        """`matmul_batched`: nb independent products over the slowest axis
        (tpg_matmul_batched; tcgen05 for 16-bit operands)."""
        dd, dord, mode, ctx = _store(store)
        da, aord = _codec(a_unpack)
        db, bord = _codec(b_unpack)
        dptr, aptr, bptr = rt.address(d_buf), rt.address(a_buf), rt.address(b_buf)
        st = rt.current(rt.blocks[dptr][0])
        for ptr in (aptr, bptr):
            rt.before_read(ptr)
        rt.before_write(dptr)
        temps = _Temps(st)
        a = _operand(aptr, a_base, da, aord, temps, (m, k, nb), a_strides)
        b = _operand(bptr, b_base, db, bord, temps, (k, n, nb), b_strides)
        dop = abi.make_operand(dptr, d_base, dd.wire_code, dord == "big")
        ds, as_, bs = ((C.c_int64 * 3)(*x) for x in (d_strides, a_strides, b_strides))
        comp = _compute(da)
        _run(st, mode, ctx, dd, lambda: L.tpg_matmul_batched(
            st.handle, nb, C.byref(dop), ds, C.byref(a), as_, C.byref(b), bs, m, n, k, comp,
            MODE_CODE[mode]))
        temps.done()

    table = {}
    for op in abi.BINARY_CODE:
        table[op] = binary(op)
    for op in abi.UNARY_CODE:
        if op != "identity":
            table[op] = unary(op)
    # copy: lossless gpu->gpu conversions are recorded in C (the _try_lazy
    # rule, tpg_pyfast.c FastEntry kind 1), everything else in Python
    table["copy"] = rt.entries.entry(1, 0, unary("identity"))
    for op in abi.REDUCE_CODE:
        table[f"reduce_{op}" if op in ("minimum", "maximum") else op] = reduce_(op)
    table.update(matmul=matmul, fill=fill, arange=arange, byteswap=byteswap, gather=gather,
                 scatter=scatter, scatter_fill=scatter_fill)
    ref_dispatch.register_device_impl("core", "gpu", table)
    ref_dispatch.add_op("core", "gpu", "ewise_chain", chain_entry)
    ref_dispatch.add_op("core", "gpu", "matmul_batched", matmul_batched_entry)

    n = C.c_int(0)
    L.tpg_device_count(C.byref(n))
    n = n.value if count is None else min(n.value, count)
    devs = [GpuDevice(i) for i in range(n)]
    rt.devices = {d.index: d for d in devs}
    if n > 1 and hasattr(L, "tpg_enable_peer_all"):
        rt.check(L.tpg_enable_peer_all(C.byref(C.c_int(0))), "peer access")
    ref_devices._devices.extend(devs)

    # the registry is rebuilt by configure(); keep the gpu devices in it
    orig_configure = ref_devices.configure

    def configure(*a, **k):
        orig_configure(*a, **k)
        ref_devices._devices.extend(devs)
    ref_devices.configure = configure

    # streams created for a gpu device are CUDA streams
    orig_create_stream = ref_devices.create_stream

    def create_stream(device):
        if device.type is gpu_type:
            return GpuStream(device)
        return orig_create_stream(device)
    ref_devices.create_stream = create_stream
    tp.create_stream = create_stream

    # status visibility: drain every gpu stream before the reference reads
    # or clears its status set (ops.py:31-38)
    orig_get, orig_clear = ref_ops.get_status, ref_ops.clear_status

    def _drain_all():
        for d in devs:
            for st in list(rt.streams.get(d.index, ())):
                st.sync()

    def get_status():
        _drain_all()
        return orig_get()

    def clear_status():
        _drain_all()
        orig_clear()
    ref_ops.get_status, ref_ops.clear_status = get_status, clear_status
    tp.get_status, tp.clear_status = get_status, clear_status

    # -- descriptor transfers -----------------------------------------
    orig_raw_gather = ref_tensors._raw_gather

    def raw_gather(src, dst):
        """tensors._raw_gather (tensors.py:686-699) for gpu endpoints: one
        canonical 2-view plan and one kernel instead of a Python pair list;
        host endpoints move as one bulk PCIe copy of the touched span."""
        sg, dg = src.device.type is gpu_type, dst.device.type is gpu_type
        if not (sg or dg) or src.dtype.size != dst.dtype.size or src.dims != dst.dims:
            return orig_raw_gather(src, dst)
        total = 1
        for e in dst.dims:
            total *= e
        if total == 0:
            return
        plan = ref_tensors.canonicalize(dst, src)
        size = src.dtype.size
        if not dg:
            # gpu -> host: dense host destinations only (one D2H of the span)
            if not _is_dense(plan.extents, plan.strides[0], size):
                return orig_raw_gather(src, dst)
            src.storage.stream.sync()
            _gather_to_host(plan, src, dst, size)
            return
        if src.storage.stream is not dst.storage.stream:
            src.storage.stream.sync()
        sptr, dptr = rt.address(src.storage.view()), rt.address(dst.storage.view())
        st = dst.storage.stream if isinstance(dst.storage.stream, GpuStream) else \
            dst.device.default_stream()
        rt.before_read(sptr)
        rt.before_write(dptr)
        temps = _Temps(st)
        soff = src.offset
        if not rt.is_gpu(sptr):
            lo, hi = _span(plan.extents, plan.strides[1], src.offset, size)
            sptr = temps.stage(sptr, lo, hi)
        p = _plan(plan)
        rt.stats.bump("gather_plan")
        rt.check(L.tpg_gather_plan(st.handle, C.byref(p), dptr, dst.offset, sptr, soff, size),
                 "gather")
        temps.done()

    def _gather_to_host(plan, src, dst, size):
        st = src.device.default_stream()
        sptr = rt.address(src.storage.view())
        rt.before_read(sptr)
        lo, hi = _span(plan.extents, plan.strides[0], dst.offset, size)
        tmp = C.c_void_p()
        rt.check(L.tpg_malloc_on(st.handle, hi - lo, C.byref(tmp)), "staging")
        p = _plan(plan)
        rt.check(L.tpg_gather_plan(st.handle, C.byref(p), tmp.value - lo, dst.offset, sptr,
                                   src.offset, size), "gather")
        hptr = rt.address(dst.storage.view())
        rt.check(L.tpg_memcpy_d2h(hptr + lo, tmp.value, hi - lo, st.handle), "D2H")
        L.tpg_free(src.device.index, tmp.value, st.handle)
        rt.check(L.tpg_stream_sync(st.handle), "sync")
        rt.stats.bump("gather_to_host")

    raw_gather.reference = orig_raw_gather
    ref_tensors._raw_gather = raw_gather

    # value copies gpu -> cpu (`cast(gpu_t, device=cpu)`, ops._run_copy,
    # ops.py:668-687): the cpu table's `copy` would unpack every element
    # through managed memory; for a gpu source, convert on the GPU into a
    # staging block laid out like the (dense) host destination, then one D2H.
    def cpu_copy_wrapper(original):
        def h(plan, d_buf, store, s_buf, s_unpack, fn, bases):
            sptr = rt.address(s_buf)
            dd, dord, mode, ctx = _store(store)
            if (not rt.is_gpu(sptr) or plan.total == 0
                    or not _is_dense(plan.extents, plan.strides[0], dd.size)):
                return original(plan, d_buf, store, s_buf, s_unpack, fn, bases)
            ds_, sord = _codec(s_unpack)
            dev = rt.blocks[sptr][0]
            st = rt.devices[dev].default_stream()
            rt.before_read(sptr)
            lo, hi = _span(plan.extents, plan.strides[0], bases[0], dd.size)
            tmp = C.c_void_p()
            rt.check(L.tpg_malloc_on(st.handle, hi - lo, C.byref(tmp)), "staging")
            dop = abi.make_operand(tmp.value - lo, bases[0], dd.wire_code, dord == "big")
            sop = abi.make_operand(sptr, bases[1], ds_.wire_code, sord == "big")
            p = _plan(plan)
            args = (st.handle, 10, C.byref(p), C.byref(dop), C.byref(sop), ds_.wire_code,
                    MODE_CODE[mode], 0)
            try:
                _run(st, mode, ctx, dd, lambda: L.tpg_unary(*args),
                     lambda: L.tpg_unary_check(*args))
                hptr = rt.address(d_buf)
                rt.check(L.tpg_memcpy_d2h(hptr + lo, tmp.value, hi - lo, st.handle), "D2H")
                rt.check(L.tpg_stream_sync(st.handle), "sync")
                rt.stats.bump("cpu_copy_from_gpu")
            finally:
                L.tpg_free(dev, tmp.value, st.handle)
        return h

    rt.cpu_copy_restore = ref_dispatch.override_op("core", "cpu", "copy", cpu_copy_wrapper)
    rt.cpu_copy_wrapper = cpu_copy_wrapper
    register.runtime = rt
    _REGISTERED[id(tp)] = (tp, rt)
    return devs


# ---------------------------------------------------------------------------
# extension operators over the reference's own tensors (the reference API
# has no chain and no batched product; these drive the extension entries
# through the reference's dispatch, validation and cast machinery)
# ---------------------------------------------------------------------------
_REGISTERED: dict = {}


def _ref_of(t):
    import sys
    root = type(t).__module__.split(".")[0]
    tp = sys.modules[root]
    if id(tp) not in _REGISTERED:
        raise RuntimeError("tidepool_plugin.register() has not been called for this reference")
    return tp


def chain(x, steps, dest=None, mode="standard"):
    """Fused elementwise chain on a reference tensor:
    `steps` = [(op, scalar) or (op, scalar, scalar_first), ...]; the result
    equals running `tidepool.<op>` step by step (each step's result dtype is
    promote(previous dtype, scalar dtype), ops.py:218-245, and rounds once to
    it) in ONE pass over memory on the gpu device."""
    tp = _ref_of(x)
    dt, tz, ops = tp.dtypes, tp.tensors, tp.ops
    mode = dt.check_mode(mode)
    if not isinstance(x, tz.Tensor):
        raise tp.errors.ShapeError("chain needs a tensor operand")
    if not steps or len(steps) > 8:
        raise ValueError("chain takes 1..8 steps")
    cur, desc = x.dtype, []
    for step in steps:
        op, s = step[0], ops.as_operand(step[1])
        if op not in tp.kernels.BINARY_OPS:
            raise ValueError(f"unknown binary op {op!r}")
        if not isinstance(s, tz.Scalar):
            raise tp.errors.ShapeError("chain steps take scalar operands")
        nxt = cur if not dt.implicit_casting() else dt.promote(cur, s.dtype)
        desc.append((op, nxt, s.value, bool(step[2]) if len(step) > 2 else False))
        cur = nxt
    if dest is None:
        dest = tz.tensor_create(x.dims, cur, x.device)
    else:
        ops._check_dest(dest, x.dims, x.device, cur, mode)
    cleanups = []
    x = ops._resolve_aliasing(x, dest, cleanups, True)
    plan = tz.canonicalize(dest, x)
    ctx = dt.CastContext(mode)
    store = ops._make_store(dest, mode, ctx)
    unpack, _ = dt.codec(x.dtype, x.byteorder)
    handle = tp.dispatch.lookup("core", dest.device.type.name, "ewise_chain")
    ops._sync_other_streams(dest.storage.stream, x)
    d_buf, a_buf = dest.storage.view(), x.storage.view()

    def run():
        handle(plan, d_buf, store, a_buf, unpack, desc, (dest.offset, x.offset))
        ctx.flush()

    dest.storage.stream.submit(run)
    ops._finish(dest.storage.stream, cleanups)
    return dest


def matmul_batched(a, b, dest=None, mode="standard"):
    """Batched product over the slowest axis of reference tensors:
    a (m, k, nb) x b (k, n, nb) -> (m, n, nb); slice i equals
    `tidepool.matmul(a[:, :, i], b[:, :, i])` (its oracle, at the gemm
    tolerance for 16-bit operands)."""
    tp = _ref_of(a)
    dt, tz, ops = tp.dtypes, tp.tensors, tp.ops
    mode = dt.check_mode(mode)
    if a.ndim != 3 or b.ndim != 3:
        raise tp.errors.ShapeError("matmul_batched needs 3-D (rows, cols, batch) operands")
    (m, k, nb), (k2, n, nb2) = a.dims, b.dims
    if (k, nb) != (k2, nb2):
        raise tp.errors.ShapeError(f"batched dims disagree: {a.dims} x {b.dims}")
    device = a.device
    rdtype = dt.promote(a.dtype, b.dtype)
    if dest is None:
        dest = tz.tensor_create((m, n, nb), rdtype, device)
    else:
        ops._check_dest(dest, (m, n, nb), device, rdtype, mode)
    a = ops._prepare(a, device, rdtype, mode)
    b = ops._prepare(b, device, rdtype, mode)
    cleanups = []
    a = ops._resolve_aliasing(a, dest, cleanups, False)
    b = ops._resolve_aliasing(b, dest, cleanups, False)
    ctx = dt.CastContext(mode)
    store = ops._make_store(dest, mode, ctx)
    a_unpack, _ = dt.codec(a.dtype, a.byteorder)
    b_unpack, _ = dt.codec(b.dtype, b.byteorder)
    handle = tp.dispatch.lookup("core", device.type.name, "matmul_batched")
    ops._sync_other_streams(dest.storage.stream, a, b)
    d_buf, a_buf, b_buf = dest.storage.view(), a.storage.view(), b.storage.view()

    def run():
        handle(d_buf, dest.offset, dest.strides, store, a_buf, a.offset, a.strides, a_unpack,
               b_buf, b.offset, b.strides, b_unpack, m, n, k, nb)
        ctx.flush()

    dest.storage.stream.submit(run)
    ops._finish(dest.storage.stream, cleanups)
    return dest
