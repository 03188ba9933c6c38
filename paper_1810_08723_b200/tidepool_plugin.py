"""Drop-in adapter: the gpu table for an UNMODIFIED reference `tidepool`.

The reference hands Python closures across its function table (SURVEY.md
§8b): `store` (ops._make_store, ops.py:145-152), codec `unpack` functions
(dtypes.codec, dtypes.py:357-391), scalar `fn`s (kernels.py:50-158) and
reduction (init, step, fin) triples (ops.py:522-556).  This module recovers
the descriptors those closures encode (dtype, byte order, mode, op, compute
dtype, norm order) by introspection, so the same C-ABI kernels serve the
reference's own pipeline:

    import tidepool
    from paper_1810_08723_b200 import tidepool_plugin
    tidepool_plugin.register(tidepool)      # adds device type "gpu"
    x = tidepool.cast(t, device=tidepool.devices.by_name("gpu0"))

The decoding helpers are also used by tests/golden/make_golden.py to turn
captured reference table calls into golden vectors.
"""

from __future__ import annotations


def _cells(fn) -> dict:
    code = getattr(fn, "__code__", None)
    if code is None or fn.__closure__ is None:
        return {}
    return {n: c.cell_contents for n, c in zip(code.co_freevars, fn.__closure__)}


def decode_codec(ref_dtypes, fn):
    """(dtype name, byteorder) of a reference codec unpack/pack function."""
    for (d, order), pair in ref_dtypes._CODEC_CACHE.items():
        if fn is pair[0] or fn is pair[1]:
            return d.name, order
    raise LookupError("function is not a reference codec")


def prime_codecs(ref_dtypes) -> None:
    """Populate every (dtype, byteorder) codec so reverse lookups succeed."""
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
    cells = _cells(step)
    return float(cells.get("p", 2.0))


# ---------------------------------------------------------------------------
# registration into the reference
# ---------------------------------------------------------------------------
class _Cudart:
    """Minimal libcudart access for managed allocations and pointer kinds."""

    def __init__(self):
        import ctypes as C
        self.C = C
        self.lib = C.CDLL("libcudart.so.12", mode=C.RTLD_GLOBAL)

    def malloc_managed(self, n: int) -> int:
        C = self.C
        ptr = C.c_void_p()
        rc = self.lib.cudaMallocManaged(C.byref(ptr), C.c_size_t(max(n, 1)), C.c_uint(1))
        if rc != 0:
            raise MemoryError(f"cudaMallocManaged({n}) failed ({rc})")
        return ptr.value

    def free(self, ptr: int) -> None:
        self.lib.cudaDeviceSynchronize()
        self.lib.cudaFree(self.C.c_void_p(ptr))

    def place_on_device(self, ptr: int, n: int, device: int) -> None:
        """Preferred location = the GPU and migrate there now, so the first
        kernel touching a fresh buffer does not page-fault it over
        (cudaMemAdviseSetPreferredLocation = 3, SetAccessedBy = 5 for the
        host reads the reference does)."""
        C = self.C
        self.lib.cudaMemAdvise(C.c_void_p(ptr), C.c_size_t(n), C.c_int(3), C.c_int(device))
        self.lib.cudaMemAdvise(C.c_void_p(ptr), C.c_size_t(n), C.c_int(5), C.c_int(-1))
        self.lib.cudaMemPrefetchAsync(C.c_void_p(ptr), C.c_size_t(n), C.c_int(device), None)
        self.lib.cudaGetLastError()

    def is_device_accessible(self, ptr: int) -> bool:
        """True for device / managed / pinned memory (cudaPointerGetAttributes)."""
        C = self.C

        class Attr(C.Structure):
            _fields_ = [("type", C.c_int), ("device", C.c_int), ("devicePointer", C.c_void_p),
                        ("hostPointer", C.c_void_p)]

        a = Attr()
        rc = self.lib.cudaPointerGetAttributes(C.byref(a), C.c_void_p(ptr))
        if rc != 0:
            self.lib.cudaGetLastError()
            return False
        return a.type in (1, 2, 3)


def register(tidepool_module, count: int | None = None):
    """Attach B200 gpu devices and the ("core", "gpu") table to `tidepool`.

    Storage of gpu tensors must stay host-addressable in the reference object
    model (storage.view() memoryviews), so buffers are CUDA
    managed allocations exposed as ctypes arrays that kernels read and write
    in place.  Host (cpu-device) source buffers are staged into managed
    memory for the duration of one call.  Returns the registered devices.
    """
    import ctypes as C

    import numpy as np

    from . import _native
    from . import dtypes as D
    from . import table as tb
    from .plan import IterPlan

    tp = tidepool_module
    ref_devices, ref_dispatch, ref_dtypes = tp.devices, tp.dispatch, tp.dtypes
    prime_codecs(ref_dtypes)
    L = _native.lib()
    rt = _Cudart()
    gpu_type = ref_devices.DeviceType("gpu", supports_byteswapped=True, async_capable=False)

    class GpuDevice(ref_devices.Device):
        def __init__(self, index):
            super().__init__(gpu_type, index)

        def allocate(self, nbytes):
            if nbytes < 0:
                raise tp.errors.AllocationError("negative allocation size")
            self.alloc_count += 1
            size = max(nbytes, 1)
            # caching: every op allocates its result (and the pipeline its
            # converted intermediates); reuse managed blocks of the same size
            # released earlier (the plugin syncs after each table call, so a
            # released block has no kernel in flight)
            pool = _cache.setdefault((self.index, size), [])
            if pool:
                ptr = pool.pop()
            else:
                ptr = rt.malloc_managed(size)
                if size >= (1 << 20):
                    rt.place_on_device(ptr, size, self.index)
            arr = (C.c_ubyte * size).from_address(ptr)
            arr._tpg_free = _Free(ptr, (self.index, size))  # back to the cache with the last ref
            return arr

        @property
        def properties(self):
            props = super().properties
            props.update(tb_props(self.index))
            return props

    _cache: dict = {}
    _cache_limit = 64  # blocks kept per (device, size)

    class _Free:
        def __init__(self, ptr, key=None):
            self.ptr = ptr
            self.key = key

        def __del__(self):
            try:
                pool = _cache.get(self.key) if self.key is not None else None
                if pool is not None and len(pool) < _cache_limit:
                    pool.append(self.ptr)
                else:
                    rt.free(self.ptr)
            except Exception:
                pass

    def tb_props(index):
        from . import abi
        p = abi.DeviceProps()
        L.tpg_device_props_get(index, C.byref(p))
        return {"name": p.name.decode(), "processor-count": str(p.sm_count),
                "free-memory": str(p.free_mem)}

    class _Buf:
        """Device-visible pointer for a reference memoryview (staged when
        the buffer is ordinary host memory)."""
        __slots__ = ("ptr", "_tmp")

        def __init__(self, mv):
            self._tmp = None
            if mv is None:
                self.ptr = None
                return
            n = len(mv)
            host = int(np.frombuffer(mv, dtype=np.uint8).ctypes.data) if n else 0
            if n == 0 or rt.is_device_accessible(host):
                self.ptr = host
            else:
                self._tmp = _Free(rt.malloc_managed(n))
                C.memmove(self._tmp.ptr, host, n)
                self.ptr = self._tmp.ptr

    def _codec(fn):
        name, order = decode_codec(ref_dtypes, fn)
        return tb.Codec(D.by_name(name), order)

    def _store(store):
        name, order, mode = decode_store(ref_dtypes, store)
        return tb.Store(D.by_name(name), order, mode)

    def _plan(pl):
        return IterPlan(pl.extents, pl.strides)

    def _sync():
        _native.check(L.tpg_stream_sync(None), "sync")

    def binary(op):
        entry = tb.binary_entry(op)

        def h(plan, d_buf, store, a_buf, a_unpack, b_buf, b_unpack, fn, bases):
            ca = _codec(a_unpack)
            entry(_plan(plan), _Buf(d_buf), _store(store), _Buf(a_buf), ca, _Buf(b_buf),
                  _codec(b_unpack), tb.BinaryFn(op, D.widen_for_compute(ca.dtype)), bases)
            _sync()
        return h

    def unary(op):
        entry = tb.unary_entry(op)

        def h(plan, d_buf, store, a_buf, a_unpack, fn, bases):
            ca = _codec(a_unpack)
            fc = op != "identity" and unary_forces_complex(fn) and not ca.dtype.is_complex
            entry(_plan(plan), _Buf(d_buf), _store(store), _Buf(a_buf), ca,
                  tb.UnaryFn(op, D.widen_for_compute(ca.dtype), "standard", fc), bases)
            _sync()
        return h

    def reduce_(op):
        entry = tb.reduce_entry(op)

        def h(outer, inner, d_buf, store, a_buf, a_unpack, init, step, fin, bases):
            ca = _codec(a_unpack)
            p = norm_order(step) if op == "norm" else 2.0
            acc = tb.ReduceAcc(op, D.widen_for_compute(ca.dtype), p)
            entry(_plan(outer), _plan(inner), _Buf(d_buf), _store(store), _Buf(a_buf), ca,
                  acc, acc, acc, bases)
            _sync()
        return h

    def matmul(d_buf, d_base, d_strides, store, a_buf, a_base, a_strides, a_unpack, b_buf,
               b_base, b_strides, b_unpack, m, n, k, mul, init, step, fin):
        ca = _codec(a_unpack)
        tb.matmul_entry(_Buf(d_buf), d_base, d_strides, _store(store), _Buf(a_buf), a_base,
                        a_strides, ca, _Buf(b_buf), b_base, b_strides, _codec(b_unpack), m, n, k,
                        tb.MatmulFn(D.widen_for_compute(ca.dtype)), None, None, None)
        _sync()

    def fill(plan, buf, pack, value, base):
        tb.fill_entry(_plan(plan), _Buf(buf), _codec(pack), value, base)
        _sync()

    def arange(plan, buf, pack, cast_fn, base):
        tb.arange_entry(_plan(plan), _Buf(buf), _codec(pack), cast_fn, base)
        _sync()

    def byteswap(buf, base, plan, dtype):
        tb.byteswap_entry(_Buf(buf), base, _plan(plan), D.by_name(dtype.name))
        _sync()

    def gather(dst_buf, src_buf, pairs, size):
        tb.gather_entry(_Buf(dst_buf), _Buf(src_buf), pairs, size)
        _sync()

    def scatter(pairs, d_buf, store, s_buf, s_unpack):
        tb.scatter_entry(pairs, _Buf(d_buf), _store(store), _Buf(s_buf), _codec(s_unpack))
        _sync()

    def scatter_fill(offsets, d_buf, pack, value):
        tb.scatter_fill_entry(offsets, _Buf(d_buf), _codec(pack), value)
        _sync()

    table = {}
    for op in tb.BINARY_OPS:
        table[op] = binary(op)
    for op in tb.UNARY_OPS:
        table[op] = unary(op)
    table["copy"] = unary("identity")
    for op in tb.REDUCE_OPS:
        table[f"reduce_{op}" if op in ("minimum", "maximum") else op] = reduce_(op)
    table.update(matmul=matmul, fill=fill, arange=arange, byteswap=byteswap, gather=gather,
                 scatter=scatter, scatter_fill=scatter_fill)
    ref_dispatch.register_device_impl("core", "gpu", table)

    n = C.c_int(0)
    L.tpg_device_count(C.byref(n))
    n = n.value if count is None else min(n.value, count)
    devs = [GpuDevice(i) for i in range(n)]
    ref_devices._devices.extend(devs)
    orig_configure = ref_devices.configure

    def configure(*a, **k):
        orig_configure(*a, **k)
        ref_devices._devices.extend(devs)

    ref_devices.configure = configure

    # descriptor-based raw gather.  The reference builds
    # a Python list of (dst, src) byte-offset pairs for every clone,
    # reshape copy and byte-order-preserving transfer (tensors.py:686-699);
    # for gpu -> same-gpu moves the plugin replaces that with one
    # canonical plan and the tpg_gather_plan kernel.  tensors._raw_gather
    # is looked up at call time by its callers (ops.py:115,195,
    # tensors.contiguous_clone), so rebinding the module attribute is
    # enough.  Other device pairs keep the reference path (table "gather").
    ref_tensors = tp.tensors
    orig_raw_gather = ref_tensors._raw_gather

    def raw_gather(src, dst):
        if (dst.device.type is gpu_type and src.device is dst.device
                and src.dtype.size == dst.dtype.size and src.dims == dst.dims):
            n = 1
            for e in dst.dims:
                n *= e
            if n == 0:
                return
            if src.storage.stream is not dst.storage.stream:
                src.storage.stream.sync()
            plan = _plan(ref_tensors.canonicalize(dst, src)).to_c()
            _native.check(L.tpg_gather_plan(None, C.byref(plan), _Buf(dst.storage.view()).ptr,
                                            dst.offset, _Buf(src.storage.view()).ptr, src.offset,
                                            src.dtype.size), "gather")
            _sync()
            return
        return orig_raw_gather(src, dst)

    raw_gather.reference = orig_raw_gather
    ref_tensors._raw_gather = raw_gather
    return devs
