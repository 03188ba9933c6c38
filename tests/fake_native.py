"""CPU test double of libtidepool_gpu.so (TEST INFRASTRUCTURE ONLY).

Implements the subset of the C ABI (include/tidepool_gpu.h) the drop-in
plugin calls, with "device" memory in host buffers and the kernels executed
by the C oracle (oracle/tp_oracle.c, same plan / operand descriptors).  It
lets the CPU suite drive tidepool_plugin.register() end to end - closure
decoding, status / cast-loss routing into the unmodified reference, lazy
casts, staging and descriptor transfers - without a GPU.  The product never
loads it: register() only takes it through its `lib=` test hook.
"""

from __future__ import annotations

import ctypes as C

from paper_1810_08723_b200 import abi

_DT_SIZE = {0: 1, 1: 1, 2: 1, 3: 2, 4: 2, 5: 4, 6: 4, 7: 8, 8: 8, 9: 2, 10: 4, 11: 8, 12: 4,
            13: 8, 14: 16}
_RAW = {1: 2, 2: 4, 4: 6, 8: 8, 16: 14}   # element size -> a dtype whose identity copy is byte-exact


def _obj(ref):
    return ref._obj if hasattr(ref, "_obj") else ref


class FakeNative:
    """Duck-typed stand-in for the ctypes library object."""

    def __init__(self, oracle_lib, ndev=1):
        self.o = oracle_lib
        self.ndev = ndev
        self.mem = {}          # ptr -> ctypes buffer (keeps host memory alive)
        self.flags = [0] * ndev
        self.inject = 0        # extra bits the next kernel reports (routing tests)
        self.calls = []        # (name, ...) of every kernel launched
        self.managed = set()

    # -- runtime --------------------------------------------------------------
    def tpg_last_error(self):
        return b"fake error"

    def tpg_device_count(self, out):
        _obj(out).value = self.ndev
        return 0

    def tpg_device_props_get(self, dev, props):
        p = _obj(props)
        p.sm_count, p.total_mem, p.free_mem = 148, 1 << 30, 1 << 30
        p.name = b"fake B200"
        return 0

    def _alloc(self, n):
        buf = C.create_string_buffer(max(int(n), 1))
        ptr = C.addressof(buf)
        self.mem[ptr] = buf
        return ptr

    def tpg_malloc_managed(self, dev, n, out):
        ptr = self._alloc(n)
        self.managed.add(ptr)
        _obj(out).value = ptr
        return 0

    def tpg_free_managed(self, ptr):
        self.mem.pop(_int(ptr), None)
        return 0

    def tpg_malloc_on(self, stream, n, out):
        _obj(out).value = self._alloc(n)
        return 0

    def tpg_free(self, dev, ptr, stream):
        self.mem.pop(_int(ptr), None)
        return 0

    def tpg_malloc(self, dev, n, out):
        _obj(out).value = self._alloc(n)
        return 0

    def tpg_host_alloc(self, n, out):
        _obj(out).value = self._alloc(n)
        return 0

    def tpg_host_free(self, ptr):
        self.mem.pop(_int(ptr), None)
        return 0

    def tpg_init(self):
        return 0

    def tpg_version(self):
        return b"fake"

    def tpg_mem_stats(self, dev, a, b, c):
        _obj(a).value = sum(len(v) for v in self.mem.values())
        _obj(b).value = 0
        _obj(c).value = len(self.mem)
        return 0

    def tpg_stream_wait(self, a, b):
        return 0

    def tpg_stream_destroy(self, s):
        return 0

    def tpg_event_create(self, out):
        _obj(out).value = 0x3001
        return 0

    def tpg_event_destroy(self, ev):
        return 0

    def tpg_event_elapsed(self, a, b, out):
        _obj(out).value = 0.0
        return 0

    def tpg_memcpy_d2d(self, dst, src, n, s):
        C.memmove(_int(dst), _int(src), n)
        return 0

    def tpg_memset(self, dst, v, n, s):
        C.memset(_int(dst), v, n)
        return 0

    def tpg_memcpy2d(self, dst, dpitch, src, spitch, width, height, s):
        for r in range(height):
            C.memmove(_int(dst) + r * dpitch, _int(src) + r * spitch, width)
        return 0

    def tpg_flags_get(self, dev, out):
        _obj(out).value = self.flags[dev]
        return 0

    def tpg_flags_clear(self, dev):
        self.flags[dev] = 0
        return 0

    def tpg_default_stream(self, dev, out):
        _obj(out).value = 0x1000 + dev
        return 0

    def tpg_stream_create(self, dev, out):
        _obj(out).value = 0x2000 + dev
        return 0

    def tpg_stream_sync(self, s):
        return 0

    def tpg_event_create_untimed(self, out):
        _obj(out).value = 0x3000
        return 0

    def tpg_event_record(self, ev, s):
        return 0

    def tpg_event_query(self, ev):
        return 0

    def tpg_event_sync(self, ev):
        return 0

    def tpg_memcpy_h2d(self, dst, src, n, s):
        C.memmove(_int(dst), src if isinstance(src, (bytes, bytearray)) else _int(src), n)
        return 0

    tpg_memcpy_d2h = tpg_memcpy_h2d

    def _dev_of(self, stream):
        s = _int(stream)
        return (s & 0xff) if s else 0

    def tpg_flags_take(self, stream, out):
        d = self._dev_of(stream)
        _obj(out).value = self.flags[d]
        self.flags[d] = 0
        return 0

    def _flag(self, st):
        self.flags[0] |= st.value | self.inject
        self.inject = 0

    # NCCL stand-in: the all-reduce runs over torch.distributed (gloo) on
    # the host bytes when a process group is up, else it is the identity of
    # a single rank
    def tpg_nccl_get_unique_id(self, out):
        return 0

    def tpg_nccl_init(self, dev, nranks, rank, uid):
        import torch.distributed as dist
        if nranks == 1 or (dist.is_initialized() and dist.get_world_size() == nranks):
            self.nccl = (nranks, rank)
            return 0
        return -4

    def tpg_nccl_info(self, n, r):
        _obj(n).value, _obj(r).value = getattr(self, "nccl", (1, 0))
        return 0

    def tpg_nccl_allreduce(self, s, buf, count, dtype, op):
        import numpy as np
        import torch
        import torch.distributed as dist
        if not dist.is_initialized() or dist.get_world_size() == 1:
            return 0
        npd = {0: np.uint8, 1: np.int8, 2: np.uint8, 5: np.int32, 6: np.uint32, 7: np.int64,
               8: np.uint64, 10: np.float32, 11: np.float64}[dtype]
        raw = (C.c_ubyte * (count * np.dtype(npd).itemsize)).from_address(_int(buf))
        arr = np.frombuffer(raw, dtype=npd)
        wide = torch.from_numpy(arr.astype(np.int64 if npd == np.uint64 else npd).copy())
        if npd == np.uint64 and op in (2, 3):   # order of unsigned keys: bias into int64
            wide = torch.from_numpy((arr ^ np.uint64(1 << 63)).view(np.int64).copy())
        rop = [dist.ReduceOp.SUM, dist.ReduceOp.PRODUCT, dist.ReduceOp.MAX, dist.ReduceOp.MIN][op]
        dist.all_reduce(wide, op=rop)
        res = wide.numpy()
        if npd == np.uint64:
            res = (res.view(np.uint64) ^ np.uint64(1 << 63)) if op in (2, 3) else res.view(np.uint64)
        arr[:] = res.astype(npd)
        return 0

    def tpg_nccl_destroy(self):
        return 0

    def tpg_shard_pack(self, s, is_max, kind, has, payload, first, fdt, fbig):
        import numpy as np
        fnan = 0
        if first:
            npd = {11: "f8", 10: "f4", 9: "f2"}.get(fdt)
            if npd is not None:
                raw = (C.c_ubyte * 8).from_address(_int(first))
                v = np.frombuffer(bytes(raw)[:np.dtype(npd).itemsize],
                                  dtype=(">" if fbig else "<") + npd)[0]
                fnan = 1 if v != v else 0
        if kind == 0:
            p = np.frombuffer((C.c_ubyte * 16).from_address(_int(payload)), dtype=np.float64)
            v = p[0]
            p[0] = (v if is_max else -v) if (has and v == v) else -np.inf
            p[1] = fnan
        else:
            p = np.frombuffer((C.c_ubyte * 16).from_address(_int(payload)), dtype=np.int64)
            k = p[0]
            if kind == 2:  # unsigned source: flip the sign bit (order-preserving)
                k = np.array([p.view(np.uint64)[0] ^ np.uint64(1 << 63)],
                             dtype=np.uint64).view(np.int64)[0]
            p[0] = (k if is_max else ~k) if has else np.iinfo(np.int64).min
            p[1] = 0
        return 0

    def tpg_shard_unpack(self, s, is_max, kind, payload):
        import numpy as np
        if kind == 0:
            p = np.frombuffer((C.c_ubyte * 16).from_address(_int(payload)), dtype=np.float64)
            p[0] = np.nan if p[1] != 0 else (p[0] if is_max else -p[0])
        else:
            p = np.frombuffer((C.c_ubyte * 16).from_address(_int(payload)), dtype=np.int64)
            k = p[0] if is_max else ~p[0]
            if kind == 2:
                k = np.array([np.array([k], dtype=np.int64).view(np.uint64)[0]
                              ^ np.uint64(1 << 63)], dtype=np.uint64).view(np.int64)[0]
            p[0] = k
        return 0

    # -- kernels (oracle) ---------------------------------------------------------
    def tpg_binary(self, s, op, plan, d, a, b, comp, mode):
        self.calls.append(("binary", op, _obj(a).dtype, _obj(b).dtype))
        st = C.c_uint32(0)
        rc = self.o.tpo_binary(op, plan, d, a, b, comp, mode, C.byref(st))
        self._flag(st)
        return rc

    def tpg_binary_check(self, s, op, plan, d, a, b, comp, mode):
        st = C.c_uint32(0)
        with _Scratch(self, d) as dd:
            rc = self.o.tpo_binary(op, plan, C.byref(dd), a, b, comp, mode, C.byref(st))
        self._flag(st)
        return rc

    def tpg_unary(self, s, op, plan, d, a, comp, mode, fc):
        self.calls.append(("unary", op, _obj(a).dtype, _obj(d).dtype))
        st = C.c_uint32(0)
        rc = self.o.tpo_unary(op, plan, d, a, comp, mode, fc, C.byref(st))
        self._flag(st)
        return rc

    def tpg_unary_check(self, s, op, plan, d, a, comp, mode, fc):
        st = C.c_uint32(0)
        with _Scratch(self, d) as dd:
            rc = self.o.tpo_unary(op, plan, C.byref(dd), a, comp, mode, fc, C.byref(st))
        self._flag(st)
        return rc

    def tpg_reduce(self, s, op, p, po, pi, d, a, comp, mode):
        self.calls.append(("reduce", op))
        st = C.c_uint32(0)
        rc = self.o.tpo_reduce(op, p, po, pi, d, a, comp, mode, C.byref(st))
        self._flag(st)
        return rc

    def tpg_matmul(self, s, d, ds, a, as_, b, bs, m, n, k, comp, mode):
        self.calls.append(("matmul",))
        st = C.c_uint32(0)
        rc = self.o.tpo_matmul(d, ds, a, as_, b, bs, m, n, k, comp, mode, C.byref(st))
        self._flag(st)
        return rc

    def tpg_matmul_batched(self, s, nb, d, ds, a, as_, b, bs, m, n, k, comp, mode):
        self.calls.append(("matmul_batched",))
        dd, aa, bb = _obj(d), _obj(a), _obj(b)
        st = C.c_uint32(0)
        for q in range(nb):
            do = abi.make_operand(dd.base, dd.offset + q * ds[2], dd.dtype, dd.big_endian)
            ao = abi.make_operand(aa.base, aa.offset + q * as_[2], aa.dtype, aa.big_endian)
            bo = abi.make_operand(bb.base, bb.offset + q * bs[2], bb.dtype, bb.big_endian)
            d2, a2, b2 = ((C.c_int64 * 2)(x[0], x[1]) for x in (ds, as_, bs))
            rc = self.o.tpo_matmul(C.byref(do), d2, C.byref(ao), a2, C.byref(bo), b2, m, n, k,
                                   comp, mode, C.byref(st))
            if rc:
                return rc
        self._flag(st)
        return 0

    def _chain(self, plan, d, a, nsteps, steps, mode, dry):
        """x <- op_i(x, s_i) step by step through tpo_binary, rounding to
        each step's dtype in a scratch copy laid out like the destination."""
        dd, aa = _obj(d), _obj(a)
        p = _obj(plan)
        st = C.c_uint32(0)
        ext = [p.extent[k] for k in range(p.ndim)]
        n = 1
        for e in ext:
            n *= e
        cur = abi.make_operand(aa.base, aa.offset, aa.dtype, aa.big_endian)
        cur_strides = [p.stride[1][k] for k in range(p.ndim)]
        keep = []
        for i in range(nsteps):
            sp = steps[i]
            last = i == nsteps - 1
            if last and not dry:
                out = abi.make_operand(dd.base, dd.offset, dd.dtype, dd.big_endian)
                out_strides = [p.stride[0][k] for k in range(p.ndim)]
            else:
                size = _DT_SIZE[sp.dtype]
                buf = C.create_string_buffer(max(n * size, 1))
                keep.append(buf)
                out = abi.make_operand(C.addressof(buf), 0, sp.dtype, False)
                out_strides, acc = [], size
                for e in ext:
                    out_strides.append(acc)
                    acc *= e
            imm = abi.make_operand(None, 0, sp.scalar_dtype, False, bytes(sp.scalar))
            pl = abi.make_plan(ext, [out_strides, cur_strides, [0] * p.ndim])
            x, y = (imm, cur) if sp.scalar_first else (cur, imm)
            if sp.scalar_first:
                pl = abi.make_plan(ext, [out_strides, [0] * p.ndim, cur_strides])
            rc = self.o.tpo_binary(sp.op, C.byref(pl), C.byref(out), C.byref(x), C.byref(y),
                                   sp.compute, mode, C.byref(st))
            if rc:
                return rc
            cur, cur_strides = out, out_strides
        self._flag(st)
        return 0

    def tpg_chain(self, s, plan, d, a, nsteps, steps, mode):
        self.calls.append(("chain",))
        return self._chain(plan, d, a, nsteps, steps, mode, False)

    def tpg_chain_check(self, s, plan, d, a, nsteps, steps, mode):
        return self._chain(plan, d, a, nsteps, steps, mode, True)

    def tpg_fill(self, s, plan, d, value, size):
        self.calls.append(("fill",))
        return self.o.tpo_fill(plan, d, value, size)

    def tpg_arange(self, s, plan, d):
        self.calls.append(("arange",))
        return self.o.tpo_arange(plan, d)

    def tpg_byteswap(self, s, plan, d):
        self.calls.append(("byteswap",))
        return self.o.tpo_byteswap(plan, d)

    def tpg_gather_plan(self, s, plan, dst, doff, src, soff, size):
        self.calls.append(("gather_plan",))
        dt = _RAW[size]
        d = abi.make_operand(_int(dst), doff, dt, False)
        a = abi.make_operand(_int(src), soff, dt, False)
        st = C.c_uint32(0)
        return self.o.tpo_unary(10, plan, C.byref(d), C.byref(a), dt, 0, 0, C.byref(st))

    def tpg_gather(self, s, dst, src, pairs, n, size):
        self.calls.append(("gather",))
        for i in range(n):
            C.memmove(_int(dst) + pairs[2 * i], _int(src) + pairs[2 * i + 1], size)
        return 0

    def tpg_scatter(self, s, pairs, n, d, sop, mode):
        self.calls.append(("scatter",))
        dd, ss = _obj(d), _obj(sop)
        st = C.c_uint32(0)
        for i in range(n):
            p = abi.make_plan([], [[], []])
            do = abi.make_operand(dd.base, pairs[2 * i], dd.dtype, dd.big_endian)
            so = abi.make_operand(ss.base, pairs[2 * i + 1], ss.dtype, ss.big_endian)
            self.o.tpo_unary(10, C.byref(p), C.byref(do), C.byref(so), ss.dtype, mode, 0,
                             C.byref(st))
        self._flag(st)
        return 0

    def tpg_scatter_fill(self, s, offsets, n, dbase, value, size):
        self.calls.append(("scatter_fill",))
        for i in range(n):
            C.memmove(_int(dbase) + offsets[i], value, size)
        return 0


class _Scratch:
    """Dry-run destination: the kernel writes into a throwaway copy."""

    def __init__(self, fake, dref):
        self.fake, self.d = fake, _obj(dref)

    def __enter__(self):
        base = self.d.base
        for ptr, buf in self.fake.mem.items():
            if ptr <= base < ptr + len(buf):
                self.copy = C.create_string_buffer(buf.raw, len(buf))
                o = abi.make_operand(C.addressof(self.copy) + (base - ptr), self.d.offset,
                                     self.d.dtype, self.d.big_endian)
                return o
        raise AssertionError("dry-run destination outside fake device memory")

    def __exit__(self, *exc):
        return False


def _int(p):
    if isinstance(p, int):
        return p
    if p is None:
        return 0
    if isinstance(p, C.Array):
        return C.addressof(p)
    v = getattr(p, "value", p)
    return int(v or 0)
