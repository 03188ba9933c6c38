"""Multi-GPU sharding of the hot path, one process per GPU.

Elementwise ops, casts and batched gemm shard along the slowest axis (the
last axis of a column-major tensor, or the batch axis) into contiguous
slabs, one per rank, with no data-path collective.  A full reduction runs
locally on each slab to one partial and is finished by ONE all-reduce:

    sum      partial sums in double, all-reduce SUM
    norm     partial sum |x|^p in double, all-reduce SUM, then ^(1/p)
    product  partial products, all-reduce PROD
    min/max  partial extreme over non-NaN values, all-reduce MIN/MAX, plus
             the reference's first-element rule (ops.py:533-544: the
             result is NaN iff the first element in plan order is NaN),
             carried as a flag from the rank holding element 0
    any/all  all-reduce MAX / MIN of 0/1

The reference itself is single-process with placement-only multi-device
support (devices.py:195, ops.py:110-118); sharding and the all-reduce are
new.  The communicator is pluggable: NcclComm drives libnccl through the C
ABI (tpg_nccl_*) over NVLink/NVSwitch; TorchComm uses torch.distributed
(gloo on CPU for the host-logic tests).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native

SUM, PROD, MAX, MIN = 0, 1, 2, 3


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slab of n units for `rank` (balanced, ordered)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed all-reduce on small host arrays (any backend)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce(self, values: np.ndarray, op: int) -> np.ndarray:
        import torch
        t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64).copy())
        rop = {SUM: self.dist.ReduceOp.SUM, PROD: self.dist.ReduceOp.PRODUCT,
               MAX: self.dist.ReduceOp.MAX, MIN: self.dist.ReduceOp.MIN}[op]
        self.dist.all_reduce(t, op=rop, group=self.group)
        return t.numpy()


class NcclComm:
    """libnccl over NVLink through the C ABI; rendezvous via any object
    exchange (e.g. torch.distributed.broadcast_object_list)."""

    def __init__(self, device, rank: int, world: int, share_id):
        L = _native.lib()
        uid = (C.c_char * 128)()
        if rank == 0:
            _native.check(L.tpg_nccl_get_unique_id(uid), "nccl unique id")
        raw = share_id(bytes(uid) if rank == 0 else None)
        C.memmove(uid, raw, 128)
        _native.check(L.tpg_nccl_init(device.index, world, rank, uid), "nccl init")
        self.device, self.rank, self.world = device, rank, world
        self._buf = device.allocate(64)

    def allreduce(self, values: np.ndarray, op: int) -> np.ndarray:
        L = _native.lib()
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = self.device.default_stream()
        _native.check(L.tpg_memcpy_h2d(self._buf, v.ctypes.data, v.nbytes, s.handle))
        _native.check(L.tpg_nccl_allreduce(s.handle, self._buf, v.size, 11, op), "allreduce")
        out = np.empty_like(v)
        _native.check(L.tpg_memcpy_d2h(out.ctypes.data, self._buf, v.nbytes, s.handle))
        s.sync()
        return out

    def allreduce_device(self, ptr: int, count: int, op: int, stream, dtype: int = 11) -> None:
        """In-place all-reduce of `count` elements (dtype wire code, default
        double) already on this device, enqueued on `stream` (no host round
        trip)."""
        _native.check(_native.lib().tpg_nccl_allreduce(stream.handle, ptr, count, dtype, op),
                      "allreduce")

    def info(self) -> dict:
        """The communicator as NCCL sees it (logged by bench.py)."""
        n, r = C.c_int(0), C.c_int(0)
        _native.check(_native.lib().tpg_nccl_info(C.byref(n), C.byref(r)), "nccl info")
        return {"nranks": n.value, "rank": r.value}

    def close(self):
        _native.lib().tpg_nccl_destroy()


class P2pComm:
    """The device finish over NVLink peer memory instead of NCCL
    (tpg_p2p_*): every rank's payload is stored straight into every peer's
    mailbox (CUDA IPC mappings) by ONE exchange kernel enqueued after the
    local reduction, which then combines the world's payloads in rank order
    (deterministic).  `share_all(bytes) -> [bytes per rank]` is any
    all-gather (e.g. torch.distributed.all_gather_object)."""

    def __init__(self, device, rank: int, world: int, share_all):
        L = _native.lib()
        h = (C.c_char * 64)()
        _native.check(L.tpg_p2p_init(device.index, rank, world, h), "p2p init")
        handles = share_all(bytes(h))
        if len(handles) != world or any(len(x) != 64 for x in handles):
            raise ValueError("p2p: share_all must return one 64-byte handle per rank")
        blob = b"".join(handles)
        _native.check(L.tpg_p2p_connect(blob), "p2p connect")
        self.device, self.rank, self.world = device, rank, world
        self.epoch = 0

    def allreduce_device(self, ptr: int, count: int, op: int, stream, dtype: int = 11) -> None:
        self.epoch += 1
        _native.check(_native.lib().tpg_p2p_allreduce(stream.handle, ptr, count, dtype, op,
                                                      self.epoch), "p2p allreduce")

    def check(self) -> None:
        """Raise if an exchange timed out waiting for a peer (status bit 31)."""
        f = C.c_uint32(0)
        _native.check(_native.lib().tpg_flags_get(self.device.index, C.byref(f)), "flags")
        if f.value & 0x80000000:
            _native.lib().tpg_flags_clear(self.device.index)
            raise RuntimeError("p2p all-reduce: a peer never arrived (timeout)")

    def info(self) -> dict:
        return {"nranks": self.world, "rank": self.rank, "transport": "nvlink peer memory"}

    def close(self):
        _native.lib().tpg_p2p_destroy()


# ---------------------------------------------------------------------------
# combining local partials (pure host logic, tested with gloo on CPU)
# ---------------------------------------------------------------------------
def combine_partials(op: str, partial: float, comm, *, holds_first: bool = False,
                     first_is_nan: bool = False, has_values: bool = True, p: float = 2.0):
    """Finish a full reduction from one local partial per rank."""
    if op in ("sum", "norm"):
        s = float(comm.allreduce(np.array([partial]), SUM)[0])
        return s if op == "sum" else (math.sqrt(s) if p == 2.0 else s ** (1.0 / p))
    if op == "product":
        return float(comm.allreduce(np.array([partial]), PROD)[0])
    if op in ("minimum", "maximum"):
        mx = op == "maximum"
        val = partial if (has_values and not math.isnan(partial)) else (-math.inf if mx else math.inf)
        flag = 1.0 if (holds_first and first_is_nan) else 0.0
        cnt = 1.0 if has_values else 0.0
        v = comm.allreduce(np.array([val]), MAX if mx else MIN)[0]
        f, c = comm.allreduce(np.array([flag, cnt]), SUM)
        if f > 0:
            return math.nan
        if c == 0:
            raise TypeError(f"{op} of an empty range")
        return float(v)
    if op == "any":
        return bool(comm.allreduce(np.array([1.0 if partial else 0.0]), MAX)[0])
    if op == "all":
        return bool(comm.allreduce(np.array([1.0 if partial else 0.0]), MIN)[0])
    raise ValueError(op)


# ---------------------------------------------------------------------------
# device-side sharded operations
# ---------------------------------------------------------------------------
class Sharded:
    """A tensor split into contiguous slabs along `axis`, one per rank."""

    def __init__(self, local, dims, axis, lo, rank, world):
        self.local, self.dims, self.axis, self.lo = local, tuple(dims), axis, lo
        self.rank, self.world = rank, world

    @classmethod
    def from_numpy(cls, arr, rank, world, device, axis=None):
        from . import tensors as tz
        axis = arr.ndim - 1 if axis is None else axis
        lo, hi = shard_bounds(arr.shape[axis], world, rank)
        sl = [slice(None)] * arr.ndim
        sl[axis] = slice(lo, hi)
        return cls(tz.from_numpy(np.asfortranarray(arr[tuple(sl)]), device), arr.shape, axis, lo,
                   rank, world)

    def map(self, fn, *others):
        """Apply a local op slab by slab (no communication)."""
        out = fn(self.local, *[o.local if isinstance(o, Sharded) else o for o in others])
        return Sharded(out, self.dims, self.axis, self.lo, self.rank, self.world)

    def reduce_full(self, op: str, comm, p: float = 2.0):
        """Full reduction as a host value (one 0-dim read of
        `reduce_full_tensor`; host-combined for communicators without a
        device all-reduce, e.g. gloo)."""
        if hasattr(comm, "allreduce_device") and not (op == "norm" and p != 2.0):
            return self.reduce_full_tensor(op, comm, p).item()
        return self._reduce_full_host(op, comm, p)

    def reduce_full_tensor(self, op: str, comm, p: float = 2.0):
        """Full reduction finished on the devices: the local
        kernel writes this rank's partial into a small device payload, ONE
        all-reduce combines the payloads in place over NVLink, and the
        result lands in a 0-dim device tensor of the reference's result
        dtype (ops.py:457-478).  No host round trip.

        sum      int64 / uint64 payload for integer data (exact, wraps like
                 the reference), double otherwise; SUM
        norm     p = 2: |x|^2 partial in double; SUM; sqrt on the device
        product  int64 / uint64 (exact mod 2^64) or double; PROD
        min/max  [order key, first-element-NaN flag]; ONE MAX
                 (tpg_shard_pack / tpg_shard_unpack)
        any/all  bool; MAX / MIN
        """
        from . import dtypes, ops
        from . import tensors as tz
        t = self.local
        src = t.dtype
        if src.is_complex and op in ("minimum", "maximum"):
            raise ValueError("sharded min/max of complex data is not supported")
        if op in ("minimum", "maximum") and math.prod(self.dims) == 0:
            raise TypeError(f"{op} of an empty range")  # the reference's fin(None) fails
        if op == "norm" and p != 2.0:
            raise ValueError("device-finished norm supports p = 2 (use reduce_full)")
        has = t.nelem > 0
        if (op in ("sum", "norm", "minimum", "maximum") and isinstance(comm, P2pComm)
                and src in (dtypes.FLOAT, dtypes.DOUBLE) and self.dims[self.axis] >= self.world
                and (op in ("sum", "norm") or self.axis == len(self.dims) - 1)):
            fused = self._sum_fused_p2p(comm, op)
            if fused is not None:
                return fused
        rdtype = (dtypes.BOOL if op in ("any", "all") else
                  (dtypes.real_counterpart(src) if src.is_float else dtypes.DOUBLE)
                  if op == "norm" else src)
        integer = src.is_integer or src is dtypes.BOOL
        if op in ("any", "all"):
            pdt, red = dtypes.BOOL, MAX if op == "any" else MIN
        elif op in ("sum", "product") and integer:
            pdt = dtypes.UINT64 if src is dtypes.UINT64 else dtypes.INT64
            red = SUM if op == "sum" else PROD
        elif op in ("minimum", "maximum") and integer:
            pdt, red = dtypes.INT64, MAX
        else:
            pdt, red = dtypes.DOUBLE, {"sum": SUM, "norm": SUM, "product": PROD}.get(op, MAX)
        pay = tz.tensor_create((2,), pdt, t.device)
        slot0 = tz.Tensor(pay.storage, 0, (), (), dtypes.UINT64 if src is dtypes.UINT64 and
                          op in ("minimum", "maximum", "sum", "product") else pdt)
        st = pay.storage.stream
        with _implicit():
            if not has:
                ops.fill(slot0, {"product": 1, "all": True}.get(op, 0))
            elif op == "norm":
                ops.reduce("norm", t, dest=slot0, p=2.0)
                ops.multiply(slot0, slot0, dest=slot0)  # |x|_2^2 (1 ulp)
            elif op in ("minimum", "maximum"):
                ops.reduce(op, t, dest=slot0, p=-1.0)   # extreme over non-NaN values
            else:
                ops.reduce(op, t, dest=slot0)
            if op in ("minimum", "maximum"):
                kind = 0 if not integer else (2 if src is dtypes.UINT64 else 1)
                first = self.lo == 0 and has and src.is_float
                L = _native.lib()
                t.storage.order(st)
                pay.storage.order(st)
                _native.check(L.tpg_shard_pack(
                    st.handle, int(op == "maximum"), kind, int(has), pay.storage.ptr,
                    (t.storage.ptr + t.offset) if first else None, src.code,
                    int(t.byteorder == "big")), "shard pack")
                comm.allreduce_device(pay.storage.ptr, 2, red, st, pdt.code)
                _native.check(L.tpg_shard_unpack(st.handle, int(op == "maximum"), kind,
                                                 pay.storage.ptr), "shard unpack")
            else:
                comm.allreduce_device(pay.storage.ptr, 1, red, st, pdt.code)
            if op == "norm":
                ops.square_root(slot0, dest=slot0)
            out = tz.tensor_create((), rdtype, t.device)
            ops.copy(slot0, out)
        return out

    def _sum_fused_p2p(self, comm, op="sum"):
        """ONE kernel for compute + collective (tpg_reduce_sum_p2p): the
        local single-pass sum's final block exchanges the rank's
        double-double partial with every peer's mailbox over NVLink and
        merges the world's in rank order.  Every rank takes this path for
        the same global layout (f32 / f64, no empty slab), so all ranks
        agree bit for bit.  None when the local layout is not eligible."""
        from . import abi, dtypes, ops
        from . import tensors as tz
        from .plan import build_plan
        t = self.local
        dst = tz.tensor_create((), dtypes.DOUBLE, t.device)
        st = dst.storage.stream
        t.storage.order(st)
        outer = build_plan((), [(), ()])
        inner = build_plan(t.dims, [t.strides])
        d = abi.make_operand(dst.storage.ptr, dst.offset, dtypes.DOUBLE.code, False)
        a = abi.make_operand(t.storage.ptr, t.offset, t.dtype.code, t.byteorder == "big")
        comm.epoch += 1
        L = _native.lib()
        args = (C.byref(outer.to_c()), C.byref(inner.to_c()), C.byref(d), C.byref(a), comm.epoch)
        if op in ("minimum", "maximum"):
            # global plan index of this slab's first element (slabs along the
            # slowest axis of a column-major tensor: a constant offset)
            base = self.lo * math.prod(self.dims[:-1])
            rc = L.tpg_reduce_minmax_p2p(st.handle, abi.REDUCE_CODE[op], *args, base)
        else:
            entry = L.tpg_reduce_sum_p2p if op == "sum" else L.tpg_reduce_norm2_p2p
            rc = entry(st.handle, *args)
        if rc == -4:  # not eligible: nothing launched
            comm.epoch -= 1
            return None
        _native.check(rc, "reduce_sum_p2p")
        t.storage.note_use(st)
        if t.dtype is dtypes.DOUBLE:
            return dst
        out = tz.tensor_create((), t.dtype, t.device)
        with _implicit():
            ops.copy(dst, out)
        return out

    def _reduce_full_host(self, op: str, comm, p: float):
        """Host-side finish for communicators without device buffers."""
        from . import ops
        from . import tensors as tz
        t = self.local
        has = t.nelem > 0
        if op in ("sum", "norm"):
            part = (_local_sum(t) if op == "sum" else _local_power_sum(t, p)) if has else 0.0
            return combine_partials(op, part, comm, p=p)
        if op in ("minimum", "maximum"):
            first_nan = False
            part = math.nan
            if has:
                if self.lo == 0:
                    v0 = tz.read_values(tz.apply_index(t, tuple(0 for _ in t.dims)) if t.ndim else t)
                    first_nan = isinstance(v0[0], float) and math.isnan(v0[0])
                part = _local_extreme(t, op)
            return combine_partials(op, part, comm, holds_first=self.lo == 0,
                                    first_is_nan=first_nan, has_values=has)
        if op == "product":
            return combine_partials(op, float(ops.reduce("product", t).item()) if has else 1.0,
                                    comm)
        if op in ("any", "all"):
            v = bool(ops.reduce(op, t).item()) if has else (op == "all")
            return combine_partials(op, v, comm)
        raise ValueError(op)

    def matmul_batched(self, other: "Sharded"):
        """Batched gemm sharded along the batch axis: every rank
        multiplies its own batch slab; no exchange.  Both operands must be
        split along their batch axis (2) with the same bounds."""
        from . import ops
        if self.axis != 2 or other.axis != 2 or self.lo != other.lo \
                or self.local.dims[2] != other.local.dims[2]:
            raise ValueError("sharded batched gemm needs both operands split along the batch "
                             "axis with the same bounds")
        m, _, nb = self.dims
        n = other.dims[1]
        out = ops.matmul_batched(self.local, other.local)
        return Sharded(out, (m, n, nb), 2, self.lo, self.rank, self.world)


class _implicit:
    """Internal reductions into payload slots of another dtype are exempt
    from strict mode: implicit casting on for the block."""

    def __enter__(self):
        from . import dtypes
        self.prev = dtypes.implicit_casting()
        dtypes.set_implicit_casting(True)

    def __exit__(self, *exc):
        from . import dtypes
        dtypes.set_implicit_casting(self.prev)


def _scalar_double(t):
    from . import dtypes
    from . import tensors as tz
    return tz.tensor_create((), dtypes.DOUBLE, t.device)


def _local_sum(t) -> float:
    """Slab sum, compensated on the device, stored once as a double."""
    from . import ops
    dst = _scalar_double(t)
    ops.reduce("sum", t, dest=dst)
    return float(dst.item())


def _local_power_sum(t, p) -> float:
    from . import ops
    dst = _scalar_double(t)
    ops.reduce("norm", t, dest=dst, p=p)
    return float(dst.item()) ** p


def _local_extreme(t, op) -> float:
    """Extreme over the non-NaN values of the slab, on the device (the
    reduce kernel's NaN-skipping variant, selected by p < 0)."""
    from . import ops
    dst = _scalar_double(t)
    ops.reduce(op, t, dest=dst, p=-1.0)
    return float(dst.item())
