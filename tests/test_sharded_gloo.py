"""Multi-process (world_size 2, gloo on CPU) checks of the sharding host
logic: slab bounds and the all-reduce finish of full reductions, including
the reference's first-element NaN rule for min/max (ops.py:533-544).  The
per-slab partials here come from numpy (the device kernels need a GPU);
the GPU path is covered by tests/test_gpu_sharded.py."""

import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1810_08723_b200.sharded import combine_partials, shard_bounds


def test_shard_bounds_partition():
    for n in (0, 1, 7, 8, 1023, 1 << 20):
        for world in (1, 2, 3, 8):
            got = [shard_bounds(n, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[i][1] == got[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1


def _ref_full(op, x):
    """Reference semantics of a full reduction over x in plan order."""
    if op == "sum":
        return math.fsum(x)
    if op == "norm":
        return math.sqrt(math.fsum(v * v for v in x))
    if op in ("minimum", "maximum"):
        acc = None
        for v in x:
            if acc is None or (v < acc if op == "minimum" else v > acc):
                acc = v
        return acc
    if op == "any":
        return any(v != 0 for v in x)
    if op == "all":
        return all(v != 0 for v in x)


def _worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1810_08723_b200.sharded import TorchComm
    comm = TorchComm()
    out = []
    for op, x in cases:
        lo, hi = shard_bounds(len(x), world, rank)
        s = np.asarray(x[lo:hi], dtype=np.float64)
        has = s.size > 0
        if op == "sum":
            part = math.fsum(s)
        elif op == "norm":
            part = math.fsum(s * s)
        elif op in ("minimum", "maximum"):
            v = s[~np.isnan(s)]
            part = (v.max() if op == "maximum" else v.min()) if v.size else math.nan
        elif op == "any":
            part = bool(np.any(s != 0))
        else:
            part = bool(np.all(s != 0)) if has else True
        first_nan = lo == 0 and has and math.isnan(s[0])
        out.append(combine_partials(op, part, comm, holds_first=lo == 0, first_is_nan=first_nan,
                                    has_values=has))
    q.put((rank, out))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_full_reduction_finish_world2():
    rng = np.random.default_rng(0)
    x = list(rng.standard_normal(1001))
    nan_first = [math.nan] + x[1:]
    nan_mid = x[:600] + [math.nan] + x[601:]
    cases = [("sum", x), ("norm", x), ("maximum", x), ("minimum", x), ("maximum", nan_first),
             ("minimum", nan_mid), ("maximum", [0.0, -0.0]), ("any", [0.0] * 10 + [1.0]),
             ("all", [1.0] * 9 + [0.0]), ("sum", [1.0])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == res[1] or all(
        (isinstance(a, float) and math.isnan(a) and math.isnan(b)) or a == b
        for a, b in zip(res[0], res[1]))
    for (op, xs), got in zip(cases, res[0]):
        want = _ref_full(op, xs)
        if isinstance(want, float) and math.isnan(want):
            assert math.isnan(got), op
        elif op in ("sum", "norm"):
            assert got == pytest.approx(want, rel=1e-12), op
        else:
            assert got == want, (op, got, want)


# ---------------------------------------------------------------------------
# the DEVICE path at world size 2: every rank drives the sharded code over
# the CPU test double of the C ABI (tests/fake_native.py; kernels by the C
# oracle, the NCCL all-reduce of the payload over gloo), so the payload
# encoding (tpg_shard_pack / unpack semantics), the slab partitioning and
# the sharded batched gemm run multi-process here
# ---------------------------------------------------------------------------
def _device_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    sys.path[:0] = [str(here), str(here.parent)]
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from fake_native import FakeNative
    from oracle import oracle
    from paper_1810_08723_b200 import _native
    _native._lib = FakeNative(oracle.lib())
    import paper_1810_08723_b200 as tp
    from paper_1810_08723_b200.sharded import NcclComm, Sharded
    def share(uid):
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    comm = NcclComm(tp.gpu(0), rank, world, share)
    assert comm.info() == {"nranks": world, "rank": rank}
    out = {}
    for name, x in _device_cases():
        S = Sharded.from_numpy(x, rank, world, tp.gpu(0))
        for op in ("sum", "product", "minimum", "maximum", "any", "all", "norm"):
            if x.dtype.kind == "u" and op == "norm":
                continue
            out[(name, op)] = S.reduce_full_tensor(op, comm).item()
    a = np.random.default_rng(5).uniform(-1, 1, (16, 12, 5)).astype(np.float16)
    b = np.random.default_rng(6).uniform(-1, 1, (12, 8, 5)).astype(np.float16)
    C = Sharded.from_numpy(a, rank, world, tp.gpu(0), axis=2).matmul_batched(
        Sharded.from_numpy(b, rank, world, tp.gpu(0), axis=2))
    out["gemm"] = (C.lo, tp.to_numpy(C.local))
    q.put((rank, out))
    dist.destroy_process_group()


def _device_cases():
    r = np.random.default_rng(7)
    f = r.standard_normal(1001)
    return [("f64", f), ("f64_nan_first", np.concatenate([[np.nan], f[1:]])),
            ("f64_nan_rank1", np.concatenate([f[:700], [np.nan], f[701:]])),
            ("f32", r.standard_normal(777).astype(np.float32)),
            ("i64_big", r.integers(-(1 << 62), 1 << 62, 513)),
            ("u64", r.integers(0, 1 << 63, 301).astype(np.uint64) * np.uint64(2) + np.uint64(1)),
            ("i8_wrap", r.integers(-128, 128, 999).astype(np.int8)),
            ("one_element", np.array([3.5]))]


def test_device_finish_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    # expected: the single-device reductions of the whole tensor, same fake backend
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from fake_native import FakeNative
    from oracle import oracle
    from paper_1810_08723_b200 import _native
    saved = _native._lib
    _native._lib = FakeNative(oracle.lib())
    try:
        import paper_1810_08723_b200 as tp
        for name, x in _device_cases():
            T = tp.from_numpy(x)
            for op in ("sum", "product", "minimum", "maximum", "any", "all", "norm"):
                if (name, op) not in res[0]:
                    continue
                want = tp.reduce(op, T).item()
                for rank in (0, 1):
                    got = res[rank][(name, op)]
                    if isinstance(want, float) and math.isnan(want):
                        assert math.isnan(got), (name, op, rank)
                    elif op in ("sum", "norm", "product") and isinstance(want, float):
                        assert got == pytest.approx(want, rel=1e-12, abs=0) or got == want, \
                            (name, op, got, want)
                    else:
                        assert got == want, (name, op, rank, got, want)
        a = np.random.default_rng(5).uniform(-1, 1, (16, 12, 5)).astype(np.float16)
        b = np.random.default_rng(6).uniform(-1, 1, (12, 8, 5)).astype(np.float16)
        full = tp.to_numpy(tp.matmul_batched(tp.from_numpy(np.asfortranarray(a)),
                                             tp.from_numpy(np.asfortranarray(b))))
        slabs = sorted(res[r]["gemm"] for r in (0, 1))
        assert slabs[0][0] == 0 and slabs[1][0] == 3   # batch slabs [0,3) and [3,5)
        assert np.array_equal(np.concatenate([s[1] for s in slabs], axis=2), full)
    finally:
        _native._lib = saved
