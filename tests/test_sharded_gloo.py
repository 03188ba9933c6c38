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
