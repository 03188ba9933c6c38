"""The sharded full-reduction finish over peer memory (tpg_p2p_*, no NCCL):
world 1 in-process, and world 2 as two processes sharing the test box's GPU
(CUDA IPC mappings of each other's mailbox; the exchange kernels of the two
contexts time-slice), against the single-device reductions."""

import math
import os
import socket

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200.sharded import P2pComm, Sharded

pytestmark = pytest.mark.gpu

OPS = ("sum", "product", "minimum", "maximum", "any", "all", "norm")


def _cases():
    r = np.random.default_rng(11)
    f = r.standard_normal(1001)
    return [("f64", f), ("f64_nan_first", np.concatenate([[np.nan], f[1:]])),
            ("f32", r.standard_normal(777).astype(np.float32)),
            ("i64_big", r.integers(-(1 << 62), 1 << 62, 513)),
            ("u64", r.integers(0, 1 << 63, 301).astype(np.uint64) * np.uint64(2) + np.uint64(1)),
            ("i8", r.integers(-128, 128, 999).astype(np.int8))]


def _same(g, w):
    if isinstance(w, float) and math.isnan(w):
        return math.isnan(g)
    if isinstance(w, float):
        return g == pytest.approx(w, rel=1e-12, abs=0) or g == w
    return g == w


def test_p2p_world1_matches_single_device():
    comm = P2pComm(tp.gpu(0), 0, 1, lambda h: [h])
    try:
        for name, x in _cases():
            S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
            T = tp.from_numpy(x)
            for op in OPS:
                if x.dtype.kind == "u" and op == "norm":
                    continue
                g, w = S.reduce_full_tensor(op, comm).item(), tp.reduce(op, T).item()
                assert _same(g, w), (name, op, g, w)
        # the f32 / f64 full sums took the fused single-kernel path
        x = np.random.default_rng(3).standard_normal(100_000)
        fused = Sharded.from_numpy(x, 0, 1, tp.gpu(0))._sum_fused_p2p(comm)
        assert fused is not None
        assert fused.item() == pytest.approx(tp.reduce("sum", tp.from_numpy(x)).item(), rel=1e-12)
        fused = Sharded.from_numpy(x, 0, 1, tp.gpu(0))._sum_fused_p2p(comm, "norm")
        assert fused.item() == pytest.approx(tp.reduce("norm", tp.from_numpy(x)).item(), rel=1e-12)
        for op in ("minimum", "maximum"):
            f = Sharded.from_numpy(x, 0, 1, tp.gpu(0))._sum_fused_p2p(comm, op)
            assert f.item() == tp.reduce(op, tp.from_numpy(x)).item()
        comm.check()
        assert comm.info()["nranks"] == 1
    finally:
        comm.close()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1810_08723_b200 as tpw
        from paper_1810_08723_b200.sharded import P2pComm as P, Sharded as Sh

        def share_all(h):
            out = [None] * world
            dist.all_gather_object(out, h)
            return out
        comm = P(tpw.gpu(0), rank, world, share_all)
        res = {}
        for name, x in _cases():
            S = Sh.from_numpy(x, rank, world, tpw.gpu(0))
            for op in OPS:
                if x.dtype.kind == "u" and op == "norm":
                    continue
                res[(name, op)] = S.reduce_full_tensor(op, comm).item()
        x = np.random.default_rng(3).standard_normal(100_001)
        f = Sh.from_numpy(x, rank, world, tpw.gpu(0))._sum_fused_p2p(comm)
        res["fused_sum"] = None if f is None else f.item()
        # min / max: the tie / signed-zero / NaN-first rules across ranks
        for tag, y in (("ties", np.array([0.0, 1.0, -0.0, 5.0, 5.0, -0.0, 0.0, 5.0])),
                       ("nan_first", np.array([np.nan, 1.0, 2.0, np.nan, 3.0, 0.5])),
                       ("nan_rank1", np.array([1.0, 2.0, 0.5, np.nan, 3.0, 0.5])),
                       ("rand", x)):
            for op in ("minimum", "maximum"):
                f = Sh.from_numpy(y, rank, world, tpw.gpu(0))._sum_fused_p2p(comm, op)
                res[("mm", tag, op)] = None if f is None else f.item()
        comm.check()
        comm.close()
        q.put((rank, res))
    except Exception as exc:  # surfaced by the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_p2p_world2_two_processes_one_gpu():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        assert isinstance(res[r], dict), res[r]
    xs = np.random.default_rng(3).standard_normal(100_001)
    want = tp.reduce("sum", tp.from_numpy(xs)).item()
    assert res[0]["fused_sum"] == res[1]["fused_sum"]          # ranks agree bit for bit
    assert res[0]["fused_sum"] == pytest.approx(want, rel=1e-12)
    for tag, y in (("ties", np.array([0.0, 1.0, -0.0, 5.0, 5.0, -0.0, 0.0, 5.0])),
                   ("nan_first", np.array([np.nan, 1.0, 2.0, np.nan, 3.0, 0.5])),
                   ("nan_rank1", np.array([1.0, 2.0, 0.5, np.nan, 3.0, 0.5])),
                   ("rand", xs)):
        for op in ("minimum", "maximum"):
            w = tp.reduce(op, tp.from_numpy(y)).item()
            for r in (0, 1):
                g = res[r][("mm", tag, op)]
                assert g is not None
                assert (math.isnan(g) and math.isnan(w)) or (g == w and math.copysign(1, g) ==
                                                             math.copysign(1, w)), (tag, op, r, g, w)
    for name, x in _cases():
        T = tp.from_numpy(x)
        for op in OPS:
            if (name, op) not in res[0]:
                continue
            w = tp.reduce(op, T).item()
            for r in (0, 1):
                assert _same(res[r][(name, op)], w), (name, op, r, res[r][(name, op)], w)
