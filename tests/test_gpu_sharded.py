"""Sharded full reductions on the device: local kernel partials + NCCL
all-reduce (world 1 on the test box; the multi-rank host logic is covered
with gloo in test_sharded_gloo.py)."""

import math

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200.sharded import NcclComm, Sharded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = NcclComm(tp.gpu(0), 0, 1, lambda uid: uid)
    yield c
    c.close()


def test_sharded_full_reductions_match_single_device(comm):
    rng = np.random.default_rng(1)
    x = rng.random((512, 256))
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    T = tp.from_numpy(np.asfortranarray(x))
    assert S.reduce_full("sum", comm) == pytest.approx(tp.reduce("sum", T).item(), rel=1e-13)
    assert S.reduce_full("norm", comm) == pytest.approx(tp.reduce("norm", T).item(), rel=1e-13)
    assert S.reduce_full("maximum", comm) == tp.reduce("maximum", T).item()
    assert S.reduce_full("minimum", comm) == tp.reduce("minimum", T).item()


def test_nan_rules(comm):
    x = np.array([1.0, np.nan, 5.0, -2.0])
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    assert S.reduce_full("maximum", comm) == 5.0  # NaN not first: skipped
    y = np.array([np.nan, 1.0, 5.0])
    S2 = Sharded.from_numpy(y, 0, 1, tp.gpu(0))
    assert math.isnan(S2.reduce_full("maximum", comm))  # first element NaN


def test_sharded_map_is_local(comm):
    rng = np.random.default_rng(2)
    x = rng.random(1 << 16).astype(np.float32)
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    out = S.map(lambda t, s: tp.multiply(t, s), tp.Scalar(1.5, tp.float))
    assert np.array_equal(tp.to_numpy(out.local), (x.astype(np.float64) * 1.5).astype(np.float32))


CASES = [
    ("float64", lambda r: r.standard_normal(1000)),
    ("float32", lambda r: r.standard_normal(777).astype(np.float32)),
    ("int64", lambda r: r.integers(-(1 << 62), 1 << 62, 513)),
    ("uint64", lambda r: r.integers(0, 1 << 63, 300).astype(np.uint64) * np.uint64(2) + np.uint64(1)),
    ("int8", lambda r: r.integers(-128, 128, 999).astype(np.int8)),
]


@pytest.mark.parametrize("name,make", CASES)
def test_device_finish_matches_single_device(comm, name, make):
    """Every full reduction finished on the device (payload + one NCCL
    all-reduce, tpg_shard_pack / unpack) equals the single-device result,
    including integers above 2^53 (exact int64 / uint64 payloads)."""
    x = make(np.random.default_rng(len(name)))
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    T = tp.from_numpy(x)
    for op in ("sum", "product", "minimum", "maximum", "any", "all", "norm"):
        got = S.reduce_full_tensor(op, comm)
        want = tp.reduce(op, T)
        assert got.dtype is want.dtype, (name, op)
        g, w = got.item(), want.item()
        if op in ("sum", "norm", "product") and isinstance(w, float):
            assert g == pytest.approx(w, rel=1e-12, abs=0) or (math.isnan(g) and math.isnan(w)) \
                or (math.isinf(g) and g == w), (name, op, g, w)
        else:
            assert g == w, (name, op, g, w)


def test_device_finish_nan_first_and_all_nan(comm):
    for data, want in (([np.nan, 1.0, 5.0], "nan"), ([1.0, np.nan, 5.0], 5.0),
                       ([np.nan, np.nan], "nan")):
        S = Sharded.from_numpy(np.array(data), 0, 1, tp.gpu(0))
        g = S.reduce_full_tensor("maximum", comm).item()
        assert (math.isnan(g) if want == "nan" else g == want), (data, g)


def test_sharded_batched_gemm_matches_full(comm):
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (64, 48, 6)).astype(np.float16)
    b = rng.uniform(-1, 1, (48, 40, 6)).astype(np.float16)
    A = Sharded.from_numpy(a, 0, 1, tp.gpu(0), axis=2)
    B = Sharded.from_numpy(b, 0, 1, tp.gpu(0), axis=2)
    C = A.matmul_batched(B)
    assert C.dims == (64, 40, 6) and C.axis == 2
    full = tp.to_numpy(tp.matmul_batched(tp.from_numpy(np.asfortranarray(a)),
                                         tp.from_numpy(np.asfortranarray(b))))
    assert np.array_equal(tp.to_numpy(C.local), full)


def test_nccl_sees_the_ranks(comm):
    assert comm.info() == {"nranks": 1, "rank": 0}
