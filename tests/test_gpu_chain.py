"""Fused elementwise chains (extension) are
bit-identical to running the same binary ops one after another (each of
which is oracle-checked in test_gpu_pipeline / test_gpu_golden), including
the sticky status flags; SURVEY cfg5's multiply-then-add is checked
against a numpy restatement of the reference's double-compute, round-once
semantics."""

import random

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import dtypes as D
from test_gpu_pipeline import rand_tensor

pytestmark = pytest.mark.gpu


def _bits(t):
    a = tp.to_numpy(t)
    return a.view(np.uint8).tobytes() if a.dtype != np.bool_ else a.tobytes()


def test_cfg5_chain_matches_sequential_and_numpy():
    n = (1 << 20) + 5
    y = np.random.default_rng(8).uniform(-1e3, 1e3, n).astype(np.float32)
    Y = tp.from_numpy(y)
    k15, km2 = tp.Scalar(1.5, tp.float), tp.Scalar(-2.0, tp.float)
    Z = tp.chain(Y, [("multiply", k15), ("add", km2)])
    seq = tp.add(tp.multiply(Y, k15), km2)
    assert Z.dtype is tp.float
    assert _bits(Z) == _bits(seq)
    want = ((y.astype(np.float64) * 1.5).astype(np.float32).astype(np.float64) - 2.0).astype(
        np.float32)
    assert np.array_equal(tp.to_numpy(Z), want)
    # offset (misaligned) and reversed views take the generic traversal
    for v in (tp.apply_index(Y, (slice(3, None),)), tp.apply_index(Y, (slice(None, None, -1),))):
        assert _bits(tp.chain(v, [("multiply", k15), ("add", km2)])) == \
            _bits(tp.add(tp.multiply(v, k15), km2))


OPS = ("add", "subtract", "multiply", "divide", "minimum", "maximum")
SCALARS = [lambda r: tp.Scalar(r.randint(-5, 5), tp.int16),
           lambda r: tp.Scalar(r.uniform(-3, 3), tp.float),
           lambda r: tp.Scalar(r.uniform(-3, 3), tp.half),
           lambda r: r.randint(-4, 4),            # host int -> int64
           lambda r: r.uniform(-2, 2),            # host float -> double
           lambda r: tp.Scalar(complex(r.uniform(-1, 1), r.uniform(-1, 1)), D.CFLOAT),
           lambda r: tp.Scalar(0, tp.int32)]      # integer division by zero


def test_random_chains_match_sequential_ops():
    rng, pr = np.random.default_rng(31), random.Random(31)
    n = 0
    while n < 200:
        x = rand_tensor(rng, pr, max_axes=3, max_extent=9)
        if x.dtype is D.CHALF:
            continue
        steps = []
        for _ in range(pr.randint(1, 4)):
            steps.append((pr.choice(OPS), pr.choice(SCALARS)(pr), pr.random() < 0.3))
        tp.clear_status()
        seq = x
        for op, s, sf in steps:
            seq = getattr(tp, op)(s, seq) if sf else getattr(tp, op)(seq, s)
        st_seq = tp.get_status()
        tp.clear_status()
        got = tp.chain(x, steps)
        st_got = tp.get_status()
        assert got.dtype is seq.dtype, (steps, x.dtype)
        assert tp.array_equal(got, seq), (steps, x.dtype, x.dims)
        assert st_got == st_seq, (steps, x.dtype)
        n += 1


def test_chain_into_dest_of_other_dtype():
    y = np.random.default_rng(3).uniform(-100, 100, 4096).astype(np.float32)
    Y = tp.from_numpy(y)
    d = tp.tensor_create((4096,), tp.int16)
    tp.chain(Y, [("multiply", tp.Scalar(3.0, tp.float)), ("add", tp.Scalar(0.5, tp.float))], dest=d)
    d2 = tp.tensor_create((4096,), tp.int16)
    tp.add(tp.multiply(Y, tp.Scalar(3.0, tp.float)), tp.Scalar(0.5, tp.float), dest=d2)
    assert _bits(d) == _bits(d2)


def test_chain_error_mode_raises_without_writing():
    x = tp.from_numpy(np.arange(1, 65, dtype=np.int32))
    d = tp.zeros((64,), tp.int32)
    with pytest.raises(tp.DomainError):
        tp.chain(x, [("divide", tp.Scalar(0, tp.int32))], dest=d, mode="error")
    assert np.all(tp.to_numpy(d) == 0)


def test_f32_chain_float_arithmetic_edges():
    """The all-float chain computes + - * with float-exact scalars in float
    arithmetic; that must equal the reference's compute-in-double, round
    once to float (ops.py:145-152, dtypes.py:270-278) on the edges where
    double rounding could show: subnormals, results that overflow to inf,
    signed zeros, inf / NaN operands and ties at the float rounding point."""
    rng = np.random.default_rng(41)
    fmax = np.finfo(np.float32).max
    tiny = np.finfo(np.float32).tiny
    edge = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, fmax, -fmax, tiny, -tiny, tiny / 3,
                     -tiny / 7, 1.0 + 2.0 ** -23, 1.0 + 2.0 ** -24, 3.0 * 2.0 ** -25, 16777217.0,
                     -16777215.0], np.float64).astype(np.float32)
    body = rng.standard_normal((1 << 16) + 3).astype(np.float32) * np.float32(
        2.0) ** rng.integers(-140, 127, (1 << 16) + 3).astype(np.float32)
    y = np.concatenate([np.tile(edge, 64), body]).astype(np.float32)
    Y = tp.from_numpy(y)
    scal = [tp.Scalar(v, tp.float) for v in (1.5, -2.0, 2.0 ** -24, 3.0e38, -0.0, 1.0 + 2.0 ** -23)]
    chains = [[("multiply", scal[0]), ("add", scal[1])],
              [("add", scal[2]), ("multiply", scal[3])],
              [("subtract", scal[4]), ("multiply", scal[5]), ("add", scal[2])],
              [("multiply", scal[3]), ("subtract", scal[1])]]
    for ch in chains:
        Z = tp.chain(Y, ch)
        seq = Y
        want = y.astype(np.float64)
        for op, s in ch:
            seq = getattr(tp, op)(seq, s)
            w = float(np.float32(s.value))
            with np.errstate(all="ignore"):
                want = {"add": want + w, "subtract": want - w, "multiply": want * w}[op]
                want = want.astype(np.float32).astype(np.float64)
        z = tp.to_numpy(Z)
        for ref in (tp.to_numpy(seq), want.astype(np.float32)):
            same = (z.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(z) & np.isnan(ref))
            assert same.all(), (ch, np.flatnonzero(~same)[:5])
