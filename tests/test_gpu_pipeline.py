"""GPU pipeline parity: random strided programs through the public API
(the pattern of the reference's tests/test_ops.py:144-174 and
tests/test_device_parity.py:17-57), every table call shadow-checked
against the C oracle on the same bytes."""

import math
import random

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import dtypes as D
from shadow import ShadowOracle

pytestmark = pytest.mark.gpu

ALL = D.ALL_DTYPES


def rand_array(rng, d, dims):
    n = int(np.prod(dims)) if dims else 1
    if d is D.BOOL:
        return (rng.random(n) < 0.5).reshape(dims)
    if d.is_complex:
        npd = D.NUMPY_NAME[d] or "complex64"
        v = (rng.uniform(-100, 100, n) + 1j * rng.uniform(-100, 100, n)).astype(npd)
        return v.reshape(dims)
    if d.is_float:
        v = rng.uniform(-300, 300, n)
        sel = rng.random(n)
        v[sel < 0.05] = np.nan
        v[(sel > 0.05) & (sel < 0.08)] = np.inf
        v[(sel > 0.08) & (sel < 0.1)] = -0.0
        return v.astype(D.NUMPY_NAME[d]).reshape(dims)
    lo, hi = D.int_range(d)
    return rng.integers(max(lo, -1000), min(hi, 1000), n, endpoint=True).astype(
        D.NUMPY_NAME[d]).reshape(dims)


def rand_tensor(rng, pyrng, d=None, max_axes=3, max_extent=6, min_axes=0):
    d = d or pyrng.choice(ALL)
    if d is D.CHALF:
        d = D.CFLOAT
    dims = tuple(pyrng.randint(1, max_extent) for _ in range(pyrng.randint(min_axes, max_axes)))
    t = tp.from_numpy(np.asfortranarray(rand_array(rng, d, dims)))
    parts = []
    for e in t.dims:
        c = pyrng.random()
        if c < 0.2:
            s = pyrng.randrange(e)
            parts.append(slice(s, s + 1))
        elif c < 0.6:
            parts.append(slice(None, None, pyrng.choice([1, 2, -1, -2])))
        else:
            parts.append(slice(None))
    v = tp.apply_index(t, tuple(parts)) if parts else t
    if v.ndim > 1 and pyrng.random() < 0.5:
        order = list(range(v.ndim))
        pyrng.shuffle(order)
        v = tp.permute_axes(v, order)
    if pyrng.random() < 0.25:
        tp.byteswap(v)
    return v


def test_random_binary_programs():
    rng, pr = np.random.default_rng(5), random.Random(5)
    with ShadowOracle() as so:
        n = 0
        while n < 300:
            a = rand_tensor(rng, pr)
            b = rand_tensor(rng, pr)
            try:
                tp.tensors.broadcast_result_dims(a.dims, b.dims)
            except tp.ShapeError:
                continue
            op = pr.choice(tp.ops.BINARY_OPS)
            getattr(tp, op)(a, b)
            n += 1
    assert so.calls >= 300
    assert not so.failures, so.failures[:5]


def test_scalar_operands_by_value():
    rng, pr = np.random.default_rng(6), random.Random(6)
    with ShadowOracle() as so:
        for _ in range(80):
            a = rand_tensor(rng, pr, min_axes=1)
            s = pr.choice([2, -3, 1.5, -0.25, 2.0 + 1.0j, True, 1e10,
                           tp.Scalar(1.5, tp.float), tp.Scalar(-2.0, tp.float)])
            op = pr.choice(tp.ops.BINARY_OPS)
            getattr(tp, op)(a, s) if pr.random() < 0.5 else getattr(tp, op)(s, a)
    assert not so.failures, so.failures[:5]


def test_random_unary_and_copy():
    rng, pr = np.random.default_rng(7), random.Random(7)
    with ShadowOracle() as so:
        for op in tp.ops.UNARY_OPS:
            for d in ALL:
                a = rand_tensor(rng, pr, d, min_axes=1)
                getattr(tp, op)(a)
        for _ in range(200):
            a = rand_tensor(rng, pr, min_axes=1)
            tp.cast(a, pr.choice(ALL))
    assert not so.failures, so.failures[:5]


def test_random_reductions():
    rng, pr = np.random.default_rng(8), random.Random(8)
    with ShadowOracle(tol=None) as so:
        for op in tp.ops.REDUCE_OPS:
            for d in ALL:
                a = rand_tensor(rng, pr, d, min_axes=1, max_extent=9)
                axes = None if pr.random() < 0.3 else tuple(
                    sorted(pr.sample(range(a.ndim), pr.randint(1, a.ndim))))
                tp.reduce(op, a, axes=axes, p=pr.choice([1.0, 2.0, 3.0]))
    assert not so.failures, so.failures[:5]


def test_random_matmul():
    rng, pr = np.random.default_rng(9), random.Random(9)
    with ShadowOracle() as so:
        for d in ALL:
            for _ in range(3):
                m, n, k = pr.randint(1, 70), pr.randint(1, 70), pr.randint(0, 90)
                A = rand_tensor(rng, pr, d, min_axes=2, max_axes=2, max_extent=2)
                A = tp.from_numpy(np.asfortranarray(rand_array(rng, d if d is not D.CHALF
                                                                else D.CFLOAT, (k, m))))
                A = tp.transpose(A)
                B = tp.from_numpy(np.asfortranarray(rand_array(rng, d if d is not D.CHALF
                                                                else D.CFLOAT, (k, n))))
                tp.matmul(A, B)
    assert not so.failures, so.failures[:5]


def test_modes_and_status():
    tp.clear_status()
    a = tp.from_nested([1, 2], tp.int32)
    z = tp.from_nested([0, 1], tp.int32)
    out = tp.divide(a, z)
    assert tp.read_values(out) == [0, 2]
    assert "integer-division-by-zero" in tp.get_status()
    tp.clear_status()
    with pytest.raises(tp.DomainError):
        tp.divide(a, z, mode="error")
    neg = tp.from_nested([-1.0, 4.0], tp.double)
    r = tp.square_root(neg)
    v = tp.read_values(r)
    assert math.isnan(v[0]) and v[1] == 2.0
    assert "domain-violation" in tp.get_status()
    c = tp.square_root(neg, mode="complex")
    assert c.dtype is tp.complex_double
    assert tp.read_values(c)[0] == 1j
    with pytest.raises(tp.DomainError):
        tp.cast(tp.from_nested([1e20], tp.double), tp.int8, mode="error")
    msgs = []
    tp.set_warning_handler(msgs.append)
    try:
        tp.cast(tp.from_nested([1e20, 3.0], tp.double), tp.int8, mode="warning")
    finally:
        tp.set_warning_handler(None)
    assert len(msgs) == 1
    tp.clear_status()


def test_reference_examples():
    # reference tests/test_ops.py examples
    a = tp.from_nested([1, 2], tp.int8)
    b = tp.from_nested([3, 4], tp.uint8)
    out = tp.add(a, b)
    assert out.dtype is tp.int16 and tp.read_values(out) == [4, 6]
    q = tp.divide(tp.from_nested([7, -7, 7, -7], tp.int32), tp.from_nested([2, 2, -2, -2], tp.int32))
    assert tp.read_values(q) == [3, -3, -3, 3]
    assert tp.reduce("sum", tp.arange(25)).item() == 300
    assert tp.reduce("norm", tp.from_nested([3.0, 4.0])).item() == 5.0
    m = tp.reshape(tp.arange(25), (5, 5))
    assert tp.read_values(tp.reduce("sum", m, axes=(0,))) == [10, 35, 60, 85, 110]
    assert tp.reduce("sum", tp.from_nested([100, 100, 40], tp.int8)).item() == -16
    assert tp.inner(tp.from_nested([1.0, 2.0, 3.0]), tp.from_nested([4.0, 5.0, 6.0])).value == 32.0
    o = tp.outer(tp.from_nested([1.0, 2.0]), tp.from_nested([3.0, 4.0]))
    assert o.tolist() == [[3.0, 4.0], [6.0, 8.0]]
    i2 = tp.matmul(tp.from_nested([[1, 2], [3, 4]], tp.int32), tp.from_nested([[1, 2], [3, 4]], tp.int32))
    assert i2.tolist() == [[7, 10], [15, 22]]
    assert tp.read_values(tp.cast(tp.from_nested([256, 130, -1]), tp.uint8)) == [0, 130, 255]
    assert tp.read_values(tp.cast(tp.from_nested([2049.0, 1e6]), tp.half)) == [2048.0, math.inf]
    s = tp.reduce("sum", tp.from_nested([16777216.0, 1.0, 1.0], tp.float)).item()
    assert s == 16777218.0
    e = tp.reduce("sum", tp.tensor_create((0,), tp.double)).item()
    assert e == 0.0


def test_fsum_within_one_ulp_any_axis_order():
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (10, 10, 10)) * 10.0 ** rng.integers(-5, 5, (10, 10, 10))
    t = tp.from_numpy(np.asfortranarray(x))
    for order in ((0, 1, 2), (2, 0, 1), (1, 2, 0)):
        v = tp.permute_axes(t, order)
        got = tp.reduce("sum", v).item()
        want = math.fsum(x.ravel())
        assert abs(got - want) <= math.ulp(want)
