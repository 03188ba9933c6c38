"""GPU reductions at sizes that split every output into many chunks
(single-pass vector kernels with last-block finalize, and the scalar
fallbacks): sum / norm / min / max over f64 and f32 sources, row mode
(reduced axis unit-stride), column mode (outputs unit-stride) and full
reductions, with misaligned starts, reversed and strided views and odd
extents.  Every table call is replayed through the C oracle (reference
ops.reduce / kernels.reduce_strided semantics, ops.py:437-513,
kernels.py:305-320); sums and norms compare within rel 1e-12 (f64 result)
or exactly after rounding to f32, min/max bit-exact including the
first-element-NaN rule (kernels.py:58-65 via ops.py:527-544)."""

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from shadow import ShadowOracle

pytestmark = pytest.mark.gpu

OPS = ("sum", "norm", "minimum", "maximum")


def _views(x):
    X = tp.from_numpy(np.asfortranarray(x))
    yield "plain", X
    yield "offset", tp.apply_index(X, (slice(1, None), slice(None)))      # misaligned start
    yield "reversed", tp.apply_index(X, (slice(None, None, -1), slice(None)))
    yield "strided", tp.apply_index(X, (slice(None), slice(None, None, 2)))
    yield "transposed", tp.transpose(X)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_reduce_multichunk(dtype):
    rng = np.random.default_rng(11)
    x = rng.uniform(-4, 4, (3002, 1030)).astype(dtype)
    x[5, 7] = x[900, 7]          # ties for min/max
    with ShadowOracle() as so:
        for _name, V in _views(x):
            for op in OPS:
                for axes in ((0,), (1,), None):
                    tp.reduce(op, V, axes=axes)
    assert so.calls >= 5 * 4 * 3
    assert not so.failures, so.failures[:3]


def test_reduce_full_large_f64():
    rng = np.random.default_rng(12)
    x = rng.random(1 << 22)
    X = tp.from_numpy(x)
    s = tp.read_values(tp.reduce("sum", X))[0]
    assert abs(s - np.sum(x)) <= 1e-12 * abs(np.sum(x))
    with ShadowOracle() as so:
        for op in OPS:
            tp.reduce(op, X)
            tp.reduce(op, tp.apply_index(X, (slice(3, None),)))
    assert not so.failures, so.failures[:3]


def test_reduce_nan_first_and_inner():
    x = np.random.default_rng(13).random((4096, 300))
    x[0, 3] = np.nan      # first element of column 3 (axis-0 reduce): NaN result
    x[77, 5] = np.nan     # inner NaN: skipped by min/max
    y = x.T.copy()        # row-mode counterpart
    with ShadowOracle() as so:
        for arr in (x, y):
            X = tp.from_numpy(np.asfortranarray(arr))
            for op in ("minimum", "maximum", "sum"):
                for axes in ((0,), (1,), None):
                    tp.reduce(op, X, axes=axes)
    assert not so.failures, so.failures[:3]


def test_reduce_repeatable():
    """Results do not depend on which block finishes last."""
    x = np.random.default_rng(14).standard_normal((8192, 512))
    X = tp.from_numpy(np.asfortranarray(x))
    for axes in ((0,), (1,), None):
        a = tp.to_numpy(tp.reduce("sum", X, axes=axes))
        for _ in range(3):
            b = tp.to_numpy(tp.reduce("sum", X, axes=axes))
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_signed_zero_ties_keep_first():
    """min/max ties between -0.0 and +0.0 resolve to the FIRST element in
    plan order (kernels.py:58-65 via ops.py:527-544), in every kernel."""
    rng = np.random.default_rng(15)
    x = -rng.random((2500, 1030))            # all negative ...
    z = rng.random((2500, 1030)) < 0.5
    x[:, ::3] = np.where(z[:, ::3], -0.0, 0.0)   # ... some columns all-zero, random signs
    x[::7, :] = np.where(z[::7, :], -0.0, 0.0)   # ... and some rows
    with ShadowOracle() as so:
        for arr in (x, -x):
            X = tp.from_numpy(np.asfortranarray(arr))
            for op in ("minimum", "maximum"):
                for axes in ((0,), (1,), None):
                    tp.reduce(op, X, axes=axes)
    assert not so.failures, so.failures[:3]


@pytest.mark.parametrize("shape", [(256, 20000), (3000, 700), (160000, 40)])
def test_column_chunking_regimes(shape):
    """Column mode (outputs unit-stride) across its row-chunk regimes:
    few outputs / long rows (C capped at 64), C rounded down to whole
    finalize batches, and many outputs (C = 1, no finalize); NaN in a
    chunk's first row, ties and signed zeros straddling chunk edges."""
    rng = np.random.default_rng(16)
    x = rng.uniform(-2, 2, shape)
    o, n = shape
    x[3, :] = 0.0
    x[3, n // 2:] = -0.0                 # a zero extreme whose sign is set by the first zero
    x[5, n // 3] = np.nan                # inner NaN (skipped by min/max)
    x[7, 0] = np.nan                     # first element NaN: NaN result
    x[9, n - 1] = x[9, :].max()          # tie at the last row
    with ShadowOracle() as so:
        for dt in (np.float64, np.float32):
            X = tp.from_numpy(np.asfortranarray(x.astype(dt)))
            for op in OPS:
                tp.reduce(op, X, axes=(1,))
    assert so.calls >= 8
    assert not so.failures, so.failures[:3]
