"""Parity at BASELINE.json's stated sizes (SURVEY §8d "Parity at measurement
scale"): cfg3 (f64 8192^2 reductions), cfg4 (8192^3 gemm, batched
64 x 2048^3) and cfg5 (2^30-element casts and the fused chain) on the B200,
against the C oracle or exact numpy restatements of the reference rules.

Tolerances (north_star): reductions rel 1e-12 (f64; max exact); gemm
|C - C_ref| <= 1e-2 * sum|a||b| for f16/bf16 and 1e-5 for f32; casts and
the chain bit-exact.
"""

import ctypes as C

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import abi
from paper_1810_08723_b200.plan import build_plan

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- cfg3
@pytest.fixture(scope="module")
def cfg3():
    x = np.asfortranarray(np.random.default_rng(5).random((8192, 8192)))
    return x, tp.from_numpy(x)


def _oracle_reduce(op, x, axes, p=2.0):
    """tpo_reduce (the C restatement of ops.reduce / _reduction_acc,
    OpenMP) on the host copy, with the reference's outer/inner plans
    (ops.py:490-495)."""
    from oracle import oracle
    n0, n1 = x.shape
    strides = (8, 8 * n0)
    if axes is None:
        kept, red = [], [0, 1]
    else:
        kept, red = [k for k in (0, 1) if k not in axes], list(axes)
    rdims = tuple(x.shape[k] for k in kept)
    out = np.zeros(max(1, int(np.prod(rdims))) if rdims else 1, dtype=np.float64)
    dstr = tuple(8 * int(np.prod(rdims[:i])) for i in range(len(rdims)))
    outer = build_plan(rdims, [dstr, tuple(strides[k] for k in kept)])
    inner = build_plan(tuple(x.shape[k] for k in red), [tuple(strides[k] for k in red)])
    code = abi.REDUCE_CODE[op]
    d = abi.make_operand(out.ctypes.data, 0, tp.double.code, False)
    a = abi.make_operand(x.ctypes.data, 0, tp.double.code, False)
    st = C.c_uint32(0)
    oracle.lib().tpo_reduce(code, p, C.byref(outer.to_c()), C.byref(inner.to_c()), C.byref(d),
                            C.byref(a), tp.double.code, 0, C.byref(st))
    return out


@pytest.mark.parametrize("op", ["sum", "maximum", "norm"])
@pytest.mark.parametrize("axes", [(0,), (1,), None])
def test_cfg3_reductions_full_size(cfg3, op, axes):
    x, X = cfg3
    got = tp.to_numpy(tp.reduce(op, X, axes=axes)).reshape(-1)
    want = _oracle_reduce(op, x, axes)
    if op == "maximum":
        assert np.array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)


# ---------------------------------------------------------------- cfg4
def _gemm_inputs(dt, rng, rows, cols, pad=0, batch=None):
    shape = (rows + pad, cols) if batch is None else (rows, cols, batch)
    base = rng.uniform(-1, 1, shape).astype(np.float32)
    if dt is tp.bfloat16:
        raw = np.asfortranarray((base.view(np.uint32) >> 16).astype(np.uint16))
        host = (raw.astype(np.uint32) << 16).view(np.float32)
        t = tp.from_numpy(raw, dtype=tp.bfloat16)
    else:
        npd = np.float16 if dt is tp.half else np.float32
        host = np.asfortranarray(base.astype(npd))
        t = tp.from_numpy(host)
    if pad:
        t = tp.apply_index(t, (slice(0, rows), slice(None)))
        host = host[:rows]
    return host.astype(np.float64), t


def _download(t):
    if t.dtype is tp.bfloat16:
        raw = tp.to_numpy(tp.tensors.Tensor(t.storage, t.offset, t.dims, t.strides, tp.uint16))
        return (raw.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return tp.to_numpy(t).astype(np.float64)


@pytest.mark.parametrize("dt,tol", [(tp.half, 1e-2), (tp.bfloat16, 1e-2), (tp.float, 1e-5)])
def test_cfg4_gemm_8192_sampled(dt, tol):
    """SURVEY cfg4: A = transpose of a column-major base (K-major), B a
    column-major view with padded leading dimension, C column-major;
    512 sampled (i, j) entries against float64 dot products."""
    m = 8192
    rng = np.random.default_rng(6)
    at, Ab = _gemm_inputs(dt, rng, m, m)           # (k, m) base
    b, B = _gemm_inputs(dt, rng, m, m, pad=64)
    Cg = tp.matmul(tp.transpose(Ab), B)
    assert Cg.dtype is dt
    got = _download(Cg)
    i = rng.integers(0, m, 512)
    j = rng.integers(0, m, 512)
    a_rows = at[:, i]                              # column i of the base = row i of A
    want = np.einsum("ks,ks->s", a_rows, b[:, j])
    bound = np.einsum("ks,ks->s", np.abs(a_rows), np.abs(b[:, j]))
    err = np.abs(got[i, j] - want)
    assert np.all(err <= tol * bound), float((err / bound).max())


def test_cfg4_batched_64x2048_sampled():
    nb, s = 64, 2048
    rng = np.random.default_rng(7)
    a, A = _gemm_inputs(tp.half, rng, s, s, batch=nb)
    b, B = _gemm_inputs(tp.half, rng, s, s, batch=nb)
    got = _download(tp.matmul_batched(A, B))
    for q in range(nb):
        i = rng.integers(0, s, 16)
        j = rng.integers(0, s, 16)
        want = np.einsum("sk,ks->s", a[i, :, q], b[:, j, q])
        bound = np.einsum("sk,ks->s", np.abs(a[i, :, q]), np.abs(b[:, j, q]))
        assert np.all(np.abs(got[i, j, q] - want) <= 1e-2 * bound), q


# ---------------------------------------------------------------- cfg5
N5 = 1 << 30
Q = N5 // 4


def _quarter_slices(t):
    """2^22 elements from each quarter (each of the four shard slabs)."""
    out = []
    for qi in range(4):
        lo = qi * Q + (Q // 2)
        out.append((lo, tp.to_numpy(tp.apply_index(t, (slice(lo, lo + (1 << 22)),)))))
    return out


def _big_endian_source(dtype_np, dt, host):
    """2^30-element big-endian tensor built on the device from four copies
    of a 2^28 host slab (the bench's construction)."""
    chunk = tp.from_numpy(host.astype(dtype_np), None)
    S = tp.tensor_create((N5,), dt)
    S.byteorder = "big"
    for i in range(4):
        tp.copy(chunk, tp.apply_index(S, (slice(i * Q, (i + 1) * Q),)))
    return S


def test_cfg5_casts_and_chain_full_size():
    rng = np.random.default_rng(8)
    slab = rng.uniform(-1e3, 1e3, Q)
    S = _big_endian_source(">f8", tp.double, slab)
    Y = tp.cast(S, tp.float)
    del S
    want_y = slab.astype(np.float32)
    idx = rng.integers(0, N5, 100_000)
    for lo, got in _quarter_slices(Y):
        assert np.array_equal(got, want_y[(lo % Q):(lo % Q) + (1 << 22)])
    y_all = tp.to_numpy(Y)
    assert np.array_equal(y_all[idx], want_y[idx % Q])
    del y_all
    # multiply then add: sequential and fused chain, bit-identical to the
    # reference's double compute + one rounding per op
    k15, km2 = tp.Scalar(1.5, tp.float), tp.Scalar(-2.0, tp.float)
    Z = tp.add(tp.multiply(Y, k15), km2)
    Zc = tp.chain(Y, [("multiply", k15), ("add", km2)])
    want_z = ((want_y.astype(np.float64) * 1.5).astype(np.float32).astype(np.float64)
              - 2.0).astype(np.float32)
    for t in (Z, Zc):
        for lo, got in _quarter_slices(t):
            assert np.array_equal(got, want_z[(lo % Q):(lo % Q) + (1 << 22)])
    z_all = tp.to_numpy(Zc)
    assert np.array_equal(z_all[idx], want_z[idx % Q])
    del Y, Z, Zc, z_all
    # int16 big-endian -> half
    s16 = np.random.default_rng(9).integers(-3000, 3000, Q).astype(np.int16)
    S16 = _big_endian_source(">i2", tp.int16, s16)
    H = tp.cast(S16, tp.half)
    want_h = s16.astype(np.float16)
    for lo, got in _quarter_slices(H):
        assert np.array_equal(got.view(np.uint16),
                              want_h[(lo % Q):(lo % Q) + (1 << 22)].view(np.uint16))
    del S16, H
