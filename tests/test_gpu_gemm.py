"""Tensor-core gemm parity (tcgen05 path) against the C oracle.

Tolerance: |C - C_oracle| <= 1e-2 * sum_k |a_ik||b_kj| for
half / bfloat16 operands (fp32 accumulation in TMEM vs the reference's
compensated double sum, one rounding each), 1e-5 for float operands (3xTF32
split products, fp32 accumulation; north_star's fp32 tolerance).  Layouts follow SURVEY §8d
cfg4: A a transposed column-major base (K-major), B column-major with a
padded leading dimension, a strided B (pack path), column-major C.
"""

import ctypes as C

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import abi

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _host(t):
    """numpy values of a gpu tensor as float64 (bf16 decoded)."""
    if t.dtype is tp.bfloat16:
        raw = tp.to_numpy(tp.tensors.Tensor(t.storage, t.offset, t.dims, t.strides, tp.uint16))
        return (raw.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return tp.to_numpy(t).astype(np.float64)


def _make(rng, dt, rows, cols, pad=0):
    base = rng.uniform(-1, 1, (rows + pad, cols)).astype(np.float32)
    if dt is tp.bfloat16:
        raw = np.asfortranarray((base.view(np.uint32) >> 16).astype(np.uint16))
        t = tp.from_numpy(raw, dtype=tp.bfloat16)
    elif dt is tp.float:
        t = tp.from_numpy(np.asfortranarray(base))
    else:
        t = tp.from_numpy(np.asfortranarray(base.astype(np.float16)))
    return tp.apply_index(t, (slice(0, rows), slice(None))) if pad else t


def _oracle_block(A, B, rows, cols, out_dtype):
    """Oracle C[rows, cols] via tpo_matmul on host copies of A rows / B cols."""
    from oracle import oracle
    a = _host(A)[rows, :]
    b = _host(B)[:, cols]
    m, k = a.shape
    n = b.shape[1]
    a64 = np.asfortranarray(a)
    b64 = np.asfortranarray(b)
    out = np.zeros((m, n), dtype=np.float64, order="F")
    L = oracle.lib()
    d = abi.make_operand(out.ctypes.data, 0, tp.double.code, False)
    ao = abi.make_operand(a64.ctypes.data, 0, tp.double.code, False)
    bo = abi.make_operand(b64.ctypes.data, 0, tp.double.code, False)
    st = C.c_uint32(0)
    arr = lambda s: (C.c_int64 * 2)(*s)
    L.tpo_matmul(C.byref(d), arr((8, 8 * m)), C.byref(ao), arr((8, 8 * m)), C.byref(bo),
                 arr((8, 8 * k)), m, n, k, tp.double.code, 0, C.byref(st))
    bound = np.abs(a) @ np.abs(b)
    return out, bound


def _check(Cg, A, B, rng, samples=48, tol=None):
    tol = tol if tol is not None else (1e-5 if A.dtype is tp.float else TOL)
    m, n = Cg.dims
    rows = np.sort(rng.choice(m, min(samples, m), replace=False))
    cols = np.sort(rng.choice(n, min(samples, n), replace=False))
    want, bound = _oracle_block(A, B, rows, cols, Cg.dtype)
    got = _host(Cg)[np.ix_(rows, cols)]
    err = np.abs(got - want)
    assert np.all(err <= tol * bound + 1e-30), float((err / (bound + 1e-30)).max())


@pytest.mark.parametrize("dt", [tp.half, tp.bfloat16])
@pytest.mark.parametrize("m,n,k", [(256, 256, 128), (384, 640, 320), (1000, 700, 333),
                                   (2048, 2048, 2048)])
def test_gemm_tn_layout(dt, m, n, k):
    rng = np.random.default_rng(m + n + k)
    Ab = _make(rng, dt, k, m)          # column-major (k, m) base
    A = tp.transpose(Ab)               # (m, k) K-major, as SURVEY cfg4
    B = _make(rng, dt, k, n, pad=64)   # padded leading dimension
    Cg = tp.matmul(A, B)
    assert Cg.dtype is dt
    _check(Cg, A, B, rng)


@pytest.mark.parametrize("dt", [tp.half, tp.bfloat16])
def test_gemm_pack_paths(dt):
    rng = np.random.default_rng(3)
    m, n, k = 512, 384, 256
    A = _make(rng, dt, m, k)                        # M-major A -> packed
    Bb = _make(rng, dt, 2 * k, n)
    B = tp.apply_index(Bb, (slice(None, None, 2), slice(None)))  # element stride 2 -> packed
    Cg = tp.matmul(A, B)
    _check(Cg, A, B, rng)
    # float destination (cast-on-write) and row-major destination
    Cf = tp.tensor_create((m, n), tp.float)
    tp.matmul(A, B, dest=Cf)
    _check(Cf, A, B, rng)
    Crow = tp.transpose(tp.tensor_create((n, m), dt))
    tp.matmul(A, B, dest=Crow)
    _check(Crow, A, B, rng)


def test_gemm_batched_matches_slices():
    rng = np.random.default_rng(4)
    m, n, k, nb = 256, 256, 128, 4
    a = rng.uniform(-1, 1, (m, k, nb)).astype(np.float16)
    b = rng.uniform(-1, 1, (k, n, nb)).astype(np.float16)
    A = tp.from_numpy(np.asfortranarray(a))
    B = tp.from_numpy(np.asfortranarray(b))
    Cg = tp.matmul_batched(A, B)
    got = tp.to_numpy(Cg).astype(np.float64)
    for i in range(nb):
        want = a[:, :, i].astype(np.float64) @ b[:, :, i].astype(np.float64)
        bound = np.abs(a[:, :, i]).astype(np.float64) @ np.abs(b[:, :, i]).astype(np.float64)
        assert np.all(np.abs(got[:, :, i] - want) <= TOL * bound + 1e-6)


def test_gemm_nonfinite_becomes_nan():
    a = np.ones((256, 128), dtype=np.float16)
    a[3, 5] = np.inf
    b = np.ones((128, 256), dtype=np.float16)
    Cg = tp.to_numpy(tp.matmul(tp.from_numpy(np.asfortranarray(a)),
                               tp.from_numpy(np.asfortranarray(b))))
    assert np.isnan(Cg[3]).all() and np.all(Cg[4] == 128)


@pytest.mark.parametrize("m,n,k", [(256, 256, 128), (384, 640, 320), (1000, 700, 333),
                                   (2048, 1024, 4096)])
def test_gemm_f32_tf32x3(m, n, k):
    """float x float on tcgen05 kind::tf32 (3xTF32), K-major A and B."""
    rng = np.random.default_rng(m * 7 + n + k)
    A = tp.transpose(_make(rng, tp.float, k, m))
    B = _make(rng, tp.float, k, n, pad=32)
    Cg = tp.matmul(A, B)
    assert Cg.dtype is tp.float
    _check(Cg, A, B, rng)


@pytest.mark.parametrize("dt", [tp.half, tp.bfloat16, tp.float])
def test_gemm_mn_major_operands(dt):
    """A column-major (M contiguous) and B row-major (N contiguous): both
    operands are fed MN-major to the tensor cores, no pack."""
    rng = np.random.default_rng(21)
    m, n, k = 640, 512, 448
    A = _make(rng, dt, m, k)                      # M-major
    B = tp.transpose(_make(rng, dt, n, k))        # N-major
    _check(tp.matmul(A, B), A, B, rng)
    Bk = _make(rng, dt, k, n)                     # mixed: A MN-major, B K-major
    _check(tp.matmul(A, Bk), A, Bk, rng)
    At = tp.transpose(_make(rng, dt, k, m))       # mixed: A K-major, B MN-major
    _check(tp.matmul(At, B), At, B, rng)


def test_gemm_f32_strided_and_swapped():
    """f32 operands without a unit stride or byte-swapped go through the
    generic split; result still within 1e-5 of sum|a||b|."""
    rng = np.random.default_rng(22)
    m, n, k = 384, 256, 320
    Ab = _make(rng, tp.float, 2 * m, k)
    A = tp.apply_index(Ab, (slice(None, None, 2), slice(None)))
    B = _make(rng, tp.float, k, n)
    _check(tp.matmul(A, B), A, B, rng)
    Bs = _make(rng, tp.float, k, n)
    want = tp.to_numpy(Bs).copy()
    tp.byteswap(Bs)
    Cg = tp.to_numpy(tp.matmul(A, Bs)).astype(np.float64)
    a = tp.to_numpy(A).astype(np.float64)
    bound = np.abs(a) @ np.abs(want.astype(np.float64))
    assert np.all(np.abs(Cg - a @ want.astype(np.float64)) <= 1e-5 * bound)


@pytest.mark.parametrize("dt", [tp.half, tp.float])
def test_gemm_batched_col_major(dt):
    """SURVEY cfg4 batched layout: A, B, C column-major with batch slowest
    (A MN-major, B K-major)."""
    rng = np.random.default_rng(23)
    m, n, k, nb = 384, 256, 192, 3
    npd = np.float16 if dt is tp.half else np.float32
    a = rng.uniform(-1, 1, (m, k, nb)).astype(npd)
    b = rng.uniform(-1, 1, (k, n, nb)).astype(npd)
    Cg = tp.to_numpy(tp.matmul_batched(tp.from_numpy(np.asfortranarray(a)),
                                       tp.from_numpy(np.asfortranarray(b)))).astype(np.float64)
    tol = TOL if dt is tp.half else 1e-5
    for i in range(nb):
        a64, b64 = a[:, :, i].astype(np.float64), b[:, :, i].astype(np.float64)
        bound = np.abs(a64) @ np.abs(b64)
        assert np.all(np.abs(Cg[:, :, i] - a64 @ b64) <= tol * bound + 1e-30)


@pytest.mark.parametrize("dt", [tp.half, tp.bfloat16])
@pytest.mark.parametrize("m,n,k,nb,ldpad", [(1000, 700, 333, 1, 0), (256, 288, 64, 1, 8),
                                             (330, 260, 96, 3, 0), (300, 300, 80, 1, 3)])
def test_gemm_col_major_dest_every_element(dt, m, n, k, nb, ldpad):
    """Column-major 16-bit destinations, checked element by element: whole
    32 x 32 chunks go through the bulk-tensor-store epilogue, ragged edge
    chunks through the plain-store path of the same tile, and a leading
    dimension that is not a multiple of 16 bytes (ldpad 3) takes the plain
    path throughout."""
    rng = np.random.default_rng(m + n + k + nb + ldpad)
    npd = np.float16
    a = rng.uniform(-1, 1, (m, k, nb)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n, nb)).astype(np.float32)
    if dt is tp.bfloat16:
        a = (a.view(np.uint32) & 0xffff0000).view(np.float32)
        b = (b.view(np.uint32) & 0xffff0000).view(np.float32)

    def dev(x):
        if dt is tp.bfloat16:
            raw = (np.asfortranarray(x).view(np.uint32) >> 16).astype(np.uint16)
            return tp.from_numpy(np.asfortranarray(raw), dtype=tp.bfloat16)
        return tp.from_numpy(np.asfortranarray(x.astype(npd)))

    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    if dt is tp.half:
        a64, b64 = a.astype(npd).astype(np.float64), b.astype(npd).astype(np.float64)
    base = tp.tensor_create((m + ldpad, n, nb), dt)
    Cv = tp.apply_index(base, (slice(0, m), slice(None), slice(None)))
    if nb == 1:
        A = tp.apply_index(dev(a), (slice(None), slice(None), 0))
        B = tp.apply_index(dev(b), (slice(None), slice(None), 0))
        tp.matmul(A, B, dest=tp.apply_index(Cv, (slice(None), slice(None), 0)))
    else:
        tp.matmul_batched(dev(a), dev(b), dest=Cv)
    got = _host(Cv).reshape(m, n, nb, order="F")
    for i in range(nb):
        want = a64[:, :, i] @ b64[:, :, i]
        bound = np.abs(a64[:, :, i]) @ np.abs(b64[:, :, i])
        assert np.all(np.abs(got[:, :, i] - want) <= TOL * bound + 1e-6), i
