"""Maximum-size edge cases: > 2^31 elements and > 4 GiB byte offsets go
through the elementwise, chain and reduction kernels with 64-bit indexing
(SURVEY cfg5 is 2^30 elements = 8 GiB of f64)."""

import numpy as np
import pytest

import paper_1810_08723_b200 as tp

pytestmark = pytest.mark.gpu

N = (1 << 31) + 17


def test_int8_over_2g_elements_fill_add_sum():
    x = tp.tensor_create((N,), tp.int8)
    tp.fill(x, 1)
    y = tp.add(x, tp.Scalar(2, tp.int8))            # k_contig, 2^31+17 elements
    idx = [0, 1 << 31, N - 1]
    vals = [tp.read_values(tp.apply_index(y, (slice(i, i + 1),)))[0] for i in idx]
    assert vals == [3, 3, 3]
    s = tp.reduce("sum", x, dest=tp.tensor_create((), tp.int64))   # exact int sum
    assert s.item() == N
    del x, y


def test_f64_over_4gib_reduction_and_tail_view():
    n = (1 << 29) + 5                               # 4 GiB + 40 B of doubles
    x = tp.tensor_create((n,), tp.double)
    tp.fill(x, 0.5)
    assert tp.reduce("sum", x).item() == 0.5 * n
    tail = tp.apply_index(x, (slice(n - 3, None),))  # byte offset > 4 GiB
    tp.fill(tail, 2.0)
    assert tp.reduce("maximum", x).item() == 2.0
    assert tp.read_values(tp.multiply(tail, 3.0)) == [6.0, 6.0, 6.0]
    del x


def test_chain_over_2g_elements_f16():
    n = (1 << 31) + 9
    h = tp.tensor_create((n,), tp.half)
    tp.fill(h, 1.5)
    z = tp.chain(h, [("multiply", tp.Scalar(2.0, tp.half)), ("add", tp.Scalar(1.0, tp.half))])
    assert z.dtype is tp.half
    for i in (0, 1 << 31, n - 1):
        assert tp.read_values(tp.apply_index(z, (slice(i, i + 1),)))[0] == 4.0
    del h, z
