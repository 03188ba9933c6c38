"""Error / warning modes of the standalone layer on every entry family
(dtypes.CastContext semantics, reference dtypes.py:233-255):
reductions and products report cast loss too, flags are read for the
right device after all its streams, and results produced on a
`use_stream` override are visible to host reads without an explicit
stream sync (storage stream bookkeeping)."""

import numpy as np
import pytest

import paper_1810_08723_b200 as tp

pytestmark = pytest.mark.gpu


def test_reduce_cast_loss_error_and_warning():
    x = tp.from_nested([100, 100, 100], tp.int8)
    with pytest.raises(tp.DomainError):
        tp.reduce("sum", x, mode="error")
    seen = []
    prev = tp.set_warning_handler(seen.append)
    try:
        assert tp.reduce("sum", x, mode="warning").item() == 44
        assert len(seen) == 1
        assert tp.reduce("sum", x).item() == 44      # standard: wraps silently
        assert len(seen) == 1
    finally:
        tp.set_warning_handler(prev)


def test_matmul_cast_loss_error_and_warning():
    m = tp.from_nested([[100, 100], [100, 100]], tp.int8)
    with pytest.raises(tp.DomainError):
        tp.matmul(m, m, mode="error")
    seen = []
    prev = tp.set_warning_handler(seen.append)
    try:
        out = tp.matmul(m, m, mode="warning")
        assert tp.read_values(out) == [32, 32, 32, 32]   # 20000 wraps to int8 32
        assert len(seen) == 1
    finally:
        tp.set_warning_handler(prev)


def test_no_stale_flag_after_a_standard_overflow():
    x = tp.from_nested([100, 100, 100], tp.int8)
    tp.reduce("sum", x)                                   # wraps, sets nothing visible
    seen = []
    prev = tp.set_warning_handler(seen.append)
    try:
        tp.reduce("sum", tp.from_nested([1, 2], tp.int8), mode="warning")
        assert seen == []
    finally:
        tp.set_warning_handler(prev)


def test_elementwise_error_mode_raises_before_writing():
    src = tp.from_nested([1.0, 300.0], tp.double)
    dst = tp.tensor_create((2,), tp.int8)
    tp.fill(dst, 7)
    with pytest.raises(tp.DomainError):
        tp.copy(src, dst, mode="error")
    assert tp.read_values(dst) == [7, 7]


def test_use_stream_results_visible_to_host_reads():
    dev = tp.gpu(0)
    s = dev.create_stream()
    a = tp.from_numpy(np.arange(1 << 16, dtype=np.float32))
    with tp.use_stream(s):
        y = tp.multiply(a, 2.0)
        z = tp.add(y, 1.0)
    # no s.sync(): to_numpy orders the read after every stream that wrote z
    assert np.array_equal(tp.to_numpy(z), np.arange(1 << 16, dtype=np.float32) * 2 + 1)
    assert not z.storage.users            # host read drained the bookkeeping
    with tp.use_stream(s):
        w = tp.add(z, 1.0)
    del w                                 # the free waits for s (stream-ordered)
    s.sync()
