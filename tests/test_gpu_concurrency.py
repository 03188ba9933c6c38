"""Concurrent host threads, one stream each, on disjoint tensors (the
pattern of the reference's tests/test_device_parity.py:70-106: 6 threads,
FIFO per stream): every thread's results equal the single-threaded run bit
for bit, and per-stream order holds (each step reads the previous step's
output)."""

import threading

import numpy as np
import pytest

import paper_1810_08723_b200 as tp

pytestmark = pytest.mark.gpu


def _work(seed, stream=None):
    rng = np.random.default_rng(seed)
    x = tp.from_numpy(np.asfortranarray(rng.random((700, 300))))
    h = tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (256, 192)).astype(np.float16)))
    g = tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (192, 320)).astype(np.float16)))
    out = []

    def run():
        y = x
        for i in range(6):                      # each step consumes the last
            y = tp.chain(y, [("multiply", 1.0001), ("add", float(i))])
        out.append(tp.reduce("sum", y, axes=(0,)))
        out.append(tp.reduce("maximum", y))
        out.append(tp.matmul(h, g))
        out.append(tp.add(tp.transpose(x), 1.5))
        return [tp.to_numpy(t) for t in out]

    if stream is None:
        return run()
    with tp.use_stream(stream):
        res = run()
    stream.sync()
    return res


def test_threads_with_own_streams_match_serial():
    seeds = list(range(6))
    want = {s: _work(s) for s in seeds}
    got, errs = {}, []
    dev = tp.gpu(0)

    def worker(s):
        try:
            st = dev.create_stream()
            for _ in range(3):
                got[s] = _work(s, st)
        except BaseException as exc:  # pragma: no cover - reported below
            errs.append(exc)

    ts = [threading.Thread(target=worker, args=(s,)) for s in seeds]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for s in seeds:
        for a, b in zip(want[s], got[s]):
            assert a.dtype == b.dtype and a.shape == b.shape
            assert a.tobytes() == b.tobytes(), s
