"""Probe: cfg3 axis-1 reductions on random vs constant data (device ms)."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1810_08723_b200 as tp  # noqa: E402
from paper_1810_08723_b200 import _native  # noqa: E402

L = _native.lib()
dev = tp.list_devices()[0]
stream = dev.default_stream()
fb = dev.allocate(bench.FLUSH_BYTES)
for name, arr in (("random", np.random.default_rng(5).random((8192, 8192))),
                  ("ones", np.ones((8192, 8192))), ("neg", -np.random.default_rng(5).random((8192, 8192)))):
    X = tp.from_numpy(np.asfortranarray(arr), dev)
    for op in ("sum", "maximum", "minimum"):
        for axes in ((1,), (0,)):
            f = lambda: tp.reduce(op, X, axes=axes)  # noqa: E731
            for _ in range(3):
                f()
            stream.sync()
            ms = bench.timed_steps(L, stream, f, 10, lambda: bench.l2_flush(L, stream, fb))
            m = statistics.mean(ms)
            print(f"{name:7s} {op:8s} axes={axes}  {m * 1e3:7.1f} us  {8 * 8192 ** 2 / m / 1e6:7.1f} GB/s")
    del X
