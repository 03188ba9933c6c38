"""Fixed per-step cost of bench.py's event timing: the same timed_steps
(L2 flush between steps, device-side gate) around a 1-element add, the
cfg1 add (2^20 f32) and a 2^22 / 2^24 add, so the small-op numbers can be
read against the floor."""
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
for n in (1, 1 << 20, 1 << 22, 1 << 24):
    rng = np.random.default_rng(1)
    a = tp.from_numpy(rng.standard_normal(n).astype(np.float32), dev)
    b = tp.from_numpy(rng.standard_normal(n).astype(np.float32), dev)
    o = tp.tensor_create((n,), tp.float, dev)
    f = lambda: tp.add(a, b, dest=o)  # noqa: E731
    for _ in range(3):
        f()
    stream.sync()
    ms = statistics.mean(bench.timed_steps(L, stream, f, 20, lambda: bench.l2_flush(L, stream, fb)))
    print(f"add f32 n={n:>9d}  {ms * 1e3:7.2f} us  {12 * n / ms / 1e6:8.1f} GB/s")

# the same 1-element and cfg1 adds without the L2 flush, and with a tiny
# kernel queued between the flush and the start event
tiny_a = tp.from_numpy(np.ones(1, np.float32), dev)
tiny_o = tp.tensor_create((1,), tp.float, dev)
for n in (1, 1 << 20):
    a = tp.from_numpy(np.ones(n, np.float32), dev)
    b = tp.from_numpy(np.ones(n, np.float32), dev)
    o = tp.tensor_create((n,), tp.float, dev)
    f = lambda: tp.add(a, b, dest=o)  # noqa: E731
    ms0 = statistics.mean(bench.timed_steps(L, stream, f, 20, None))
    ms1 = statistics.mean(bench.timed_steps(
        L, stream, f, 20,
        lambda: (bench.l2_flush(L, stream, fb), tp.add(tiny_a, tiny_a, dest=tiny_o))))
    print(f"add f32 n={n:>9d}  no flush {ms0 * 1e3:7.2f} us   flush + tiny kernel {ms1 * 1e3:7.2f} us")
