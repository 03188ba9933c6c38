"""cfg3 reductions timed back to back (537 MB input > L2, K launches per
event pair) with whichever libtidepool_gpu.so $TIDEPOOL_GPU_LIB selects:
A/B of reduction-kernel build variants (scripts/_variants/*)."""
import os
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
st = dev.default_stream()
xn = np.asfortranarray(np.random.default_rng(5).random((8192, 8192)))
X = tp.from_numpy(xn, dev)
tag = os.environ.get("TIDEPOOL_GPU_LIB", "product")
for op in ("sum", "maximum", "norm"):
    for axes, name in (((0,), "axis0"), ((1,), "axis1"), (None, "full")):
        f = lambda: tp.reduce(op, X, axes=axes)  # noqa: E731
        for _ in range(3):
            f()
        st.sync()
        ms = min(bench.timed_batch(L, st, f, 20)[0] for _ in range(3))
        print(f"{tag[-40:]:40s} {op:8s} {name:6s} {ms * 1e3:7.2f} us "
              f"{xn.nbytes / ms / 1e6:8.1f} GB/s", flush=True)
