"""cfg2 through the unmodified reference + tidepool_plugin on gpu0: which
kernels run per `tidepool.add(V, R)` and what they cost (run under ncu for
the launch list), plus host wall time per op."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import bench  # noqa: E402
import ref_loader  # noqa: E402
from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

tp = ref_loader.load("tidepool")
gpu = tidepool_plugin.register(tp, count=1)[0]
rt = tidepool_plugin.register.runtime
N = bench.N
x16, r = bench.cfg2_host_inputs()


def put(arr, dt):
    t = tp.tensor_create(arr.shape, dt, gpu)
    t.storage.stream.sync()
    t.storage.view()[:] = arr.tobytes(order="F")
    return t


X, R = put(x16, tp.int16), put(r, tp.float)
V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
st = gpu.default_stream()
outs = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    t0 = time.perf_counter()
    outs.append(tp.add(V, R))
    t1 = time.perf_counter()
    st.sync()
    t2 = time.perf_counter()
    print(f"op {i}: enqueue {1e3 * (t1 - t0):.3f} ms, sync {1e3 * (t2 - t1):.3f} ms", flush=True)
print(dict(rt.stats))
