"""cfg4 gemm timings (back to back, 10 launches per event pair, best of 3)
with whichever libtidepool_gpu.so $TIDEPOOL_GPU_LIB selects (A/B of gemm
build variants under scripts/_variants)."""
import os
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
tag = os.environ.get("TIDEPOOL_GPU_LIB", "product")[-34:]
rng = np.random.default_rng(6)
m = 8192
for name, dt in (("f16", np.float16),):
    A = tp.transpose(tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (m, m)).astype(dt)), dev))
    B = tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (m, m)).astype(dt)), dev)
    Cm = tp.tensor_create((m, m), tp.half, dev)
    f = lambda: tp.matmul(A, B, dest=Cm)  # noqa: E731
    for _ in range(3):
        f()
    st.sync()
    ms = min(bench.timed_batch(L, st, f, 10)[0] for _ in range(3))
    print(f"{tag:34s} {name} 8192^3   {ms * 1e3:8.1f} us {2 * m ** 3 / ms / 1e9:8.1f} TFLOP/s",
          flush=True)
    del A, B, Cm
nb, s_ = 64, 2048
Ab = tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (s_, s_, nb)).astype(np.float16)), dev)
Bb = tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (s_, s_, nb)).astype(np.float16)), dev)
Cb = tp.tensor_create((s_, s_, nb), tp.half, dev)
f = lambda: tp.matmul_batched(Ab, Bb, dest=Cb)  # noqa: E731
for _ in range(3):
    f()
st.sync()
ms = min(bench.timed_batch(L, st, f, 10)[0] for _ in range(3))
print(f"{tag:34s} batched 64x2048^3 {ms * 1e3:8.1f} us {nb * 2 * s_ ** 3 / ms / 1e9:8.1f} TFLOP/s",
      flush=True)
