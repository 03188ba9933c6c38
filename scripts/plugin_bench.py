"""Wall-clock of the cfg2 op through the UNMODIFIED reference pipeline with
the gpu table plugged in (tidepool_plugin), vs the same op on this
package's own pipeline.  Needs baseline/_ref (pip install of the reference)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import tidepool  # noqa: E402

from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

tidepool_plugin.register(tidepool, count=1)
gpu = tidepool.devices.by_name("gpu0")
N = 4096
x16 = np.asfortranarray(np.random.default_rng(3).integers(-1000, 1000, (N, N)).astype(np.int16))
r = np.asfortranarray(np.random.default_rng(4).standard_normal((1, N)).astype(np.float32))
X = tidepool.tensor_create((N, N), tidepool.int16, gpu)
np.frombuffer(X.storage.view(), np.uint8)[:] = x16.ravel(order="F").view(np.uint8)
R = tidepool.tensor_create((1, N), tidepool.float, gpu)
np.frombuffer(R.storage.view(), np.uint8)[:] = r.ravel(order="F").view(np.uint8)
V = tidepool.apply_index(tidepool.transpose(X), (slice(None, None, -1), slice(None)))
out = tidepool.tensor_create((N, N), tidepool.float, gpu)
for _ in range(3):
    tidepool.add(V, R, dest=out)
t0 = time.perf_counter()
K = 20
for _ in range(K):
    tidepool.add(V, R, dest=out)
dt = (time.perf_counter() - t0) / K
stats = tidepool.dispatch.table_stats("core", "gpu")
print(f"reference pipeline + gpu table: {dt * 1e3:.3f} ms per add(V, R) "
      f"({N * N * 6 / dt / 1e9:.1f} GB/s algorithmic); table calls {stats.get('add')} add, "
      f"{stats.get('copy')} copy")
