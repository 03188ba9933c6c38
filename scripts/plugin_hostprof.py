"""Where the host time of one cfg2 call through the unmodified reference +
tidepool_plugin goes (cProfile over back-to-back calls on gpu0), next to
the reference pipeline's own floor with a no-op table."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import bench  # noqa: E402
import ref_loader  # noqa: E402
from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

tp = ref_loader.load("tidepool")
gpu = tidepool_plugin.register(tp, count=1)[0]
N = bench.N
X = tp.tensor_create((N, N), tp.int16, gpu)
R = tp.tensor_create((1, N), tp.float, gpu)
V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
st = gpu.default_stream()
for _ in range(50):
    tp.add(V, R)
st.sync()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    tp.add(V, R)
st.sync()
print(f"plugin wall {1e6 * (time.perf_counter() - t0) / n:.1f} us/op")
print(f"reference floor {1e3 * bench._pipeline_floor(2000):.1f} us/op")
cProfile.run("for _ in range(2000): tp.add(V, R)", "/tmp/hp")
pstats.Stats("/tmp/hp").sort_stats("tottime").print_stats(25)
