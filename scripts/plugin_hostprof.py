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
pstats.Stats("/tmp/hp").sort_stats("tottime").print_stats(40)

# raw per-call costs of the C-ABI calls one plugin op makes
import ctypes as C  # noqa: E402
rt = tidepool_plugin.register.runtime
L = rt.L


def per_call(label, f, n=20000):
    f()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    print(f"{label:40s} {1e6 * (time.perf_counter() - t0) / n:7.2f} us")


ev = rt._new_event()
L.tpg_event_record(ev, st.handle)
st.sync()
per_call("tpg_event_query (completed)", lambda: L.tpg_event_query(ev))
per_call("tpg_event_record", lambda: L.tpg_event_record(ev, st.handle))
st.sync()
f = C.c_uint32(0)
per_call("tpg_flags_take", lambda: L.tpg_flags_take(st.handle, C.byref(f)), 2000)
per_call("rt.allocate+release 64 MiB class", lambda: rt.allocate(0, N * N * 4), 5000)
per_call("ctypes no-arg call (tpg_last_error)", lambda: L.tpg_last_error())
per_call("tp.tensor_create 4096^2 f32", lambda: tp.tensor_create((N, N), tp.float, gpu), 5000)
st.sync()
