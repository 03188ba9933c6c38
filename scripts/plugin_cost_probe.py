"""Where the drop-in's per-op host time goes on the box, without a profiler:
cfg2 `tidepool.add(V, R)` back to back through the unmodified reference +
tidepool_plugin, with perf_counter accumulators around the gpu table
entries and the plugin allocator, and with the kernel launch stubbed.
Prints us/op for each piece.  (Diagnostic only; not product code.)"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import bench  # noqa: E402
import ref_loader  # noqa: E402
from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

lib = None
if "--fake" in sys.argv:
    from fake_native import FakeNative
    from oracle import oracle
    lib = FakeNative(oracle.lib())
    lib.tpg_binary = lambda *a: 0
tp = ref_loader.load("tidepool")
gpu = tidepool_plugin.register(tp, count=1, lib=lib)[0]
rt = tidepool_plugin.register.runtime
N = bench.N if lib is None else 64
X = tp.tensor_create((N, N), tp.int16, gpu)
R = tp.tensor_create((1, N), tp.float, gpu)
V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
st = gpu.default_stream()


def wall(n=3000):
    for _ in range(50):
        tp.add(V, R)
    st.sync()
    t0 = time.perf_counter()
    for _ in range(n):
        tp.add(V, R)
    st.sync()
    return 1e6 * (time.perf_counter() - t0) / n


print(f"wall (first 3000 calls)      {wall():7.2f} us/op")
c0 = rt.entries.counts()
n0 = 3000
print(f"wall (steady state)          {wall(n0):7.2f} us/op")
c1 = rt.entries.counts()
for k in ("ns_allocate", "ns_release", "ns_binary", "ns_copy", "ns_launch"):
    print(f"  C {k[3:]:24s} {(c1[k] - c0[k]) / 1e3 / (n0 + 50):7.2f} us/op")
acc = {}


def timed(name, f):
    def g(*a, **k):
        t0 = time.perf_counter_ns()
        try:
            return f(*a, **k)
        finally:
            acc[name] = acc.get(name, 0) + time.perf_counter_ns() - t0
    return g


restores = []
for op in ("add", "copy"):
    restores.append(tp.dispatch.override_op("core", "gpu", op, lambda f, op=op: timed(op, f)))
orig_alloc = rt.allocate
rt.allocate = timed("allocate (+ release inside the C pool)", orig_alloc)
n = 3000
w = wall(n)
print(f"wall (instrumented)          {w:7.2f} us/op")
for k, v in acc.items():
    print(f"  {k:26s} {v / 1e3 / (n + 50):7.2f} us/op")
for r in restores:
    r()
rt.allocate = orig_alloc
L = rt.L
real = L.tpg_binary
L.tpg_binary = lambda *a: 0
print(f"wall, tpg_binary stubbed     {wall():7.2f} us/op")
L.tpg_binary = real
print(f"reference floor              {1e3 * bench._pipeline_floor(2000):7.2f} us/op")

# host cost of the launch itself: tpg_binary through ctypes on a small
# cfg2-shaped problem (same kernel path; the kernel is short so the launch
# queue never fills), next to a bare ctypes call and an event record
import ctypes as C  # noqa: E402
from paper_1810_08723_b200 import abi  # noqa: E402

n = 256
Xs = tp.tensor_create((n, n), tp.int16, gpu)
Rs = tp.tensor_create((1, n), tp.float, gpu)
Os = tp.tensor_create((n, n), tp.float, gpu)
xp, rp, op_ = (rt.address(t.storage.view()) for t in (Xs, Rs, Os))
plan = abi.make_plan([n, n], [[4, 4 * n], [-2 * n, 2], [0, 4]])
d = abi.make_operand(op_, 0, 10, False)
a = abi.make_operand(xp, (n - 1) * 2 * n, 3, False)
b = abi.make_operand(rp, 0, 10, False)
args = (st.handle, 0, C.byref(plan), C.byref(d), C.byref(a), C.byref(b), 10, 0)


def per_call(label, f, k=3000):
    for _ in range(50):
        f()
    st.sync()
    t0 = time.perf_counter()
    for i in range(k):
        f()
        if i % 200 == 199:
            st.sync()
    st.sync()
    print(f"{label:44s} {1e6 * (time.perf_counter() - t0) / k:7.2f} us/call")


per_call("ctypes tpg_binary 256^2 cfg2 shape", lambda: L.tpg_binary(*args))
per_call("ctypes tpg_last_error (bare call)", lambda: L.tpg_last_error())
ev = C.c_void_p()
L.tpg_event_create_untimed(C.byref(ev))
per_call("ctypes tpg_event_record", lambda: L.tpg_event_record(ev, st.handle))
per_call("ctypes tpg_event_query", lambda: L.tpg_event_query(ev))
per_call("ctypes tpg_memset 4 B", lambda: L.tpg_memset(C.c_void_p(op_), 0, 4, st.handle))
print("entries", rt.entries.counts())
