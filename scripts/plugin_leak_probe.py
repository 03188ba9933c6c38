"""Reference-count / allocation leak probe of the drop-in's C host path
(hostsrc/tpg_pyfast.c) on CPU: the unmodified reference + tidepool_plugin on
the C-ABI test double (or the real library), the cfg2-shaped call (lazy int16 -> float cast fused
into the add), a unary, a reduction and a lazy copy read back, run in
rounds; sys.getallocatedblocks() and the process RSS must not grow with the
number of rounds.  `--gpu`: the same through the real library on gpu0.
(Diagnostic only; not product code.)"""
import gc
import resource
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import ref_loader  # noqa: E402
from fake_native import FakeNative  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

tp = ref_loader.load("tidepool")
GPU = "--gpu" in sys.argv
if GPU:
    sys.argv.remove("--gpu")
fake = None if GPU else FakeNative(oracle.lib())
gpu = tidepool_plugin.register(tp, count=1, lib=fake)[0]
rt = tidepool_plugin.register.runtime
X = tp.cast(tp.from_nested([[i - 8 for i in range(16)] for _ in range(16)], tp.int16), device=gpu)
R = tp.cast(tp.from_nested([[0.5 * i for i in range(16)]], tp.float), device=gpu)
V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
F = tp.cast(tp.from_nested([[float(i) for i in range(16)]], tp.float), device=gpu)


CALLS = {"add_lazy": lambda: tp.add(V, R), "unary": lambda: tp.negate(F),
         "reduce": lambda: tp.reduce("sum", F), "scalar": lambda: tp.multiply(F, 2.0),
         "cast": lambda: tp.cast(V, tp.float), "add": lambda: tp.add(F, F)}
SEL = [CALLS[k] for k in (sys.argv[1:] or CALLS)]


def body():
    for f in SEL:
        f()


def rounds(n):
    for _ in range(n):
        body()
        if fake:
            fake.calls.clear()  # the test double's launch log, not the plugin
    gpu.default_stream().sync()
    gc.collect()
    return sys.getallocatedblocks(), resource.getrusage(resource.RUSAGE_SELF).ru_maxrss


rounds(500)
b0, m0 = rounds(2000)
b1, m1 = rounds(20000)
b2, m2 = rounds(20000)
print(f"allocated blocks after warm-up {b0}, +20k rounds {b1}, +20k more {b2}")
print(f"max RSS KiB {m0} -> {m1} -> {m2}")
print("entries", rt.entries.counts())
ok = abs(b2 - b1) < 200 and m2 - m1 < 8192
print("OK" if ok else "GROWTH")
sys.exit(0 if ok else 1)
