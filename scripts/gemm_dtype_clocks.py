"""Why f16 trails bf16 on the same tcgen05 kind::f16 MMA:
8192^3 gemm (the cfg4 layout) run back to back for ~3 s per case with
nvidia-smi sampling SM clock, power and throttle reasons during each case.
Cases: f16 uniform(-1,1); bf16 uniform(-1,1); f16 whose values are exactly
bf16-representable (low 3 mantissa bits zero, same magnitudes); f16 of a
coarser grid (multiples of 1/64)."""
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_08723_b200 as tp  # noqa: E402

dev = tp.list_devices()[0]
m = 8192
rng = np.random.default_rng(6)
base_a = rng.uniform(-1, 1, (m, m)).astype(np.float32)
base_b = rng.uniform(-1, 1, (m, m)).astype(np.float32)


def f16(x):
    return tp.from_numpy(np.asfortranarray(x.astype(np.float16)), dev)


def bf16(x):
    raw = np.asfortranarray((x.view(np.uint32) >> 16).astype(np.uint16))
    return tp.from_numpy(raw, dev, dtype=tp.bfloat16)


def trunc_bf16(x):  # float32 values with the bf16 mantissa (exactly representable in f16 here)
    return ((x.view(np.uint32) >> 16) << 16).view(np.float32)


cases = [("f16 uniform(-1,1)", f16(base_a), f16(base_b), tp.half),
         ("bf16 uniform(-1,1)", bf16(base_a), bf16(base_b), tp.bfloat16),
         ("f16 holding bf16-exact values", f16(trunc_bf16(base_a)), f16(trunc_bf16(base_b)),
          tp.half),
         ("f16 multiples of 1/64", f16(np.round(base_a * 64) / 64), f16(np.round(base_b * 64) / 64),
          tp.half)]

# batched 64 x 2048^3 f16 (cfg4 batched): 4x the output bytes per flop of 8192^3
bb = 64
ba = rng.uniform(-1, 1, (2048, 2048, bb)).astype(np.float16)
bbm = rng.uniform(-1, 1, (2048, 2048, bb)).astype(np.float16)
BA, BB = (tp.from_numpy(np.asfortranarray(x), dev) for x in (ba, bbm))
del ba, bbm

samples = []


def sampler(stop):
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,"
                          "clocks_event_reasons.active", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            samples.append((time.time(), line.strip()))
    p.terminate()


stop = threading.Event()
th = threading.Thread(target=sampler, args=(stop,), daemon=True)
th.start()
time.sleep(0.5)
res = []
for name, A, B, dt in cases:
    At = tp.transpose(A)
    C = tp.tensor_create((m, m), dt, dev)
    for _ in range(3):
        tp.matmul(At, B, dest=C)
    dev.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < 3.0:
        for _ in range(10):
            tp.matmul(At, B, dest=C)
        dev.synchronize()
        n += 10
    t1 = time.time()
    res.append((name, t0, t1, 2 * m ** 3 * n / (t1 - t0) / 1e12))
    time.sleep(0.3)
BC = tp.tensor_create((2048, 2048, bb), tp.half, dev)
for _ in range(3):
    tp.matmul_batched(BA, BB, dest=BC)
dev.synchronize()
t0 = time.time()
n = 0
while time.time() - t0 < 3.0:
    for _ in range(10):
        tp.matmul_batched(BA, BB, dest=BC)
    dev.synchronize()
    n += 10
t1 = time.time()
res.append(("batched f16 64 x 2048^3", t0, t1, 2 * 2048 ** 3 * bb * n / (t1 - t0) / 1e12))
stop.set()
th.join(timeout=2)
for name, t0, t1, tf in res:
    win = [s for t, s in samples if t0 + 0.5 <= t <= t1]
    clk = [float(s.split(",")[0]) for s in win]
    pw = [float(s.split(",")[1]) for s in win]
    reasons = sorted({s.split(",")[2].strip() for s in win})
    print(f"{name:34s} {tf:7.1f} TFLOP/s  sm clock median {np.median(clk):6.0f} MHz  "
          f"power median {np.median(pw):6.1f} W  reasons {reasons}  ({len(win)} samples)",
          flush=True)
