"""A/B of operand layouts for the tcgen05 gemm: A K-major (transposed view)
vs A MN-major (column-major) at cfg4's square and batched shapes.
Device ms per call (bench.timed_steps, no flush: inputs >> L2 reuse is
inside the kernel)."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1810_08723_b200 as tp  # noqa: E402
from paper_1810_08723_b200 import _native  # noqa: E402
from paper_1810_08723_b200 import tensors as tz  # noqa: E402

L = _native.lib()
dev = tp.list_devices()[0]
stream = dev.default_stream()
rng = np.random.default_rng(6)


def f16(shape):
    return tp.from_numpy(np.asfortranarray(rng.uniform(-1, 1, shape).astype(np.float16)), dev)


def run(name, f, flops):
    for _ in range(3):
        f()
    stream.sync()
    ms = statistics.mean(bench.timed_steps(L, stream, f, 5, None))
    print(f"{name:44s} {ms:8.4f} ms {flops / ms / 1e9:8.1f} TFLOP/s", flush=True)


m = 8192
B = f16((m, m))
C = tp.tensor_create((m, m), tp.half, dev)
Ak = tp.transpose(f16((m, m)))
run("8192^3 A K-major", lambda: tp.matmul(Ak, B, dest=C), 2 * m ** 3)
del Ak
Am = f16((m, m))
run("8192^3 A MN-major", lambda: tp.matmul(Am, B, dest=C), 2 * m ** 3)
del Am, B, C
n, nb = 2048, 64
Bb = f16((n, n, nb))
Cb = tp.tensor_create((n, n, nb), tp.half, dev)
Am = f16((n, n, nb))
run("batched 64x2048^3 A MN-major", lambda: tp.matmul_batched(Am, Bb, dest=Cb), 2 * nb * n ** 3)
del Am
Ak = tz.permute_axes(f16((n, n, nb)), (1, 0, 2))
run("batched 64x2048^3 A K-major", lambda: tp.matmul_batched(Ak, Bb, dest=Cb), 2 * nb * n ** 3)
Bm = tz.permute_axes(f16((n, n, nb)), (1, 0, 2))
run("batched 64x2048^3 A K-major B MN-major", lambda: tp.matmul_batched(Ak, Bm, dest=Cb), 2 * nb * n ** 3)
# row-major destination (epilogue writes each thread's 32 contiguous values)
Cr = tz.permute_axes(tp.tensor_create((n, n, nb), tp.half, dev), (1, 0, 2))
run("batched 64x2048^3 A K-major, row-major C", lambda: tp.matmul_batched(Ak, Bb, dest=Cr),
    2 * nb * n ** 3)
m = 8192
del Ak, Bb, Cb, Bm, Cr
Ak = tp.transpose(f16((m, m)))
B = f16((m, m))
Cr = tp.transpose(tp.tensor_create((m, m), tp.half, dev))
run("8192^3 A K-major, row-major C", lambda: tp.matmul(Ak, B, dest=Cr), 2 * m ** 3)
