"""One launch of each hot kernel family at its SURVEY §8d size (for ncu)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_08723_b200 as tp  # noqa: E402

X = tp.from_numpy(np.asfortranarray(np.random.default_rng(5).random((8192, 8192))))
for axes in ((0,), (1,), None):
    tp.reduce("sum", X, axes=axes)
tp.reduce("maximum", X, axes=(1,))
del X
n5 = 1 << 28
Y = tp.from_numpy(np.random.default_rng(8).uniform(-1e3, 1e3, n5).astype(np.float32))
Z = tp.chain(Y, [("multiply", tp.Scalar(1.5, tp.float)), ("add", tp.Scalar(-2.0, tp.float))])
del Y, Z
for dt, npd in ((tp.half, np.float16), (tp.float, np.float32)):
    m = 8192
    A = tp.transpose(tp.from_numpy(np.asfortranarray(
        np.random.default_rng(6).uniform(-1, 1, (m, m)).astype(npd))))
    B = tp.from_numpy(np.asfortranarray(np.random.default_rng(7).uniform(-1, 1, (m, m)).astype(npd)))
    tp.matmul(A, B)
    del A, B
a = tp.from_numpy(np.asfortranarray(np.random.default_rng(6).uniform(-1, 1, (2048, 2048, 64)).astype(np.float16)))
b = tp.from_numpy(np.asfortranarray(np.random.default_rng(7).uniform(-1, 1, (2048, 2048, 64)).astype(np.float16)))
tp.matmul_batched(a, b)
tp.gpu(0).synchronize()
print("hot kernels done")
