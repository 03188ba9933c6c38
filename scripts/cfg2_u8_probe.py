"""The cfg2 shape with 8-bit data: uint8[4096,4096] transposed reversed view
+ float32 row -> float32, through the C ABI, steady state (4 rotating
buffer sets > L2, K launches per event pair), value-checked.  Run with and
without TPG_TILE_TMA=0 for the A/B of the 1-byte TMA tile path."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
import bench  # noqa: E402
from paper_1810_08723_b200 import _native, abi  # noqa: E402

N, ROT, K = 4096, 4, 40
L = _native.lib()
sh = C.c_void_p()
L.tpg_default_stream(0, C.byref(sh))
st = bench._S(L, sh.value)
rng = np.random.default_rng(5)
x8 = np.asfortranarray(rng.integers(0, 256, (N, N)).astype(np.uint8))
r = np.asfortranarray(rng.standard_normal((1, N)).astype(np.float32))
R = bench._dmalloc(L, N * 4)
L.tpg_memcpy_h2d(R, r.ctypes.data, r.nbytes, st.handle)
sets = []
for _ in range(ROT):
    X, O = bench._dmalloc(L, N * N), bench._dmalloc(L, N * N * 4)
    L.tpg_memcpy_h2d(X, x8.ctypes.data, x8.nbytes, st.handle)
    plan = abi.make_plan([N, N], [[4, 4 * N], [-N, 1], [0, 4]])
    d = abi.make_operand(O, 0, 10, False)
    a = abi.make_operand(X, (N - 1) * N, 2, False)   # uint8 wire code 2
    b = abi.make_operand(R, 0, 10, False)
    sets.append((X, O, (st.handle, 0, C.byref(plan), C.byref(d), C.byref(a), C.byref(b), 10, 0),
                 (plan, d, a, b)))
k = [0]


def step():
    rc = L.tpg_binary(*sets[k[0] % ROT][2])
    assert rc == 0, L.tpg_last_error()
    k[0] += 1


for _ in range(8):
    step()
st.sync()
ms = min(bench.timed_batch(L, st, step, K)[0] for _ in range(5))
nbytes = N * N * 5 + N * 4
got = np.empty((N, N), np.float32, order="F")
L.tpg_memcpy_d2h(got.ctypes.data, sets[1][1], got.nbytes, st.handle)
st.sync()
want = (x8.T[::-1, :].astype(np.float64) + r.astype(np.float64)).astype(np.float32)
assert np.array_equal(got, want), "mismatch"
print(f"uint8 cfg2 shape: {1e3 * ms:.2f} us/launch, {nbytes / ms / 1e6:.1f} GB/s (bit-exact)")
