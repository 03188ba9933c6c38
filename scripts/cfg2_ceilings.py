"""Steady-state (back-to-back, rotating buffers > L2) ceilings for the cfg2
byte mix on one B200, next to the product kernel, all through the C ABI:

  * the headline tpg_binary (k_tile_f32: transposing int16 -> f32 + row),
  * the same byte mix without the transpose (contiguous int16 -> f32 cast,
    k_contig): 2 B read + 4 B written per element,
  * a 1:1 device copy of the same total bytes (cudaMemcpyAsync D2D),
  * a pure 64 MiB write (cudaMemsetAsync).

Each row: ROT sets rotated, K launches between one event pair, best of 5.
"""
import ctypes as C
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1810_08723_b200 import _native, abi  # noqa: E402

L = _native.lib()
N = bench.N
ROT, K = 4, 40
sh = C.c_void_p()
L.tpg_default_stream(0, C.byref(sh))
st = bench._S(L, sh.value)
x16, r = bench.cfg2_host_inputs()
R = bench._dmalloc(L, N * 4)
L.tpg_memcpy_h2d(R, r.ctypes.data, r.nbytes, st.handle)
Xs = [bench._dmalloc(L, N * N * 2) for _ in range(ROT)]
Os = [bench._dmalloc(L, N * N * 4) for _ in range(ROT)]
for x in Xs:
    L.tpg_memcpy_h2d(x, x16.ctypes.data, x16.nbytes, st.handle)
st.sync()


def measure(name, launches, nbytes, gate=True):
    k = [0]

    def step():
        launches[k[0] % len(launches)]()
        k[0] += 1
    for _ in range(8):
        step()
    st.sync()
    best = min(bench.timed_batch(L, st, step, K, gate)[0] for _ in range(5))
    name += "" if gate else " [no gate]"
    print(f"{name:58s} {best * 1e3:8.2f} us  {nbytes / best / 1e6:8.1f} GB/s  "
          f"({nbytes / 1e6:.1f} MB)", flush=True)
    return best


rows = []
descs = [bench.cfg2_plan(abi, Xs[i], R, Os[i]) for i in range(ROT)]
heads = [(lambda d=d: L.tpg_binary(st.handle, 0, C.byref(d[0]), C.byref(d[1]), C.byref(d[2]),
                                   C.byref(d[3]), 10, 0)) for d in descs]
measure("headline tpg_binary cfg2 (k_tile_f32)", heads, bench.CFG2_BYTES)
measure("headline tpg_binary cfg2 (k_tile_f32)", heads, bench.CFG2_BYTES, gate=False)
cplan = abi.make_plan([N * N], [[4], [2]])
conv = []
for i in range(ROT):
    d = abi.make_operand(Os[i], 0, 10, False)
    a = abi.make_operand(Xs[i], 0, 3, False)
    conv.append(lambda d=d, a=a: L.tpg_unary(st.handle, 10, C.byref(cplan), C.byref(d),
                                             C.byref(a), 3, 0, 0))
measure("contiguous int16 -> f32 cast, same bytes (k_contig)", conv, N * N * 6)
measure("contiguous int16 -> f32 cast, same bytes (k_contig)", conv, N * N * 6, gate=False)
half = N * N * 3
cps = [(lambda i=i: L.tpg_memcpy_d2d(Os[i], Os[(i + 2) % ROT], half, st.handle))
       for i in range(ROT)]
measure("D2D memcpy 50.3 MB -> 50.3 MB", cps, 2 * half)
ms = [(lambda i=i: L.tpg_memset(Os[i], i, N * N * 4, st.handle)) for i in range(ROT)]
measure("memset 67.1 MB", ms, N * N * 4)
big = [bench._dmalloc(L, 1 << 30) for _ in range(2)]
measure("D2D memcpy 1 GiB -> 1 GiB (STREAM-style peak)",
        [lambda: L.tpg_memcpy_d2d(big[0], big[1], 1 << 30, st.handle),
         lambda: L.tpg_memcpy_d2d(big[1], big[0], 1 << 30, st.handle)], 2 << 30)
