"""Device time of the cfg2 kernel (tpg_binary) on buffers from different
allocators: cudaMalloc (the product's own storage), CUDA managed memory
with and without placement advice, after a host write of the inputs (the
drop-in plugin's storage path).  Back-to-back launches, one event pair."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1810_08723_b200 import _native, abi  # noqa: E402

L = _native.lib()
rt = C.CDLL("libcudart.so.12")
N = bench.N
sh = C.c_void_p()
L.tpg_default_stream(0, C.byref(sh))
st = bench._S(L, sh.value)
x16, r = bench.cfg2_host_inputs()


class Loc(C.Structure):
    _fields_ = [("type", C.c_int), ("id", C.c_int)]


def managed(n, prefer=False, accessed=False, prefetch=False):
    p = C.c_void_p()
    assert rt.cudaMallocManaged(C.byref(p), C.c_size_t(n), 1) == 0
    if prefer:
        rt.cudaMemAdvise_v2(p, C.c_size_t(n), 3, Loc(1, 0))
    if accessed:
        rt.cudaMemAdvise_v2(p, C.c_size_t(n), 5, Loc(2, 0))
    return p.value


def run(name, alloc, prefetch=False, host_write=True):
    X, R, O = alloc(N * N * 2), alloc(N * 4), alloc(N * N * 4)
    if host_write:
        C.memmove(X, x16.ctypes.data, x16.nbytes)
        C.memmove(R, r.ctypes.data, r.nbytes)
    else:
        L.tpg_memcpy_h2d(X, x16.ctypes.data, x16.nbytes, st.handle)
        L.tpg_memcpy_h2d(R, r.ctypes.data, r.nbytes, st.handle)
    if prefetch:
        for p_, n in ((X, N * N * 2), (R, N * 4), (O, N * N * 4)):
            rt.cudaMemPrefetchAsync_v2(C.c_void_p(p_), C.c_size_t(n), Loc(1, 0), 0,
                                       C.c_void_p(st.handle and None))
        rt.cudaDeviceSynchronize()
    d = bench.cfg2_plan(abi, X, R, O)
    step = lambda: L.tpg_binary(st.handle, 0, C.byref(d[0]), C.byref(d[1]), C.byref(d[2]),  # noqa
                                C.byref(d[3]), 10, 0)
    for _ in range(5):
        step()
    st.sync()
    best = min(bench.timed_batch(L, st, step, 20)[0] for _ in range(3))
    print(f"{name:60s} {best * 1e3:8.2f} us  {bench.CFG2_BYTES / best / 1e6:8.1f} GB/s", flush=True)


def dmalloc(n):
    return bench._dmalloc(L, n)


run("cudaMallocAsync (product storage)", dmalloc, host_write=False)
run("managed, no advice, host-written inputs", lambda n: managed(n))
run("managed, no advice, host-written, prefetched", lambda n: managed(n), prefetch=True)
run("managed, preferred=GPU", lambda n: managed(n, prefer=True))
run("managed, preferred=GPU + prefetch", lambda n: managed(n, prefer=True), prefetch=True)
run("managed, preferred=GPU + accessedBy host", lambda n: managed(n, True, True))
run("managed, preferred=GPU + accessedBy host + prefetch", lambda n: managed(n, True, True),
    prefetch=True)
run("managed, H2D-copied inputs (no host touch)", lambda n: managed(n), host_write=False)
pl = C.c_void_p()
L.tpg_malloc_managed(0, 64, C.byref(pl))
run("tpg_malloc_managed (plugin path), host-written",
    lambda n: (L.tpg_malloc_managed(0, n, C.byref(pl)), pl.value)[1])
