"""Host<->device transfer of a 67 MB pageable host buffer (a reference cpu
tensor's bytearray) three ways: plain cudaMemcpy from/to pageable memory,
cudaHostRegister-in-place + DMA, and a pinned staging buffer + host memcpy."""
import ctypes as C
import time

import numpy as np

rt = C.CDLL("libcudart.so.12")
n = 4096 * 4096 * 4
dev = C.c_void_p()
assert rt.cudaMalloc(C.byref(dev), C.c_size_t(n)) == 0
pin = C.c_void_p()
assert rt.cudaHostAlloc(C.byref(pin), C.c_size_t(n), 0) == 0


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        rt.cudaDeviceSynchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


for direction, kind in (("D2H", 2), ("H2D", 1)):
    host = bytearray(n)
    hp = C.addressof(C.c_char.from_buffer(host))

    def plain():
        if kind == 2:
            rt.cudaMemcpy(C.c_void_p(hp), dev, C.c_size_t(n), kind)
        else:
            rt.cudaMemcpy(dev, C.c_void_p(hp), C.c_size_t(n), kind)

    def registered():
        lo = hp & ~4095
        size = ((hp + n + 4095) & ~4095) - lo
        assert rt.cudaHostRegister(C.c_void_p(lo), C.c_size_t(size), 0) == 0
        plain()
        rt.cudaHostUnregister(C.c_void_p(lo))

    def staged():
        if kind == 2:
            rt.cudaMemcpy(pin, dev, C.c_size_t(n), kind)
            C.memmove(hp, pin, n)
        else:
            C.memmove(pin, hp, n)
            rt.cudaMemcpy(dev, pin, C.c_size_t(n), kind)

    def staged_np():
        src = np.frombuffer((C.c_ubyte * n).from_address(pin.value), dtype=np.uint8)
        dst = np.frombuffer(host, dtype=np.uint8)
        if kind == 2:
            rt.cudaMemcpy(pin, dev, C.c_size_t(n), kind)
            np.copyto(dst, src)
        else:
            np.copyto(src, dst)
            rt.cudaMemcpy(dev, pin, C.c_size_t(n), kind)

    def alloc_only():
        bytearray(n)

    for name, f in (("pageable cudaMemcpy", plain), ("register in place + DMA", registered),
                    ("pinned staging + memmove", staged), ("pinned staging + numpy copy", staged_np),
                    ("bytearray(67 MB) allocation", alloc_only)):
        ms = t(f)
        print(f"{direction} {name:32s} {ms:8.2f} ms  {n / ms / 1e6:7.2f} GB/s", flush=True)
