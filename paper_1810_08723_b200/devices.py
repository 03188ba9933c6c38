"""The gpu device type, device instances and CUDA streams.

Mirrors the reference DeviceType / Device / Stream objects
(pkg/src/tidepool/devices.py:29-192): a device owns a default stream and
allocates raw buffers; a stream is a FIFO execution context.  Here a
stream is a CUDA stream: `submit` runs the (already asynchronous) launch
closure inline and `sync` waits on the CUDA stream, re-raising the first
failure captured since the last sync (devices.py:74-98 semantics).
Buffers come from the library's stream-ordered caching allocator; frees
are deferred past the owning stream (see csrc/tpg_runtime.cu).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _native, abi
from .errors import DeviceError

ENV_GPU_DEVICES = "TIDEPOOL_GPU_DEVICES"


class DeviceType:
    __slots__ = ("name", "supports_byteswapped", "async_capable")

    def __init__(self, name, *, supports_byteswapped, async_capable):
        self.name = name
        self.supports_byteswapped = supports_byteswapped
        self.async_capable = async_capable

    def __repr__(self):
        return f"<device type {self.name}>"


GPU_TYPE = DeviceType("gpu", supports_byteswapped=True, async_capable=True)


class GpuStream:
    def __init__(self, device, handle, owned):
        self.device = device
        self.handle = handle
        self._owned = owned
        self._pending: BaseException | None = None

    def submit(self, task) -> None:
        # launches are asynchronous on the CUDA stream; host-side failures
        # (argument errors, error-mode checks) raise here, synchronously
        task()

    def sync(self) -> None:
        _native.check(_native.lib().tpg_stream_sync(self.handle), "stream sync")
        if self._pending is not None:
            exc, self._pending = self._pending, None
            raise exc

    def wait_for(self, other: "GpuStream") -> None:
        """Order this stream after everything submitted to `other`."""
        _native.check(_native.lib().tpg_stream_wait(self.handle, other.handle), "stream wait")

    def __del__(self):
        try:
            if self._owned and _native._lib is not None:
                _native._lib.tpg_stream_destroy(self.handle)
        except Exception:
            pass

    def __repr__(self):
        return f"<stream on {self.device.name}>"


class GpuDevice:
    def __init__(self, index: int):
        self.type = GPU_TYPE
        self.index = index
        self.alloc_count = 0
        self._stream = None
        self._lock = threading.Lock()

    @property
    def name(self) -> str:
        return f"gpu{self.index}"

    @property
    def is_host(self) -> bool:
        return False

    @property
    def properties(self) -> dict:
        p = abi.DeviceProps()
        _native.check(_native.lib().tpg_device_props_get(self.index, C.byref(p)), "props")
        return {"device-type": "gpu", "supports-byteswapped": "true",
                "name": p.name.decode(), "processor-count": str(p.sm_count),
                "compute-capability": f"{p.cc_major}.{p.cc_minor}",
                "free-memory": str(p.free_mem), "total-memory": str(p.total_mem),
                "l2-bytes": str(p.l2_bytes)}

    def default_stream(self) -> GpuStream:
        with self._lock:
            if self._stream is None:
                h = C.c_void_p()
                _native.check(_native.lib().tpg_default_stream(self.index, C.byref(h)), "stream")
                self._stream = GpuStream(self, h.value, False)
            return self._stream

    def create_stream(self) -> GpuStream:
        h = C.c_void_p()
        _native.check(_native.lib().tpg_stream_create(self.index, C.byref(h)), "stream create")
        return GpuStream(self, h.value, True)

    def allocate(self, nbytes: int) -> int:
        ptr = C.c_void_p()
        _native.check(_native.lib().tpg_malloc(self.index, max(int(nbytes), 1), C.byref(ptr)),
                      f"{self.name}: allocate {nbytes} bytes")
        self.alloc_count += 1
        return ptr.value

    def release(self, ptr: int, stream: GpuStream | None) -> None:
        if _native._lib is None or ptr is None:
            return
        _native._lib.tpg_free(self.index, ptr, stream.handle if stream else None)

    def mem_stats(self) -> dict:
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _native.check(_native.lib().tpg_mem_stats(self.index, C.byref(a), C.byref(b), C.byref(c)))
        return {"in-use": a.value, "cached": b.value}

    def synchronize(self) -> None:
        self.default_stream().sync()

    def __repr__(self):
        return f"<device {self.name}>"


_devices: list[GpuDevice] = []


def configure(count: int | None = None) -> None:
    """(Re)build the gpu device list (cap with TIDEPOOL_GPU_DEVICES)."""
    n = _native.device_count()
    cap = os.environ.get(ENV_GPU_DEVICES)
    if count is None and cap is not None:
        count = int(cap)
    if count is not None:
        n = min(n, count)
    _devices.clear()
    _devices.extend(GpuDevice(i) for i in range(n))
    if n > 1:  # cross-device transfers and peer reads go over NVLink directly
        import ctypes as C
        import warnings
        try:
            _native.check(_native.lib().tpg_enable_peer_all(C.byref(C.c_int(0))), "peer access")
        except DeviceError as exc:  # copies still work through the host path
            warnings.warn(f"peer access not enabled: {exc}")


def list_devices() -> list:
    if not _devices:
        configure()
    return list(_devices)


def gpu(index: int = 0) -> GpuDevice:
    devs = list_devices()
    for d in devs:
        if d.index == index:
            return d
    raise DeviceError(f"no gpu device with index {index} ({len(devs)} visible)")


def by_name(name: str) -> GpuDevice:
    for d in list_devices():
        if d.name == name:
            return d
    raise DeviceError(f"unknown device {name!r}")
