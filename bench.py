#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 gpu module.

Workload (BASELINE.json configs[1], "cfg2"): int16 [4096,4096] viewed
transposed with a reversed axis (strides (-8192, 2)) plus a float32 [1,4096]
row broadcast, `add(V, R)` -> float32 [4096,4096].  One step = one pass of
the hot path over that batch; algorithmic bytes = 2 (int16 read) + 4 (f32
write) per element + the 16 KiB row = 100,679,680 B.  The gpu module fuses
the int16->float32 conversion into the add (one kernel).  L2 is flushed
(256 MiB memset) between timed steps.

`--impl reference` times the reference CPU implementation of the same
path (the C restatement in oracle/, all host threads) on a bounded sample.

Prints ONE JSON line.  Multi-GPU: run under torchrun; every rank runs its
own cfg2 instance (weak scaling), times are max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "elementwise/reduce HBM GB/s vs ~8 TB/s; gemm TFLOP/s; at 1/2/4/8 B200"
N = 4096
CFG2_BYTES = N * N * (2 + 4) + N * 4
FLUSH_BYTES = 256 << 20
E2E_CHUNKS = int(os.environ.get("TPG_E2E_CHUNKS", "8"))  # slabs of the pipelined e2e step
E2E_SPLIT = os.environ.get("TPG_E2E_SPLIT", "cols")  # "rows" | "cols" of the cfg2 result


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed gloo: barrier + max over ranks)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.phys = self._pin_device()
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def _pin_device(self) -> int:
        """One GPU per process: under torchrun each rank sees only GPU
        LOCAL_RANK (mod the GPUs present), so the library initialises one
        device context per process.  Returns the physical index."""
        if self.world == 1 or "CUDA_VISIBLE_DEVICES" in os.environ:
            return 0 if self.world == 1 else self.local
        try:
            out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True,
                                 timeout=30).stdout
            n = len([ln for ln in out.splitlines() if ln.startswith("GPU ")])
        except (OSError, subprocess.TimeoutExpired):
            return self.local
        if n > 0:
            os.environ["CUDA_VISIBLE_DEVICES"] = str(self.local % n)
            return self.local % n
        return self.local

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampled while the benchmark runs
# ---------------------------------------------------------------------------
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x2: "applications_clocks_setting"}


class Clocks:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 4:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), float(parts[2]),
                                         int(parts[3], 16)))
                except ValueError:
                    pass

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        load = [s for s in self.samples if s[2] > 0] or self.samples
        if not load:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set()
        for s in load:
            for bit, name in REASONS.items():
                if s[3] & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in load),
                "sm_max_mhz": max(s[1] for s in load), "reasons": sorted(reasons),
                "samples": len(load)}


# ---------------------------------------------------------------------------
# timing helpers over the C ABI
# ---------------------------------------------------------------------------
class Timer:
    def __init__(self, L, stream):
        self.L, self.stream = L, stream

    def event(self):
        e = C.c_void_p()
        self.L.tpg_event_create(C.byref(e))
        return e.value

    def elapsed(self, a, b):
        ms = C.c_float()
        self.L.tpg_event_elapsed(a, b, C.byref(ms))
        return ms.value


def timed_steps(L, stream, step, steps, flush=None, gate=True):
    """Run `steps` steps with events around each; optional L2 flush before
    each step (outside the events).  Returns per-step device ms."""
    from paper_1810_08723_b200 import _native
    t = Timer(L, stream.handle)
    evs = [(t.event(), t.event()) for _ in range(steps)]
    # under a profiler every launch is serialised, so a gate would only spin
    gate = gate and "CUDA_INJECTION64_PATH" not in os.environ
    if gate:
        _native.check(L.tpg_gate_arm(stream.handle))
    for s, e in evs:
        if flush:
            flush()
        L.tpg_event_record(s, stream.handle)
        step()
        L.tpg_event_record(e, stream.handle)
    if gate:
        L.tpg_gate_release()
    stream.sync()
    out = [t.elapsed(s, e) for s, e in evs]
    for s, e in evs:
        L.tpg_event_destroy(s)
        L.tpg_event_destroy(e)
    return out


# ---------------------------------------------------------------------------
# L2 flush between timed steps (outside the events): write a 256 MiB buffer
# (> 126 MB L2), then read it back with default-priority loads so the L2 is
# left full of clean unrelated lines (tpg_l2_flush) -- no dirty write-backs
# of the flush land inside the next step.
# ---------------------------------------------------------------------------
def l2_flush(L, stream, flush_buf):
    L.tpg_l2_flush(flush_buf, FLUSH_BYTES, stream.handle)


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def cfg2_inputs(tp, dev):
    rng3, rng4 = np.random.default_rng(3), np.random.default_rng(4)
    x16 = np.asfortranarray(rng3.integers(-1000, 1000, (N, N), endpoint=True).astype(np.int16))
    r = np.asfortranarray(rng4.standard_normal((1, N)).astype(np.float32))
    X = tp.from_numpy(x16, dev)
    R = tp.from_numpy(r, dev)
    V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
    assert V.strides == (-8192, 2), V.strides
    return x16, r, X, R, V


def bench_cfg2(tp, dev, steps, warmup, L):
    x16, r, X, R, V = cfg2_inputs(tp, dev)
    out = tp.tensor_create((N, N), tp.float, dev)
    stream = dev.default_stream()
    flush_buf = dev.allocate(FLUSH_BYTES)

    def flush():
        l2_flush(L, stream, flush_buf)

    def step():
        tp.add(V, R, dest=out)

    for _ in range(warmup):
        flush()
        step()
    stream.sync()
    ms = timed_steps(L, stream, step, steps, flush)
    # end to end through the public API with host buffers: every step
    # uploads its inputs from pinned host memory, runs the op and downloads
    # the result (tp.pinned / tp.upload / tp.download / tp.use_stream),
    # pipelined over E2E_CHUNKS slabs on three streams -- one per copy
    # engine direction plus one for the kernels -- chained by per-slab
    # waits: uploads run back to back on the H2D engine, downloads back to
    # back on the D2H engine (PCIe is full duplex), so the step costs about
    # one slab upload + the whole download (E2E_SPLIT picks the slab shape).
    hx = tp.pinned((N, N), np.int16)
    hx[...] = x16
    hr = tp.pinned((1, N), np.float32)
    hr[...] = r
    ho = tp.pinned((N, N), np.float32)
    up, comp, down = dev.create_stream(), dev.create_stream(), dev.create_stream()
    rows = N // E2E_CHUNKS
    if E2E_SPLIT == "rows":
        # V's rows [r0, r1) = X16's columns [N-r1, N-r0): contiguous upload,
        # pitched download
        vch = [tp.apply_index(V, (slice(i * rows, (i + 1) * rows), slice(None)))
               for i in range(E2E_CHUNKS)]
        och = [tp.apply_index(out, (slice(i * rows, (i + 1) * rows), slice(None)))
               for i in range(E2E_CHUNKS)]
        xch = [tp.apply_index(X, (slice(None), slice(N - (i + 1) * rows, N - i * rows)))
               for i in range(E2E_CHUNKS)]
        hxs = [hx[:, N - (i + 1) * rows:N - i * rows] for i in range(E2E_CHUNKS)]
        hos = [ho[i * rows:(i + 1) * rows, :] for i in range(E2E_CHUNKS)]
        rch = [R] * E2E_CHUNKS
    else:
        # V's columns [c0, c1) = X16's rows [c0, c1): pitched upload,
        # contiguous download (the larger direction)
        vch = [tp.apply_index(V, (slice(None), slice(i * rows, (i + 1) * rows)))
               for i in range(E2E_CHUNKS)]
        och = [tp.apply_index(out, (slice(None), slice(i * rows, (i + 1) * rows)))
               for i in range(E2E_CHUNKS)]
        xch = [tp.apply_index(X, (slice(i * rows, (i + 1) * rows), slice(None)))
               for i in range(E2E_CHUNKS)]
        hxs = [hx[i * rows:(i + 1) * rows, :] for i in range(E2E_CHUNKS)]
        hos = [ho[:, i * rows:(i + 1) * rows] for i in range(E2E_CHUNKS)]
        rch = [tp.apply_index(R, (slice(None), slice(i * rows, (i + 1) * rows)))
               for i in range(E2E_CHUNKS)]

    def e2e_step():
        up.wait_for(stream)
        tp.upload(hr, R, up)
        for i in range(E2E_CHUNKS):
            tp.upload(hxs[i], xch[i], up)
            comp.wait_for(up)
            with tp.use_stream(comp):
                tp.add(vch[i], rch[i], dest=och[i])
            down.wait_for(comp)
            tp.download(och[i], hos[i], down)
        stream.wait_for(down)

    for _ in range(2):
        e2e_step()
    stream.sync()
    e2e_steps = max(3, steps // 4)
    t0 = time.perf_counter()
    e2e_ms = timed_steps(L, stream, e2e_step, e2e_steps, None, gate=False)
    wall = (time.perf_counter() - t0) * 1e3 / e2e_steps
    # correctness spot check against the host result of the same bytes
    want = (x16.T[::-1, :].astype(np.float64) + r.astype(np.float64)).astype(np.float32)
    assert np.array_equal(ho, want), "cfg2 e2e result mismatch"
    # the PCIe bound of the e2e step on this box: the step's whole download
    # (67 MB, one contiguous copy) and whole upload, each timed alone
    d2h_ms = statistics.median(timed_steps(
        L, stream, lambda: tp.download(out, ho, stream), 5, None, gate=False))
    h2d_ms = statistics.median(timed_steps(
        L, stream, lambda: tp.upload(hx, X, stream), 5, None, gate=False))
    pcie = {"d2h_GBps": round(ho.nbytes / d2h_ms / 1e6, 1), "h2d_GBps": round(hx.nbytes / h2d_ms / 1e6, 1),
            "bound_ms": round(max(d2h_ms, h2d_ms), 3)}
    dev.release(flush_buf, stream)
    return ms, e2e_ms, wall, x16.nbytes + r.nbytes, N * N * 4, pcie


def extras(tp, dev, L, warmup=3, steps=5, only=None):
    """Kernel-level numbers for the other configs, rank 0.
    `only`: optional set of config prefixes ("cfg1", "cfg3", ...)."""
    res = {}

    def want(tag):
        return only is None or tag in only
    stream = dev.default_stream()
    flush_buf = dev.allocate(FLUSH_BYTES)

    def flush():
        l2_flush(L, stream, flush_buf)

    def run(name, step, nbytes=None, flops=None, fl=True, st=steps):
        for _ in range(warmup):
            step()
        stream.sync()
        ms = timed_steps(L, stream, step, st, flush if fl else None)
        m = statistics.median(ms)
        rec = {"ms": round(m, 4)}
        if nbytes:
            rec["GB/s"] = round(nbytes / m / 1e6, 1)
        if flops:
            rec["TFLOP/s"] = round(flops / m / 1e9, 1)
        res[name] = rec

    if want("cfg1"):
        rng = np.random.default_rng(1)
        a = tp.from_numpy(rng.standard_normal(1 << 20).astype(np.float32), dev)
        b = tp.from_numpy(rng.standard_normal(1 << 20).astype(np.float32), dev)
        o = tp.tensor_create((1 << 20,), tp.float, dev)
        run("cfg1_add_f32_2^20", lambda: tp.add(a, b, dest=o), nbytes=12 << 20)
        del a, b, o

    if want("cfg3"):
        X = tp.from_numpy(np.asfortranarray(np.random.default_rng(5).random((8192, 8192))), dev)
        nb = 8192 * 8192 * 8
        for op in ("sum", "maximum", "norm"):
            for axes, tag in (((0,), "axis0"), ((1,), "axis1"), (None, "full")):
                run(f"cfg3_{op}_{tag}_f64_8192^2",
                    lambda op=op, axes=axes: tp.reduce(op, X, axes=axes), nbytes=nb)
        del X
    if want("cfg5"):
        cfg5(tp, dev, run)
    if want("cfg4"):
        cfg4(tp, dev, run)
    dev.release(flush_buf, stream)
    return res


def cfg5(tp, dev, run):
    """SURVEY cfg5 at its full 2^30 elements: the f64 big-endian source is
    built on the device from four copies of a 2^28 host-generated slab
    (keeps host memory at 2 GiB)."""
    n5 = 1 << 30
    q = n5 // 4
    chunk = tp.from_numpy(np.random.default_rng(8).uniform(-1e3, 1e3, q).astype(">f8"), dev)
    S = tp.tensor_create((n5,), tp.double, dev)
    S.byteorder = "big"
    for i in range(4):
        tp.copy(chunk, tp.apply_index(S, (slice(i * q, (i + 1) * q),)))
    del chunk
    Y = tp.tensor_create((n5,), tp.float, dev)
    run("cfg5_cast_f64BE_to_f32_2^30", lambda: tp.copy(S, Y), nbytes=12 * n5, fl=False)
    del S
    Z = tp.tensor_create((n5,), tp.float, dev)
    k15, km2 = tp.Scalar(1.5, tp.float), tp.Scalar(-2.0, tp.float)
    run("cfg5_multiply_scalar_f32_2^30", lambda: tp.multiply(Y, k15, dest=Z), nbytes=8 * n5,
        fl=False)
    run("cfg5_add_scalar_f32_2^30", lambda: tp.add(Z, km2, dest=Y), nbytes=8 * n5, fl=False)
    # the same multiply-then-add as one fused chain:
    # 8 B/elem moved instead of 16
    run("cfg5_chain_mul_add_f32_2^30", lambda: tp.chain(Y, [("multiply", k15), ("add", km2)],
                                                          dest=Z), nbytes=8 * n5, fl=False)
    del Y, Z
    c16 = tp.from_numpy(np.random.default_rng(9).integers(-3000, 3000, q).astype(">i2"), dev)
    s16 = tp.tensor_create((n5,), tp.int16, dev)
    s16.byteorder = "big"
    for i in range(4):
        tp.copy(c16, tp.apply_index(s16, (slice(i * q, (i + 1) * q),)))
    del c16
    h16 = tp.tensor_create((n5,), tp.half, dev)
    run("cfg5_cast_i16BE_to_f16_2^30", lambda: tp.copy(s16, h16), nbytes=4 * n5, fl=False)
    del s16, h16


def cfg4(tp, dev, run):
    def gemm_operands(dt, m, k, n, batch=None):
        rng6 = np.random.default_rng(6)
        def mk(rows, cols):
            shape = (rows, cols) if batch is None else (rows, cols, batch)
            base = rng6.uniform(-1, 1, shape).astype(np.float32)
            if dt is tp.bfloat16:
                raw = (base.view(np.uint32) >> 16).astype(np.uint16)
                return tp.from_numpy(np.asfortranarray(raw), dev, dtype=tp.bfloat16)
            npd = np.float16 if dt is tp.half else np.float32
            return tp.from_numpy(np.asfortranarray(base.astype(npd)), dev)
        return mk, mk

    # SURVEY cfg4: A = transpose of a column-major base (K-major), B
    # column-major, C column-major; 2*8192^3 flop per step
    for dname, dt, m in (("f16", tp.half, 8192), ("bf16", tp.bfloat16, 8192),
                         ("f32", tp.float, 8192)):
        mk, _ = gemm_operands(dt, m, m, m)
        At = tp.transpose(mk(m, m))
        B = mk(m, m)
        Cm = tp.tensor_create((m, m), dt, dev)
        run(f"cfg4_gemm_{dname}_{m}^3", lambda: tp.matmul(At, B, dest=Cm), flops=2 * m ** 3,
            fl=False, st=3)
        del At, B, Cm
    # batched: 64 x (2048 x 2048 x 2048), batch slowest
    mk, _ = gemm_operands(tp.half, 2048, 2048, 2048, batch=64)
    Ab, Bb = mk(2048, 2048), mk(2048, 2048)
    Cb = tp.tensor_create((2048, 2048, 64), tp.half, dev)
    run("cfg4_gemm_batched_f16_64x2048^3", lambda: tp.matmul_batched(Ab, Bb, dest=Cb),
        flops=64 * 2 * 2048 ** 3, fl=False, st=3)
    del Ab, Bb, Cb


def sharded_extras(tp, dev, L, dist, steps=5, warmup=3):
    """N>1: the sharded paths of SURVEY §8e measured across all ranks (max
    over ranks of device time per step, whole-job aggregate bytes):
    cfg3 full sum of the f64 8192^2 matrix split along axis 1 (local
    single-pass reduction + ONE NCCL all-reduce over NVLink), and cfg5's
    fused multiply-add chain on 2^30 f32 elements split into slabs."""
    from paper_1810_08723_b200.sharded import NcclComm, Sharded
    import torch.distributed as tdist
    res = {}
    stream = dev.default_stream()

    def share(uid):
        if dist.world == 1:
            return uid
        obj = [uid]
        tdist.broadcast_object_list(obj, src=0)
        return obj[0]

    def timed(step):
        for _ in range(warmup):
            step()
        stream.sync()
        dist.barrier()
        ms = timed_steps(L, stream, step, steps, None, gate=False)
        dist.barrier()
        return dist.max(statistics.median(ms))

    try:
        comm = NcclComm(dev, dist.rank, dist.world, share)
        n = 8192
        cols = np.random.default_rng(5).random((n, n))  # same matrix on every rank
        S = Sharded.from_numpy(cols, dist.rank, dist.world, dev, axis=1)
        del cols
        total = {}

        def red():
            total["v"] = S.reduce_full("sum", comm)
        m = timed(red)
        res[f"cfg3_sum_full_f64_8192^2_sharded_{dist.world}gpu_nccl"] = {
            "ms": round(m, 4), "GB/s": round(n * n * 8 / m / 1e6, 1)}
        comm.close()
    except Exception as exc:  # pragma: no cover - reported, not fatal
        res["cfg3_sharded_error"] = repr(exc)[:200]
    try:
        per = (1 << 30) // dist.world
        Y = tp.tensor_create((per,), tp.float, dev)
        tp.fill(Y, 1.25)
        Z = tp.tensor_create((per,), tp.float, dev)
        k15, km2 = tp.Scalar(1.5, tp.float), tp.Scalar(-2.0, tp.float)
        m = timed(lambda: tp.chain(Y, [("multiply", k15), ("add", km2)], dest=Z))
        res[f"cfg5_chain_f32_2^30_sharded_{dist.world}gpu"] = {
            "ms": round(m, 4), "GB/s": round(dist.world * per * 8 / m / 1e6, 1)}
        del Y, Z
    except Exception as exc:  # pragma: no cover
        res["cfg5_sharded_error"] = repr(exc)[:200]
    return res


def cpu_baseline(steps: int = 5, warmup: int = 1):
    """Reference CPU implementation (oracle/tp_oracle.c, all host threads)
    on the full cfg2 workload (4096 x 4096, the same op as the GPU step):
    `warmup` untimed then `steps` timed passes; returns the median pass."""
    from oracle import oracle
    from paper_1810_08723_b200 import abi
    L = oracle.lib()
    oracle.set_threads(len(os.sched_getaffinity(0)))  # every core this process may use
    cols = N
    x16 = np.asfortranarray(np.random.default_rng(3).integers(-1000, 1000, (N, N),
                                                              endpoint=True).astype(np.int16))
    r = np.asfortranarray(np.random.default_rng(4).standard_normal((1, N)).astype(np.float32))
    out = np.zeros((N, cols), dtype=np.float32, order="F")
    # V = reversed transpose of x16: element (i, j) at x16[j, N-1-i]
    plan = abi.make_plan([N, cols], [[4, 4 * N], [-2 * N, 2], [0, 4]])
    d = abi.make_operand(out.ctypes.data, 0, 10, False)
    a = abi.make_operand(x16.ctypes.data, (N - 1) * 2 * N, 3, False)
    b = abi.make_operand(r.ctypes.data, 0, 10, False)
    st = C.c_uint32(0)
    times = []
    for _ in range(warmup + steps):
        t0 = time.perf_counter()
        L.tpo_binary(0, C.byref(plan), C.byref(d), C.byref(a), C.byref(b), 10, 0, C.byref(st))
        times.append(time.perf_counter() - t0)
    t = statistics.median(times[warmup:])
    elems = N * cols
    want = (x16.T[::-1, :cols].astype(np.float64) + r[:, :cols].astype(np.float64)).astype(np.float32)
    assert np.array_equal(out, want)
    return {"value": round(CFG2_BYTES / t / 1e9, 3), "unit": "GB/s", "cores": oracle.threads(),
            "kind": "port", "sample": f"full cfg2 ({elems} elements, {steps} timed passes, median), "
            "oracle/tp_oracle.c tpo_binary with fused int16->f32 load, OpenMP"}, t


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    dist = Dist()
    hbm_peak, tc_peak, peak_kind = peaks()
    config = {"workload": "cfg2: int16[4096,4096] transposed reversed view (strides -8192,2) "
                          "+ float32[1,4096] broadcast -> float32 add",
              "elements": N * N, "algorithmic_bytes_per_step": CFG2_BYTES,
              "l2": "flushed between timed steps (256 MiB write + read-back, outside the events)", "parallelism": f"dp{dist.world}"}

    if args.impl == "reference":
        if dist.rank != 0:
            dist.close()
            return
        base, t = cpu_baseline(args.steps, args.warmup)
        line = {"metric": METRIC, "value": base["value"], "unit": "GB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded numpy)", "config": config, "impl": "reference",
                "cpu_baseline": base,
                "e2e": {"value": base["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        dist.close()
        return

    import paper_1810_08723_b200 as tp
    from paper_1810_08723_b200 import _native
    L = _native.lib()
    devs = tp.list_devices()
    if not devs:
        raise SystemExit("no CUDA device visible")
    dev = devs[dist.local % len(devs)] if len(devs) > 1 else devs[0]
    clocks = Clocks(dist.phys)
    clocks.start()
    dist.barrier()
    ms, e2e_ms, e2e_wall, h2d, d2h, pcie = bench_cfg2(tp, dev, args.steps, args.warmup, L)
    dist.barrier()
    total = dist.max(sum(ms))
    e2e_total = dist.max(sum(e2e_ms))
    per_step = total / args.steps
    value = dist.world * CFG2_BYTES / (per_step / 1e3) / 1e9
    achieved = CFG2_BYTES / (statistics.mean(ms) / 1e3) / 1e9
    e2e_val = dist.world * CFG2_BYTES / (e2e_total / len(e2e_ms) / 1e3) / 1e9
    work = {}
    if dist.rank == 0 and dist.world == 1 and not args.no_extras:
        work = extras(tp, dev, L)
    elif dist.world > 1 and not args.no_extras:
        work = sharded_extras(tp, dev, L, dist)
    clk = clocks.stop()
    if dist.rank == 0:
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get("cfg2_add_kernel_bytes")
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy)", "config": config,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "peak_kind": peak_kind, "traffic": traffic,
                         "kernel": "tpg::k_tile_f32<add, i16 -> f32, f32 row> (fused cast + broadcast add)"},
            "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_total / len(e2e_ms), 3),
                    "wall_ms_per_step": round(e2e_wall, 3), "pcie": pcie},
            "gpu_launches": args.steps + 1 + len(e2e_ms) * E2E_CHUNKS,
            "clocks": clk,
        }
        if dist.world == 1:
            try:
                base, _ = cpu_baseline()
                line["cpu_baseline"] = base
            except Exception as exc:  # pragma: no cover
                line["cpu_baseline"] = {"error": repr(exc)}
        if work:
            line["workloads"] = work
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
