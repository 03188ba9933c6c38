"""cfg4 gemm: the product tcgen05 kernels next to cuBLAS (torch.matmul /
torch.bmm) on the same box, same shapes, same operand distribution
(uniform(-1, 1): the 1 kW power cap makes throughput depend on operand
mantissa entropy, profiles/r02_gemm_f16_vs_bf16_power.md), same
back-to-back timing (5 launches between one event pair, median of 3).
Diagnostic only: cuBLAS is the reference point for "what this box's power
cap allows", not part of the product.  Runs ours / cuBLAS twice,
interleaved, to expose drift."""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
import bench  # noqa: E402
import paper_1810_08723_b200 as tp  # noqa: E402
from paper_1810_08723_b200 import _native  # noqa: E402


def ours():
    r = bench.extras(tp, tp.gpu(0), _native.lib(), only={"cfg4"})
    return {k: v["TFLOP/s"] for k, v in r.items() if "TFLOP/s" in v}


def cublas():
    import torch
    out = {}
    g = torch.Generator(device="cuda").manual_seed(0)

    def rnd(shape, dt):
        return (torch.rand(shape, device="cuda", generator=g) * 2 - 1).to(dt)

    def timeit(fn, flops):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                fn()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b) / 5)
        return round(flops / statistics.median(ms) / 1e9, 1)
    m = 8192
    for name, dt in (("f16", torch.float16), ("bf16", torch.bfloat16)):
        A, B = rnd((m, m), dt), rnd((m, m), dt)
        C = torch.empty((m, m), device="cuda", dtype=dt)
        out[f"cfg4_gemm_{name}_{m}^3"] = timeit(lambda: torch.matmul(A, B, out=C), 2 * m ** 3)
        del A, B, C
    A, B = rnd((64, 2048, 2048), torch.float16), rnd((64, 2048, 2048), torch.float16)
    C = torch.empty((64, 2048, 2048), device="cuda", dtype=torch.float16)
    out["cfg4_gemm_batched_f16_64x2048^3"] = timeit(lambda: torch.bmm(A, B, out=C),
                                                    64 * 2 * 2048 ** 3)
    return out


def sustained(kind, seconds=3.0):
    """f16 8192^3 and batched back to back for `seconds` each, SM clock and
    power sampled by nvidia-smi meanwhile (median under load)."""
    import subprocess
    import threading
    import time
    import torch
    res = {}
    m = 8192
    if kind == "ours":
        import numpy as np
        dev = tp.gpu(0)
        h = np.asfortranarray(np.random.default_rng(6).uniform(-1, 1, (m, m)).astype(np.float16))
        h2 = np.asfortranarray(np.random.default_rng(8).uniform(-1, 1, (m, m)).astype(np.float16))
        A, B = tp.transpose(tp.from_numpy(h, dev)), tp.from_numpy(h2, dev)
        Cm = tp.tensor_create((m, m), tp.half, dev)
        hb = np.asfortranarray(np.random.default_rng(7).uniform(-1, 1, (2048, 2048, 64))
                               .astype(np.float16))
        hb2 = np.asfortranarray(np.random.default_rng(9).uniform(-1, 1, (2048, 2048, 64))
                                .astype(np.float16))
        Ab, Bb = tp.from_numpy(hb, dev), tp.from_numpy(hb2, dev)
        Cb = tp.tensor_create((2048, 2048, 64), tp.half, dev)
        cases = {"f16_8192^3": (lambda: tp.matmul(A, B, dest=Cm), 2 * m ** 3,
                                lambda: dev.default_stream().sync()),
                 "batched": (lambda: tp.matmul_batched(Ab, Bb, dest=Cb), 64 * 2 * 2048 ** 3,
                             lambda: dev.default_stream().sync())}
    else:
        A = (torch.rand((m, m), device="cuda") * 2 - 1).half()
        B = (torch.rand((m, m), device="cuda") * 2 - 1).half()
        C = torch.empty_like(A)
        Ab = (torch.rand((64, 2048, 2048), device="cuda") * 2 - 1).half()
        Bb = (torch.rand((64, 2048, 2048), device="cuda") * 2 - 1).half()
        Cb = torch.empty_like(Ab)
        cases = {"f16_8192^3": (lambda: torch.matmul(A, B, out=C), 2 * m ** 3,
                                torch.cuda.synchronize),
                 "batched": (lambda: torch.bmm(Ab, Bb, out=Cb), 64 * 2 * 2048 ** 3,
                             torch.cuda.synchronize)}
    for name, (fn, flops, sync) in cases.items():
        samples, stop = [], threading.Event()

        def poll():
            while not stop.is_set():
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                      "--format=csv,noheader,nounits", "-i", "0"],
                                     capture_output=True, text=True).stdout.split(",")
                try:
                    samples.append((float(out[0]), float(out[1])))
                except (ValueError, IndexError):
                    pass
                time.sleep(0.1)
        for _ in range(3):
            fn()
        sync()
        th = threading.Thread(target=poll)
        th.start()
        t0, n = time.perf_counter(), 0
        while time.perf_counter() - t0 < seconds:
            for _ in range(5):
                fn()
            sync()
            n += 5
        dt = time.perf_counter() - t0
        stop.set()
        th.join()
        mid = samples[len(samples) // 4:] or samples
        res[name] = {"TFLOP/s": round(flops * n / dt / 1e12, 1),
                     "sm_mhz": statistics.median(s[0] for s in mid),
                     "power_w": statistics.median(s[1] for s in mid)}
    return res


if __name__ == "__main__":
    rows = {}
    for rnd_ in range(2):
        for k, v in ours().items():
            rows.setdefault(k, {}).setdefault("ours", []).append(v)
        for k, v in cublas().items():
            rows.setdefault(k, {}).setdefault("cublas", []).append(v)
    print("| workload | ours TFLOP/s (run 1, 2) | cuBLAS TFLOP/s (run 1, 2) | ours / cuBLAS |")
    print("|---|---|---|---|")
    for k, d in rows.items():
        o, c = d.get("ours", []), d.get("cublas", [])
        ratio = (f"{statistics.mean(o) / statistics.mean(c):.3f}" if o and c else "-")
        print(f"| {k} | {', '.join(map(str, o))} | {', '.join(map(str, c))} | {ratio} |")
    print()
    print("Sustained (3 s back to back each, nvidia-smi median under load):")
    print()
    print("| impl | workload | TFLOP/s | SM MHz | power W | TFLOP/s per GHz |")
    print("|---|---|---|---|---|---|")
    for impl in ("ours", "cublas"):
        for k, v in sustained(impl).items():
            print(f"| {impl} | {k} | {v['TFLOP/s']} | {v['sm_mhz']:.0f} | {v['power_w']:.0f} | "
                  f"{1000 * v['TFLOP/s'] / max(v['sm_mhz'], 1):.0f} |")
