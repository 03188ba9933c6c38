"""Markdown table of an `ncu --page raw --csv` export of scripts/hot_kernels.py.

usage: python scripts/hot_table.py gpurun_out/prof_hot_raw.csv "title" > profiles/rNN_ncu_hot_kernels.md
Algorithmic units: reductions 8 B per f64 element read, chain
8 B per f32 element, tf32 split 12 B per element, gemm 2mnk flop.
"""
import csv
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
# order of the launches in scripts/hot_kernels.py and their algorithmic work
WORK = [("sum axis 0", 8 * 8192 ** 2, "B"), ("sum axis 1", 8 * 8192 ** 2, "B"),
        ("sum full", 8 * 8192 ** 2, "B"), ("max axis 1", 8 * 8192 ** 2, "B"),
        ("chain 2^28 f32", 8 * 2 ** 28, "B"), ("gemm f16 8192^3", 2 * 8192 ** 3, "F"),
        ("tf32 split A", 12 * 8192 ** 2, "B"), ("tf32 split B", 12 * 8192 ** 2, "B"),
        ("gemm 3xTF32 8192^3", 2 * 8192 ** 3, "F"), ("batched f16 64x2048^3", 64 * 2 * 2048 ** 3, "F")]


def main(path, title):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], [r for r in rows[2:] if r and r[0]]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, key):
        i = col[key]
        v = float(r[i].replace(",", ""))
        return v * UNIT.get(units[i], 1.0)

    print(f"# {title}\n")
    print("`ncu --set full --clock-control none`, one launch each, cold L2 (ncu flushes between "
          "passes).  Algorithmic work per SURVEY §8d; GB/s and TFLOP/s = work / ncu duration.\n")
    print("| launch | kernel | grid | regs | duration us | DRAM read MB | DRAM write MB | "
          "DRAM % peak | algorithmic | tensor pipe % active | L1/smem % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for k, r in enumerate(data):
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "")
        us = val(r, "gpu__time_duration.sum")
        label, work, kind = WORK[k] if k < len(WORK) else ("?", 0, "B")
        alg = (f"{work / us / 1e3:.0f} GB/s" if kind == "B" else f"{work / us / 1e6:.0f} TFLOP/s")
        print(f"| {label} | `{name}` | {r[col['Grid Size']]} | "
              f"{r[col['launch__registers_per_thread']]} | {us:.1f} | "
              f"{val(r, 'dram__bytes_read.sum') / 1e6:.1f} | {val(r, 'dram__bytes_write.sum') / 1e6:.1f} | "
              f"{val(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {alg} | "
              f"{val(r, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{val(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
