"""Extract the roofline-relevant metrics of an `ncu --set full` report.

usage: python scripts/ncu_report.py gpurun_out/prof.ncu-rep "title" [algorithmic_bytes]
"""

import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", None),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def main(path, title, alg_bytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# {title}\n")
    print(f"`{path}` (ncu --set full --clock-control none; cold cache, one launch)\n")
    for r in rows[2:]:
        print("| metric | value |\n|---|---|")
        dur = None
        traffic = 0.0
        for key, label in KEYS:
            if key not in hdr:
                continue
            i = hdr.index(key)
            v = r[i]
            u = units[i]
            if key == "gpu__time_duration.sum":
                dur = float(v.replace(",", "")) * (1e-3 if u in ("ns", "nsecond") else 1.0)
            if key.startswith("dram__bytes"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                traffic += float(v.replace(",", "")) * scale
            print(f"| {label or key} | {v[:90]} {u} |")
        print(f"| DRAM traffic (read+write) | {traffic / 1e6:.2f} MB |")
        if alg_bytes and dur:
            print(f"| algorithmic bytes | {alg_bytes / 1e6:.2f} MB |")
            print(f"| algorithmic GB/s under ncu | {alg_bytes / dur / 1e3:.1f} |")
        print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
