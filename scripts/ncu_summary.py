"""Summarise an ncu --csv launch list (gpu__time_duration.sum) into markdown.

usage: python scripts/ncu_summary.py gpurun_out/launches.csv "title" > profiles/rNN_launches.md
Per-launch times under ncu are cold-cache and serialised: compare shares.
"""

import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, title):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit",
                                             "Metric Value"))
    gi = hdr.index("Grid Size")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki]
        if "k_gate" in name:
            continue
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        a = agg.setdefault((name[:120], r[gi]), [0, 0.0, []])
        a[0] += 1
        a[1] += us
        a[2].append(us)
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"# {title}\n")
    print("ncu `--metrics gpu__time_duration.sum --clock-control none`; cold-cache, serialised "
          "launches: compare shares, not absolutes.\n")
    print("| kernel | grid | launches | mean us | total us | share |")
    print("|---|---|---|---|---|---|")
    for (k, g), (n, t, _) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {g} | {n} | {t / n:.2f} | {t:.1f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu launch list")
