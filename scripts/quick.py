"""Quick kernel numbers for a subset of configs (iteration aid, not the bench).

usage: python scripts/quick.py cfg3 [cfg4 ...]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1810_08723_b200 as tp  # noqa: E402
from paper_1810_08723_b200 import _native  # noqa: E402

if __name__ == "__main__":
    dev = tp.list_devices()[0]
    res = bench.extras(tp, dev, _native.lib(), only=set(sys.argv[1:]) or None)
    hbm, tc, _ = bench.peaks()
    for k, v in res.items():
        frac = v["GB/s"] / hbm if "GB/s" in v else v["TFLOP/s"] / tc
        print(f"{k:40s} {json.dumps(v):45s} frac={frac:.3f}")
