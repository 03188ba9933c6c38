"""Print bench.py's `workloads` for a subset of configs (A/B runs):
python scripts/extras_probe.py cfg5 [cfg3 ...]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
import bench  # noqa: E402
import paper_1810_08723_b200 as tp  # noqa: E402
from paper_1810_08723_b200 import _native  # noqa: E402

r = bench.extras(tp, tp.gpu(0), _native.lib(), only=set(sys.argv[1:]))
print(json.dumps({k: v.get("GB/s") or v.get("TFLOP/s") for k, v in r.items()}))
