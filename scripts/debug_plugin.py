"""Step-by-step comparison of the reference on cpu vs gpu0 (plugin debug)."""
import math
import random
import struct
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import tidepool as tp  # noqa: E402
from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

tidepool_plugin.register(tp, count=1)
gpu = tp.devices.by_name("gpu0")


def mk(device, seed):
    tz = tp.tensors
    a = tp.tensor_create((4, 3), tp.double, device)
    b = tp.tensor_create((4, 3), tp.double, device)
    st = random.Random(seed)
    for t in (a, b):
        _, pack = tp.dtypes.codec(t.dtype, t.byteorder)
        buf = t.storage.view()
        for off in tz.iter_offsets(t):
            pack(buf, off, round(st.uniform(-4, 4), 3) or 1.0)
    return a, b


def bits(v):
    return struct.pack("<d", v).hex()


for seed in range(3):
    ac, bc = mk(tp.cpu(), seed)
    ag, bg = mk(gpu, seed)
    va = tp.tensors.read_values(ac)
    vga = tp.tensors.read_values(ag)
    print("inputs equal:", va == vga, tp.tensors.read_values(bc) == tp.tensors.read_values(bg))
    cc = tp.add(ac, bc)
    cg = tp.add(ag, bg)
    x, y = tp.tensors.read_values(cc), tp.tensors.read_values(cg)
    print("add equal:", x == y, [(i, a, b) for i, (a, b) in enumerate(zip(x, y)) if a != b][:3])
    tp.multiply(cc, 2.0, dest=cc)
    tp.multiply(cg, 2.0, dest=cg)
    x, y = tp.tensors.read_values(cc), tp.tensors.read_values(cg)
    print("mul equal:", x == y, [(i, a, b, bits(a), bits(b)) for i, (a, b) in enumerate(zip(x, y)) if a != b][:3])
    print("stats", {k: v for k, v in tp.dispatch.table_stats("core", "gpu").items() if v})
