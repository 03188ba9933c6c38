"""Generate OTP1 golden blobs with the REFERENCE implementation
(interop.save_otp1_bytes, /root/reference/pkg/src/tidepool/interop.py:94-127).

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_otp1.py
Writes tests/golden/otp1_blobs.npz: for each case `<name>` the reference
blob, plus for strided cases `<name>.base` (the blob of the contiguous base
tensor) and `<name>.index` (the slice spec applied to it).
"""

import json
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tidepool as tp  # noqa: E402
from tidepool import interop  # noqa: E402
from tidepool import tensors as tz  # noqa: E402

OUT = Path(__file__).resolve().parent / "otp1_blobs.npz"


def filled(dims, dt, rng):
    t = tp.tensor(dims, dt)
    buf = t.storage.view()
    raw = bytes(rng.getrandbits(8) for _ in range(len(buf)))
    buf[:] = raw
    return t


def main():
    rng = random.Random(1810)
    blobs, meta = {}, {}
    names = [d for d in tp.dtypes.ALL_DTYPES] if hasattr(tp.dtypes, "ALL_DTYPES") else None
    dts = names or [tp.dtypes.by_wire_code(c) for c in range(15)]
    for dt in dts:
        for order in ("little", "big"):
            for dims in ((3, 4), (), (0, 2), (2, 3, 2)):
                t = filled(dims, dt, rng)
                t.byteorder = order
                key = f"{dt.name}-{order}-{'x'.join(map(str, dims)) or 'scalar'}"
                blobs[key] = np.frombuffer(interop.save_otp1_bytes(t), np.uint8)
    # strided inputs: layout normalised, bytes kept (interop.py:105-121)
    for dt in (tp.dtypes.by_wire_code(3), tp.dtypes.by_wire_code(10), tp.dtypes.by_wire_code(14)):
        base = filled((6, 5), dt, rng)
        spec = [[0, 6, 2], [4, None, -1]]
        view = tz.apply_index(base, tuple(slice(a, b, c) for a, b, c in spec)) \
            if hasattr(tz, "apply_index") else None
        if view is None:
            from tidepool import indexing
            view = indexing.apply_index(base, tuple(slice(a, b, c) for a, b, c in spec))
        key = f"strided-{dt.name}"
        blobs[key] = np.frombuffer(interop.save_otp1_bytes(view), np.uint8)
        blobs[key + ".base"] = np.frombuffer(interop.save_otp1_bytes(base), np.uint8)
        meta[key] = spec
    np.savez_compressed(OUT, **blobs, _meta=np.frombuffer(json.dumps(meta).encode(), np.uint8))
    print(f"{len(blobs)} blobs -> {OUT}")


if __name__ == "__main__":
    main()
