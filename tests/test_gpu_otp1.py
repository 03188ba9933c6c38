"""OTP1 files straight to / from the GPU against blobs
written by the reference (tests/golden/make_otp1.py): load + save is
bit-identical for all 15 dtypes x both byte orders x 0-dim / empty / N-d
shapes, strided views save exactly what the reference writes, multi-chunk
streaming through pinned buffers, on-device byte swap (native=True)."""

import io
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import otp1
from paper_1810_08723_b200.errors import FormatError

pytestmark = pytest.mark.gpu

BLOBS = np.load(Path(__file__).resolve().parent / "golden" / "otp1_blobs.npz")
META = json.loads(BLOBS["_meta"].tobytes())
KEYS = [k for k in BLOBS.files if not k.startswith("_") and not k.endswith(".base")
        and not k.startswith("strided-")]


def _device_bytes(t):
    n = t.nelem * t.dtype.size
    return bytes(t.storage.snapshot()[t.offset:t.offset + n]) if n else b""


def test_golden_round_trip_all_dtypes():
    for key in KEYS:
        blob = BLOBS[key].tobytes()
        t = otp1.load_otp1(blob)
        assert t.device.type.name == "gpu"
        dtype, order, dims = otp1.parse_header(io.BytesIO(blob))
        assert (t.dtype, t.byteorder, t.dims) == (dtype, order, dims), key
        head = len(otp1.pack_header(dtype, order, dims))
        assert _device_bytes(t) == blob[head:], key
        assert otp1.save_otp1_bytes(t) == blob, key


@pytest.mark.parametrize("key", [k for k in META])
def test_strided_views_save_like_the_reference(key):
    base = otp1.load_otp1(BLOBS[key + ".base"].tobytes())
    view = tp.apply_index(base, tuple(slice(a, b, c) for a, b, c in META[key]))
    assert otp1.save_otp1_bytes(view) == BLOBS[key].tobytes()


def test_multichunk_file_round_trip(tmp_path):
    x = np.random.default_rng(5).standard_normal((1000, 777)).astype(np.float32)
    t = tp.from_numpy(np.asfortranarray(x))
    path = str(tmp_path / "x.otp1")
    otp1.save_otp1(t, path, chunk=1 << 18)          # 12 chunks of 256 KiB
    back = otp1.load_otp1(path, chunk=(1 << 18) + 4)
    assert np.array_equal(tp.to_numpy(back), x)
    with open(path, "rb") as fh:
        blob = fh.read()
    assert otp1.save_otp1_bytes(back) == blob


def test_native_byteswap_on_device():
    key = "double-big-3x4"
    big = otp1.load_otp1(BLOBS[key].tobytes())
    nat = otp1.load_otp1(BLOBS[key].tobytes(), native=True)
    assert big.byteorder == "big" and nat.byteorder == "little"
    assert tp.array_equal(big, nat)


def test_truncated_payload():
    blob = BLOBS["float-little-3x4"].tobytes()
    with pytest.raises(FormatError, match="payload"):
        otp1.load_otp1(blob[:-4])
