"""OTP1 header logic on the host (no GPU): every golden blob written by the
reference (tests/golden/make_otp1.py, interop.py:94-127) parses back to its
own header bytes, and malformed headers raise FormatError with the
reference's distinct messages (tests/test_interop.py:80-130)."""

import io
from pathlib import Path

import numpy as np
import pytest

from paper_1810_08723_b200 import otp1
from paper_1810_08723_b200.errors import FormatError

BLOBS = np.load(Path(__file__).resolve().parent / "golden" / "otp1_blobs.npz")
KEYS = [k for k in BLOBS.files if not k.startswith("_") and not k.endswith(".base")]


@pytest.mark.parametrize("key", KEYS)
def test_golden_headers_round_trip(key):
    blob = BLOBS[key].tobytes()
    src = io.BytesIO(blob)
    dtype, order, dims = otp1.parse_header(src)
    head = otp1.pack_header(dtype, order, dims)
    assert blob[:len(head)] == head
    assert len(blob) - len(head) == int(np.prod(dims, dtype=np.int64)) * dtype.size


def _blob():
    return bytearray(BLOBS["float-little-3x4"].tobytes())


@pytest.mark.parametrize("mutate,word", [("magic", "magic"), ("reserved", "reserved"),
                                         ("dtype", "dtype"), ("ndim", "dimensions")])
def test_malformed_headers(mutate, word):
    b = _blob()
    if mutate == "magic":
        b[3] = 2
    elif mutate == "reserved":
        b[7] = 1
    elif mutate == "dtype":
        b[4] = 99
    else:
        b[6] = 9
        b += bytes(8 * 7)
    with pytest.raises(FormatError, match=word):
        otp1.parse_header(io.BytesIO(bytes(b)))


def test_truncated_header_and_dims():
    with pytest.raises(FormatError, match="header"):
        otp1.parse_header(io.BytesIO(b"OTP"))
    with pytest.raises(FormatError, match="dimension"):
        otp1.parse_header(io.BytesIO(bytes(_blob()[:12])))


def test_distinct_messages():
    seen = set()
    for mutate in ("magic", "reserved", "dtype"):
        b = _blob()
        b[{"magic": 0, "reserved": 7, "dtype": 4}[mutate]] = {"magic": 0, "reserved": 3,
                                                               "dtype": 77}[mutate]
        try:
            otp1.parse_header(io.BytesIO(bytes(b)))
        except FormatError as exc:
            seen.add(str(exc).split(" ")[0] + str(exc).split(" ")[1])
    assert len(seen) == 3
