"""Element types, promotion and host-scalar conversion for the gpu module.

A restatement of the reference dtype contract (pkg/src/tidepool/dtypes.py):
the 15 element types with their wire codes (dtypes.py:69-83), the
smallest-container promotion lattice (143-187), widen_for_compute (190-196),
float_container (131-140) and cast_scalar (281-325).  Device-side element
conversion lives in csrc/tpg_common.cuh; this module only handles what the
host decides (result dtypes, compute dtypes) and host scalars that travel to
the kernels by value.  ``bfloat16`` is an extension (wire code 15) used by
the gemm extension entry; it takes no part in the reference promotion table.
"""

from __future__ import annotations

import math
import struct
import sys

from .errors import CastError, DomainError

MODES = ("standard", "warning", "error", "complex")
MODE_CODE = {m: i for i, m in enumerate(MODES)}


def check_mode(mode: str) -> str:
    """`mode` itself when it is one of MODES (the reference's compute modes)."""
    if mode in MODE_CODE:
        return mode
    raise ValueError(f"unknown compute mode {mode!r}; expected one of {MODES}")


class DType:
    __slots__ = ("name", "code", "size", "is_signed", "is_float", "is_complex", "rank")

    def __init__(self, name, code, size, signed, floating, cmplx, rank):
        self.name = name
        self.code = code
        self.size = size
        self.is_signed = signed
        self.is_float = floating
        self.is_complex = cmplx
        self.rank = rank

    @property
    def wire_code(self) -> int:
        return self.code

    @property
    def is_integer(self) -> bool:
        return not self.is_float and self.name != "bool"

    @property
    def component_size(self) -> int:
        return self.size // 2 if self.is_complex else self.size

    def __repr__(self):
        return self.name

    def __reduce__(self):
        return (by_name, (self.name,))


BOOL = DType("bool", 0, 1, False, False, False, 0)
INT8 = DType("int8", 1, 1, True, False, False, 1)
UINT8 = DType("uint8", 2, 1, False, False, False, 2)
INT16 = DType("int16", 3, 2, True, False, False, 1)
UINT16 = DType("uint16", 4, 2, False, False, False, 2)
INT32 = DType("int32", 5, 4, True, False, False, 1)
UINT32 = DType("uint32", 6, 4, False, False, False, 2)
INT64 = DType("int64", 7, 8, True, False, False, 1)
UINT64 = DType("uint64", 8, 8, False, False, False, 2)
HALF = DType("half", 9, 2, True, True, False, 3)
FLOAT = DType("float", 10, 4, True, True, False, 3)
DOUBLE = DType("double", 11, 8, True, True, False, 3)
CHALF = DType("complex-half", 12, 4, True, True, True, 4)
CFLOAT = DType("complex-float", 13, 8, True, True, True, 4)
CDOUBLE = DType("complex-double", 14, 16, True, True, True, 4)
BFLOAT16 = DType("bfloat16", 15, 2, True, True, False, 3)  # extension

ALL_DTYPES = (BOOL, INT8, UINT8, INT16, UINT16, INT32, UINT32, INT64, UINT64,
              HALF, FLOAT, DOUBLE, CHALF, CFLOAT, CDOUBLE)
_BY_NAME = {d.name: d for d in ALL_DTYPES + (BFLOAT16,)}
_BY_CODE = {d.code: d for d in ALL_DTYPES + (BFLOAT16,)}
_REAL = {CHALF: HALF, CFLOAT: FLOAT, CDOUBLE: DOUBLE}
_CPLX = {HALF: CHALF, FLOAT: CFLOAT, DOUBLE: CDOUBLE}
_SIG = {HALF: 11, FLOAT: 24, DOUBLE: 53, BFLOAT16: 8}


def _lookup(table, key, what):
    d = table.get(key)
    if d is None:
        raise CastError(f"unknown dtype {what} {key!r}")
    return d


def by_name(name: str) -> DType:
    return _lookup(_BY_NAME, name, "name")


def by_code(code: int) -> DType:
    return _lookup(_BY_CODE, code, "wire code")


by_wire_code = by_code


def real_counterpart(d: DType) -> DType:
    return _REAL.get(d, d)


def int_range(d: DType):
    """(min, max) of an integer dtype's values."""
    span = 1 << (8 * d.size)
    lo = -(span >> 1) if d.is_signed else 0
    return lo, lo + span - 1


def float_container(d: DType) -> DType:
    """Smallest real float holding every value of d (ints: 2^p rule)."""
    if d.is_float:
        return real_counterpart(d)
    lo, hi = int_range(d) if d.is_integer else (0, 1)
    for f in (HALF, FLOAT, DOUBLE):
        lim = 1 << _SIG[f]
        if hi <= lim and -lo <= lim:
            return f
    return DOUBLE


def complex_counterpart(d: DType) -> DType:
    if d.is_complex:
        return d
    return _CPLX[float_container(d)]


def _holds(c: DType, a: DType) -> bool:
    """Every value of a is exactly representable in c."""
    if c is a:
        return True
    if a.is_complex:
        return c.is_complex and _holds(_REAL[c], _REAL[a])
    if c.is_complex:
        return _holds(_REAL[c], a)
    if a is BOOL:
        return True
    if a.is_integer:
        lo, hi = int_range(a)
        if c.is_integer:
            clo, chi = int_range(c)
            return clo <= lo and hi <= chi
        if c.is_float:
            lim = 1 << _SIG[c]
            return hi <= lim and -lo <= lim
        return False
    return c.is_float and not c.is_complex and _SIG[c] >= _SIG[a] and c.size >= a.size


_ORDER = sorted(ALL_DTYPES, key=lambda d: (d.size, d.rank, d.code))


def _promote(a: DType, b: DType) -> DType:
    for c in _ORDER:
        if _holds(c, a) and _holds(c, b):
            return c
    return CDOUBLE if (a.is_complex or b.is_complex) else DOUBLE


_PROMOTE = {(a, b): _promote(a, b) for a in ALL_DTYPES for b in ALL_DTYPES}


def promote(a: DType, b: DType) -> DType:
    if a is BFLOAT16 or b is BFLOAT16:
        if a is b:
            return a
        return promote(FLOAT if a is BFLOAT16 else a, FLOAT if b is BFLOAT16 else b)
    return _PROMOTE[(a, b)]


def widen_for_compute(d: DType) -> DType:
    if d is HALF or d is BFLOAT16:
        return FLOAT
    if d is CHALF:
        return CFLOAT
    return d


def lossless_castable(a: DType, c: DType) -> bool:
    return _holds(c, a)


# ---------------------------------------------------------------------------
# global cast policy + warnings (dtypes.py:203-255)
# ---------------------------------------------------------------------------
_implicit = True


def set_implicit_casting(enabled: bool) -> bool:
    global _implicit
    prev, _implicit = _implicit, bool(enabled)
    return prev


def implicit_casting() -> bool:
    return _implicit


def _default_handler(msg: str) -> None:
    print(f"tidepool warning: {msg}", file=sys.stderr)


_handler = _default_handler


def set_warning_handler(h):
    global _handler
    prev = _handler
    _handler = h if h is not None else _default_handler
    return prev


def emit_warning(msg: str) -> None:
    _handler(msg)


# ---------------------------------------------------------------------------
# host scalar conversion (dtypes.py:262-325)
# ---------------------------------------------------------------------------
def _wrap(v: int, d: DType) -> int:
    bits = 8 * d.size
    v &= (1 << bits) - 1
    if d.is_signed and v >= 1 << (bits - 1):
        v -= 1 << bits
    return v


def _narrow(v: float, d: DType) -> float:
    if d is DOUBLE:
        return float(v)
    if d is BFLOAT16:
        return struct.unpack("<f", struct.pack("<I", _bf16_bits(v) << 16))[0]
    fmt = "<e" if d is HALF else "<f"
    try:
        return struct.unpack(fmt, struct.pack(fmt, v))[0]
    except OverflowError:
        return math.inf if v > 0 else -math.inf


def _bf16_bits(v: float) -> int:
    if math.isnan(v):
        return 0x7FC0
    # round-to-nearest-even directly from double
    if v == 0.0 or math.isinf(v):
        f = struct.unpack("<I", struct.pack("<f", v))[0]
        return f >> 16
    m, e = math.frexp(abs(v))
    sign = 0x8000 if v < 0 else 0
    eb = e - 1
    if eb < -126:
        r = round(math.ldexp(abs(v), 133))
        return sign | (0x80 if r >= 128 else r)
    r = round(math.ldexp(m, 8))
    if r >= 256:
        r, eb = 128, eb + 1
    if eb > 127:
        return sign | 0x7F80
    return sign | ((eb + 127) << 7) | (r - 128)


def cast_scalar(value, to: DType, mode: str = "standard", loss: list | None = None):
    """Python value of `value` stored as dtype `to` (reference cast_scalar)."""
    def lost(msg):
        if mode == "error":
            raise DomainError(msg)
        if loss is not None:
            loss.append(msg)

    if isinstance(value, complex):
        if to.is_complex:
            comp = real_counterpart(to)
            return complex(_narrow(value.real, comp), _narrow(value.imag, comp))
        if value.imag != 0.0:
            lost(f"discarding nonzero imaginary part {value.imag!r}")
        value = value.real
    if to is BOOL:
        return value != 0
    if to.is_complex:
        return complex(_narrow(float(value), real_counterpart(to)), 0.0)
    if to.is_float:
        return _narrow(float(value), to)
    if isinstance(value, bool):
        return int(value)
    if isinstance(value, float):
        if math.isnan(value) or math.isinf(value):
            lost(f"cannot represent {value!r} as {to.name}")
            return 0
        value = math.trunc(value)
    lo, hi = int_range(to)
    if not lo <= value <= hi:
        lost(f"value {value} out of range for {to.name}")
    return _wrap(int(value), to)


def infer_scalar_dtype(value) -> DType:
    for kind, d in ((bool, BOOL), (int, INT64), (float, DOUBLE), (complex, CDOUBLE)):
        if isinstance(value, kind):
            return d
    raise CastError(f"{value!r} is not a bool, int, float or complex scalar")


_FMT = {BOOL: "?", INT8: "b", UINT8: "B", INT16: "h", UINT16: "H", INT32: "i",
        UINT32: "I", INT64: "q", UINT64: "Q", HALF: "e", FLOAT: "f", DOUBLE: "d"}


def pack_value(d: DType, value, byteorder: str = "little") -> bytes:
    """Element bytes of an already-cast value (reference codec pack)."""
    p = "<" if byteorder == "little" else ">"
    if d is BFLOAT16:
        return struct.pack(p + "H", _bf16_bits(float(value)))
    if d.is_complex:
        f = _FMT[real_counterpart(d)]
        return struct.pack(p + f + f, value.real, value.imag)
    return struct.pack(p + _FMT[d], value)


def unpack_value(d: DType, buf, off: int = 0, byteorder: str = "little"):
    p = "<" if byteorder == "little" else ">"
    if d is BFLOAT16:
        (h,) = struct.unpack_from(p + "H", buf, off)
        return struct.unpack("<f", struct.pack("<I", h << 16))[0]
    if d.is_complex:
        f = _FMT[real_counterpart(d)]
        re_, im = struct.unpack_from(p + f + f, buf, off)
        return complex(re_, im)
    return struct.unpack_from(p + _FMT[d], buf, off)[0]


NATIVE_ORDER = sys.byteorder

# numpy interop (tests / host staging)
NUMPY_NAME = {BOOL: "bool", INT8: "int8", UINT8: "uint8", INT16: "int16",
              UINT16: "uint16", INT32: "int32", UINT32: "uint32", INT64: "int64",
              UINT64: "uint64", HALF: "float16", FLOAT: "float32", DOUBLE: "float64",
              CHALF: None, CFLOAT: "complex64", CDOUBLE: "complex128", BFLOAT16: None}
