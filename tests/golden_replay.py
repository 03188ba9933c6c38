"""Replay the captured reference table calls (tests/golden/*.npz) through a
backend (the C oracle on host buffers, or libtidepool_gpu on device
buffers) and compare destination bytes element by element."""

from __future__ import annotations

import ctypes as C
import json
import math
import struct
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_1810_08723_b200 import abi, dtypes as D

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_table_calls.npz"


@lru_cache(maxsize=None)
def load_records():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    blob, offs = z["blob"], z["offs"]
    blobs = [bytes(blob[offs[i]:offs[i + 1]]) for i in range(len(offs) - 1)]
    return meta, blobs


def dt(name):
    return D.by_name(name)


def _plan(ext, strides):
    return abi.make_plan(ext, strides)


def _operand(ptr, off, spec):
    return abi.make_operand(ptr, off, dt(spec[0]).code, spec[1] == "big")


# ---------------------------------------------------------------------------
# destination element offsets written by a record
# ---------------------------------------------------------------------------
def _plan_offsets(ext, strides, base):
    offs = [base]
    total = math.prod(ext) if ext else 1
    if total == 0:
        return []
    out = []
    idx = [0] * len(ext)
    off = base
    for _ in range(total):
        out.append(off)
        for k, e in enumerate(ext):
            idx[k] += 1
            off += strides[k]
            if idx[k] < e:
                break
            idx[k] = 0
            off -= strides[k] * e
    _ = offs
    return out


def dest_offsets(r):
    e = r["entry"]
    if e in ("binary", "unary", "copy", "fill", "arange", "byteswap"):
        return _plan_offsets(r["ext"], r["str"][0], r["bases"][0])
    if e == "reduce":
        return _plan_offsets(r["oext"], r["ostr"][0], r["bases"][0])
    if e == "matmul":
        return [r["bases"][0] + i * r["dstr"][0] + j * r["dstr"][1]
                for j in range(r["n"]) for i in range(r["m"])]
    if e in ("gather", "scatter"):
        return [p[0] for p in r["pairs"]]
    if e == "scatter_fill":
        return list(r["offsets"])
    raise KeyError(e)


def dest_dtype(r):
    if r["entry"] == "gather":
        return None
    return dt(r["d"][0])


# ---------------------------------------------------------------------------
# backends
# ---------------------------------------------------------------------------
class HostBackend:
    """C oracle on host bytearrays."""

    def __init__(self):
        from oracle import oracle
        self.L = oracle.lib()

    def run(self, r, blobs):
        bufs = {}
        for key, bi in r["bufs"].items():
            if key.startswith("buf"):
                bufs[key] = bytearray(blobs[bi])
        ptr = {k: C.addressof(C.c_char.from_buffer(v)) if len(v) else 0 for k, v in bufs.items()}
        role = {k: r["bufs"][k] for k in ("d", "a", "b") if k in r["bufs"]}
        st = C.c_uint32(0)
        self._call(r, {k: ptr[v] for k, v in role.items()}, st, bufs, role)
        return bytes(bufs[role["d"]]), st.value

    def _call(self, r, P, st, bufs, role):
        L, e = self.L, r["entry"]
        mode = D.MODE_CODE[r.get("mode", "standard")]
        if e == "binary":
            p = _plan(r["ext"], r["str"])
            d, a, b = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("dab"))
            L.tpo_binary(abi.BINARY_CODE[r["op"]], C.byref(p), C.byref(d), C.byref(a), C.byref(b),
                         dt(r["compute"]).code, mode, C.byref(st))
        elif e in ("unary", "copy"):
            p = _plan(r["ext"], r["str"])
            d, a = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("da"))
            code = abi.UNARY_CODE["identity" if e == "copy" else r["op"]]
            L.tpo_unary(code, C.byref(p), C.byref(d), C.byref(a), dt(r["compute"]).code, mode,
                        int(r.get("force_complex", False)), C.byref(st))
        elif e == "reduce":
            po, pi = _plan(r["oext"], r["ostr"]), _plan(r["iext"], r["istr"])
            d, a = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("da"))
            op = r["op"].replace("reduce_", "")
            L.tpo_reduce(abi.REDUCE_CODE[op], r["p"], C.byref(po), C.byref(pi), C.byref(d),
                         C.byref(a), 0, mode, C.byref(st))
        elif e == "matmul":
            d, a, b = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("dab"))
            arr = lambda s: (C.c_int64 * 2)(*s)
            L.tpo_matmul(C.byref(d), arr(r["dstr"]), C.byref(a), arr(r["astr"]), C.byref(b),
                         arr(r["bstr"]), r["m"], r["n"], r["k"], dt(r["compute"]).code, mode,
                         C.byref(st))
        elif e == "fill":
            p = _plan(r["ext"], r["str"])
            d = _operand(P["d"], r["bases"][0], r["d"])
            v = bytes.fromhex(r["value"])
            L.tpo_fill(C.byref(p), C.byref(d), v, len(v))
        elif e == "arange":
            p = _plan(r["ext"], r["str"])
            d = _operand(P["d"], r["bases"][0], r["d"])
            L.tpo_arange(C.byref(p), C.byref(d))
        elif e == "byteswap":
            p = _plan(r["ext"], r["str"])
            d = _operand(P["d"], r["bases"][0], r["d"])
            L.tpo_byteswap(C.byref(p), C.byref(d))
        elif e == "gather":
            dst, src = bufs[role["d"]], bufs[role["a"]]
            for do, so in r["pairs"]:
                dst[do:do + r["size"]] = src[so:so + r["size"]]
        elif e == "scatter":
            # value moves with conversion: one-element copies through the oracle
            for do, so in r["pairs"]:
                p = _plan([], [[], []])
                d = _operand(P["d"], do, r["d"])
                a = _operand(P["a"], so, r["a"])
                L.tpo_unary(abi.UNARY_CODE["identity"], C.byref(p), C.byref(d), C.byref(a),
                            dt(r["a"][0]).code, mode, 0, C.byref(st))
        elif e == "scatter_fill":
            dst = bufs[role["d"]]
            v = bytes.fromhex(r["value"])
            for o in r["offsets"]:
                dst[o:o + len(v)] = v
        else:
            raise KeyError(e)


class GpuBackend:
    """libtidepool_gpu through its C ABI on device buffers."""

    def __init__(self):
        from paper_1810_08723_b200 import _native
        self.L = _native.lib()
        self.native = _native

    def _alloc(self, data: bytes):
        p = C.c_void_p()
        self.native.check(self.L.tpg_malloc(0, max(len(data), 1), C.byref(p)))
        if data:
            self.native.check(self.L.tpg_memcpy_h2d(p.value, data, len(data), None))
        return p.value

    def run(self, r, blobs):
        L = self.L
        keys = [k for k in r["bufs"] if k.startswith("buf")]
        host = {k: blobs[r["bufs"][k]] for k in keys}
        dev = {k: self._alloc(host[k]) for k in keys}
        role = {k: r["bufs"][k] for k in ("d", "a", "b") if k in r["bufs"]}
        P = {k: dev[v] for k, v in role.items()}
        L.tpg_flags_clear(0)
        try:
            rc = self._call(r, P)
            self.native.check(rc, r["entry"])
            self.native.check(L.tpg_stream_sync(None))
            out = bytearray(len(host[role["d"]]))
            if out:
                buf = (C.c_char * len(out)).from_buffer(out)
                self.native.check(L.tpg_memcpy_d2h(buf, P["d"], len(out), None))
                self.native.check(L.tpg_stream_sync(None))
            f = C.c_uint32(0)
            L.tpg_flags_get(0, C.byref(f))
            L.tpg_flags_clear(0)
            return bytes(out), f.value
        finally:
            for p in dev.values():
                L.tpg_free(0, p, None)

    def _call(self, r, P):
        L, e = self.L, r["entry"]
        mode = D.MODE_CODE[r.get("mode", "standard")]
        if e == "binary":
            p = _plan(r["ext"], r["str"])
            d, a, b = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("dab"))
            return L.tpg_binary(None, abi.BINARY_CODE[r["op"]], C.byref(p), C.byref(d), C.byref(a),
                                C.byref(b), dt(r["compute"]).code, mode)
        if e in ("unary", "copy"):
            p = _plan(r["ext"], r["str"])
            d, a = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("da"))
            code = abi.UNARY_CODE["identity" if e == "copy" else r["op"]]
            return L.tpg_unary(None, code, C.byref(p), C.byref(d), C.byref(a),
                               dt(r["compute"]).code, mode, int(r.get("force_complex", False)))
        if e == "reduce":
            po, pi = _plan(r["oext"], r["ostr"]), _plan(r["iext"], r["istr"])
            d, a = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("da"))
            op = r["op"].replace("reduce_", "")
            return L.tpg_reduce(None, abi.REDUCE_CODE[op], r["p"], C.byref(po), C.byref(pi),
                                C.byref(d), C.byref(a), 0, mode)
        if e == "matmul":
            d, a, b = (_operand(P[x], r["bases"][i], r[x]) for i, x in enumerate("dab"))
            arr = lambda s: (C.c_int64 * 2)(*s)
            return L.tpg_matmul(None, C.byref(d), arr(r["dstr"]), C.byref(a), arr(r["astr"]),
                                C.byref(b), arr(r["bstr"]), r["m"], r["n"], r["k"],
                                dt(r["compute"]).code, mode)
        if e == "fill":
            p = _plan(r["ext"], r["str"])
            d = _operand(P["d"], r["bases"][0], r["d"])
            v = bytes.fromhex(r["value"])
            return L.tpg_fill(None, C.byref(p), C.byref(d), v, len(v))
        if e == "arange":
            return L.tpg_arange(None, C.byref(_plan(r["ext"], r["str"])),
                                C.byref(_operand(P["d"], r["bases"][0], r["d"])))
        if e == "byteswap":
            return L.tpg_byteswap(None, C.byref(_plan(r["ext"], r["str"])),
                                  C.byref(_operand(P["d"], r["bases"][0], r["d"])))
        if e == "gather":
            pairs = np.asarray(r["pairs"], dtype=np.int64).reshape(-1)
            return L.tpg_gather(None, P["d"], P["a"], pairs.ctypes.data_as(C.POINTER(C.c_int64)),
                                len(r["pairs"]), r["size"])
        if e == "scatter":
            pairs = np.asarray(r["pairs"], dtype=np.int64).reshape(-1)
            d = _operand(P["d"], 0, r["d"])
            a = _operand(P["a"], 0, r["a"])
            return L.tpg_scatter(None, pairs.ctypes.data_as(C.POINTER(C.c_int64)),
                                 len(r["pairs"]), C.byref(d), C.byref(a), mode)
        if e == "scatter_fill":
            offs = np.asarray(r["offsets"], dtype=np.int64)
            v = bytes.fromhex(r["value"])
            return L.tpg_scatter_fill(None, offs.ctypes.data_as(C.POINTER(C.c_int64)), len(offs),
                                      P["d"], v, len(v))
        raise KeyError(e)


# ---------------------------------------------------------------------------
# comparison
# ---------------------------------------------------------------------------
def _decode(d, raw: bytes, order):
    return D.unpack_value(d, raw, 0, order)


def _ulp_dist(x: float, y: float, d) -> float:
    """distance in units of the last place of dtype d (real floats)."""
    if x == y:
        return 0.0
    if math.isnan(x) or math.isnan(y) or math.isinf(x) or math.isinf(y):
        return math.inf
    if d is D.HALF:
        ulp = 2.0 ** (max(math.frexp(max(abs(x), abs(y)))[1] - 11, -24))
    elif d is D.FLOAT:
        ulp = 2.0 ** (max(math.frexp(max(abs(x), abs(y)))[1] - 24, -149))
    else:
        ulp = math.ulp(max(abs(x), abs(y)))
    return abs(x - y) / ulp


def tolerance_class(r):
    """'exact' | ('ulp', n) | ('rel', tol) for the record's float results."""
    e, op = r["entry"], r.get("op")
    if e in ("copy", "fill", "arange", "byteswap", "gather", "scatter", "scatter_fill", "binary"):
        return "exact"
    if e == "unary":
        if dt(r["compute"]).is_complex or r.get("force_complex"):
            if op in ("negate", "conjugate"):
                return "exact"
            return ("rel", 1e-12)
        if op in ("negate", "absolute", "conjugate", "square_root"):
            return "exact"
        return ("ulp", 2)
    if e == "reduce":
        o = op.replace("reduce_", "")
        if o in ("minimum", "maximum", "any", "all"):
            return "exact"
        return ("rel", 1e-12)
    if e == "matmul":
        return ("rel", 1e-12)
    return "exact"


def compare(r, got: bytes, want: bytes, tol=None):
    """List of mismatch descriptions (empty = pass)."""
    if len(got) != len(want):
        return [f"length {len(got)} != {len(want)}"]
    d = dest_dtype(r)
    offs = dest_offsets(r)
    size = r["size"] if r["entry"] == "gather" else d.size
    mask = bytearray(len(want))
    for o in offs:
        mask[o:o + size] = b"\1" * size
    bad = []
    for i in range(len(want)):
        if not mask[i] and got[i] != want[i]:
            bad.append(f"untouched byte {i} changed")
            break
    tol = tol or tolerance_class(r)
    order = r["d"][1] if d is not None else "little"
    seen = set()
    for o in offs:
        if o in seen:
            continue
        seen.add(o)
        g, w = got[o:o + size], want[o:o + size]
        if g == w:
            continue
        if d is None or not d.is_float:
            bad.append(f"@{o}: {g.hex()} != {w.hex()}")
            continue
        gv, wv = _decode(d, g, order), _decode(d, w, order)
        if not _close(gv, wv, d, tol):
            bad.append(f"@{o}: {gv!r} != {wv!r} ({tol})")
    return bad


def _close(g, w, d, tol) -> bool:
    if isinstance(g, complex):
        rd = D.real_counterpart(d)
        if tol == "exact" or tol[0] == "ulp":
            return _close(g.real, w.real, rd, tol) and _close(g.imag, w.imag, rd, tol)
        scale = max(abs(w), 1e-300)
        if any(math.isnan(v) for v in (g.real, g.imag, w.real, w.imag)):
            return all(math.isnan(a) == math.isnan(b) for a, b in
                       ((g.real, w.real), (g.imag, w.imag)))
        if any(math.isinf(v) for v in (g.real, g.imag, w.real, w.imag)):
            return g == w
        return abs(g - w) <= tol[1] * scale + _ulp_floor(rd, scale)
    if math.isnan(g) and math.isnan(w):
        return True
    if tol == "exact":
        return g == w and math.copysign(1, g) == math.copysign(1, w)
    if tol[0] == "ulp":
        return _ulp_dist(g, w, d) <= tol[1]
    if math.isinf(g) or math.isinf(w) or math.isnan(g) or math.isnan(w):
        return g == w
    return abs(g - w) <= tol[1] * abs(w) or _ulp_dist(g, w, d) <= 1


def _ulp_floor(rd, scale):
    if rd is D.HALF:
        return scale * 2.0 ** -10
    if rd is D.FLOAT:
        return scale * 2.0 ** -23
    return 0.0
