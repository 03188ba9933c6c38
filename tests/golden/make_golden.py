"""Generate golden vectors by running the REFERENCE tidepool cpu table.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py  [--ref /root/reference/pkg/src]

Every call the reference pipeline makes into its ("core", "cpu") function
table is intercepted with dispatch.override_op (the reference's own
instrumentation hook, dispatch.py:135-137).  For each call we record the
decoded descriptors (plan, bases, operand dtypes / byte orders, store dtype
/ mode, op, compute dtype), the bytes of every input buffer before the
call and the destination buffer after it, plus the sticky status flags it
raised.  tests/test_oracle_golden.py replays the records through the C
oracle (CPU) and tests/test_gpu_golden.py through libtidepool_gpu (GPU).
"""

from __future__ import annotations

import argparse
import io
import json
import math
import os
import random
import struct
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from paper_1810_08723_b200.tidepool_plugin import (decode_codec, decode_store,  # noqa: E402
                                                   norm_order, prime_codecs,
                                                   unary_forces_complex)

SEED = 20261017


class Recorder:
    def __init__(self, tp):
        self.tp = tp
        self.records = []
        self.blobs = []
        self.enabled = True

    def blob(self, b: bytes) -> int:
        self.blobs.append(bytes(b))
        return len(self.blobs) - 1

    def bufs(self, named):
        """named: list of (role, memoryview); dedupe identical buffers."""
        ids, out = {}, {}
        for role, mv in named:
            if mv is None:
                continue
            key = id(mv.obj) if isinstance(mv, memoryview) else id(mv)
            if key not in ids:
                ids[key] = f"buf{len(ids)}"
                out[ids[key]] = self.blob(bytes(mv))
            out[role] = ids[key]
        return out, ids

    def install(self):
        tp, dispatch, dt = self.tp, self.tp.dispatch, self.tp.dtypes
        prime_codecs(dt)
        rec = self

        def key_of(mv):
            return id(mv.obj) if isinstance(mv, memoryview) else id(mv)

        def wrap(op):
            def wrapper(orig):
                def call(*args):
                    if not rec.enabled:
                        return orig(*args)
                    r = rec.capture(op, args)
                    tp.ops._status.clear()
                    out = orig(*args)
                    if r is not None:
                        dbuf = r.pop("_dbuf")
                        r["after"] = rec.blob(bytes(dbuf))
                        r["status"] = sorted(tp.ops._status)
                        rec.records.append(r)
                    return out
                return call
            return wrapper

        for op in dispatch.table_stats("core", "cpu"):
            dispatch.override_op("core", "cpu", op, wrap(op))
        self.key_of = key_of

    def capture(self, op, args):
        tp, dt = self.tp, self.tp.dtypes
        binary = ("add", "subtract", "multiply", "divide", "minimum", "maximum")
        unary = ("negate", "absolute", "square_root", "exponential", "logarithm", "sine",
                 "cosine", "arcsine", "arccosine", "conjugate", "copy")
        reduce_ = ("sum", "product", "reduce_minimum", "reduce_maximum", "any", "all", "norm")
        r = {"op": op}
        if op in binary:
            plan, d_buf, store, a_buf, a_unpack, b_buf, b_unpack, fn, bases = args
            sd, so, mode = decode_store(dt, store)
            ad, ao = decode_codec(dt, a_unpack)
            bd, bo = decode_codec(dt, b_unpack)
            bufs, _ = self.bufs([("d", d_buf), ("a", a_buf), ("b", b_buf)])
            r.update(entry="binary", ext=list(plan.extents), str=[list(s) for s in plan.strides],
                     bases=list(bases), d=[sd, so], a=[ad, ao], b=[bd, bo], mode=mode,
                     compute=dt.widen_for_compute(dt.by_name(ad)).name, bufs=bufs)
            r["_dbuf"] = d_buf
        elif op in unary:
            plan, d_buf, store, a_buf, a_unpack, fn, bases = args
            sd, so, mode = decode_store(dt, store)
            ad, ao = decode_codec(dt, a_unpack)
            bufs, _ = self.bufs([("d", d_buf), ("a", a_buf)])
            fc = op != "copy" and unary_forces_complex(fn) and not dt.by_name(ad).is_complex
            r.update(entry="copy" if op == "copy" else "unary", ext=list(plan.extents),
                     str=[list(s) for s in plan.strides], bases=list(bases), d=[sd, so],
                     a=[ad, ao], mode=mode, compute=dt.widen_for_compute(dt.by_name(ad)).name,
                     force_complex=bool(fc), bufs=bufs)
            r["_dbuf"] = d_buf
        elif op in reduce_:
            outer, inner, d_buf, store, a_buf, a_unpack, init, step, fin, bases = args
            sd, so, mode = decode_store(dt, store)
            ad, ao = decode_codec(dt, a_unpack)
            bufs, _ = self.bufs([("d", d_buf), ("a", a_buf)])
            r.update(entry="reduce", oext=list(outer.extents), ostr=[list(s) for s in outer.strides],
                     iext=list(inner.extents), istr=[list(s) for s in inner.strides],
                     bases=list(bases), d=[sd, so], a=[ad, ao], mode=mode,
                     p=norm_order(step) if op == "norm" else 2.0, bufs=bufs)
            r["_dbuf"] = d_buf
        elif op == "matmul":
            (d_buf, d_base, d_str, store, a_buf, a_base, a_str, a_unpack, b_buf, b_base, b_str,
             b_unpack, m, n, k, mul, init, step, fin) = args
            sd, so, mode = decode_store(dt, store)
            ad, ao = decode_codec(dt, a_unpack)
            bd, bo = decode_codec(dt, b_unpack)
            bufs, _ = self.bufs([("d", d_buf), ("a", a_buf), ("b", b_buf)])
            r.update(entry="matmul", d=[sd, so], a=[ad, ao], b=[bd, bo], mode=mode,
                     bases=[d_base, a_base, b_base], dstr=list(d_str), astr=list(a_str),
                     bstr=list(b_str), m=m, n=n, k=k,
                     compute=dt.widen_for_compute(dt.by_name(ad)).name, bufs=bufs)
            r["_dbuf"] = d_buf
        elif op == "fill":
            plan, buf, pack, value, base = args
            name, order = decode_codec(dt, pack)
            tmp = bytearray(dt.by_name(name).size)
            pack(tmp, 0, value)
            bufs, _ = self.bufs([("d", buf)])
            r.update(entry="fill", ext=list(plan.extents), str=[list(s) for s in plan.strides],
                     bases=[base], d=[name, order], value=tmp.hex(), bufs=bufs)
            r["_dbuf"] = buf
        elif op == "arange":
            plan, buf, pack, cast_fn, base = args
            name, order = decode_codec(dt, pack)
            bufs, _ = self.bufs([("d", buf)])
            r.update(entry="arange", ext=list(plan.extents), str=[list(s) for s in plan.strides],
                     bases=[base], d=[name, order], bufs=bufs)
            r["_dbuf"] = buf
        elif op == "byteswap":
            buf, base, plan, dtype = args
            bufs, _ = self.bufs([("d", buf)])
            r.update(entry="byteswap", ext=list(plan.extents), str=[list(s) for s in plan.strides],
                     bases=[base], d=[dtype.name, "little"], bufs=bufs)
            r["_dbuf"] = buf
        elif op == "gather":
            dst_buf, src_buf, pairs, size = args
            bufs, _ = self.bufs([("d", dst_buf), ("a", src_buf)])
            r.update(entry="gather", pairs=[list(p) for p in pairs], size=size, bufs=bufs)
            r["_dbuf"] = dst_buf
        elif op == "scatter":
            pairs, d_buf, store, s_buf, s_unpack = args
            sd, so, mode = decode_store(dt, store)
            ad, ao = decode_codec(dt, s_unpack)
            bufs, _ = self.bufs([("d", d_buf), ("a", s_buf)])
            r.update(entry="scatter", pairs=[list(p) for p in pairs], d=[sd, so], a=[ad, ao],
                     mode=mode, bufs=bufs)
            r["_dbuf"] = d_buf
        elif op == "scatter_fill":
            offsets, d_buf, pack, value = args
            name, order = decode_codec(dt, pack)
            tmp = bytearray(dt.by_name(name).size)
            pack(tmp, 0, value)
            bufs, _ = self.bufs([("d", d_buf)])
            r.update(entry="scatter_fill", offsets=list(offsets), d=[name, order],
                     value=tmp.hex(), bufs=bufs)
            r["_dbuf"] = d_buf
        else:
            return None
        return r


# ---------------------------------------------------------------------------
# value / view generators (edge-heavy)
# ---------------------------------------------------------------------------
def edge_value(rng, d, tp):
    dt = tp.dtypes
    if d is dt.BOOL:
        return rng.random() < 0.5
    if d.is_complex:
        return complex(edge_value(rng, dt.real_counterpart(d), tp),
                       edge_value(rng, dt.real_counterpart(d), tp))
    if d.is_float:
        r = rng.random()
        if r < 0.06:
            return rng.choice([math.nan, math.inf, -math.inf, -0.0, 0.0])
        if r < 0.12:
            return dt.cast_scalar(rng.choice([65504.0, 65520.0, 2049.0, 1e20, -1e20, 3e38,
                                              16777217.0, 1e-8, -300.7, 2.5, -2.5, 0.5]), d)
        return dt.cast_scalar(round(rng.uniform(-300, 300), rng.choice([0, 1, 3, 6])), d)
    lo, hi = dt.int_range(d)
    r = rng.random()
    if r < 0.15:
        return rng.choice([lo, hi, 0, 1, -1 if lo < 0 else 0, hi - 1])
    return rng.randint(max(lo, -1000), min(hi, 1000))


def fill_tensor(t, rng, tp):
    _, pack = tp.dtypes.codec(t.dtype, t.byteorder)
    buf = t.storage.view()
    for off in tp.tensors.iter_offsets(t):
        pack(buf, off, tp.dtypes.cast_scalar(edge_value(rng, t.dtype, tp), t.dtype))


def random_view(rng, base, tp):
    parts = []
    for d in base.dims:
        c = rng.random()
        if c < 0.2 and d > 0:
            s = rng.randrange(d)
            parts.append(slice(s, s + 1))
        elif c < 0.6:
            step = rng.choice([1, 2, -1, -2])
            parts.append(slice(None, None, step))
        else:
            parts.append(slice(None))
    v = tp.apply_index(base, tuple(parts))
    if v.ndim > 1 and rng.random() < 0.5:
        order = list(range(v.ndim))
        rng.shuffle(order)
        v = tp.permute_axes(v, order)
    return v


def random_tensor(rng, tp, dtype=None, max_axes=3, max_extent=5, min_axes=0):
    dt = tp.dtypes
    dtype = dtype or rng.choice(dt.ALL_DTYPES)
    dims = tuple(rng.randint(1, max_extent) for _ in range(rng.randint(min_axes, max_axes)))
    base = tp.tensor_create(dims, dtype)
    fill_tensor(base, rng, tp)
    v = random_view(rng, base, tp)
    if rng.random() < 0.25:
        tp.byteswap(v)
    return v


# ---------------------------------------------------------------------------
def generate(tp, rec: Recorder):
    rng = random.Random(SEED)
    dt = tp.dtypes
    ALL = dt.ALL_DTYPES
    BIN = ("add", "subtract", "multiply", "divide", "minimum", "maximum")
    UN = ("negate", "absolute", "square_root", "exponential", "logarithm", "sine", "cosine",
          "arcsine", "arccosine", "conjugate")

    # 1. copy/cast over every dtype pair and byte order (with edge values)
    for sd in ALL:
        for dd in ALL:
            for swap in (False, True):
                src = random_tensor(rng, tp, sd, max_axes=2, max_extent=6, min_axes=1)
                if swap and src.byteorder == "little":
                    tp.byteswap(src)
                tp.cast(src, dd)
    # big-endian destination
    for sd in ALL:
        src = random_tensor(rng, tp, sd, max_axes=2, max_extent=5, min_axes=1)
        dst = tp.tensor_create(src.dims, rng.choice(ALL))
        tp.byteswap(dst)
        tp.copy(src, dst)

    # 2. binary: random dtype pairs, strided / broadcast / byteswapped operands
    cases = 0
    while cases < 700:
        a = random_tensor(rng, tp, max_axes=3, max_extent=4)
        b = random_tensor(rng, tp, max_axes=3, max_extent=4)
        try:
            tp.tensors.broadcast_result_dims(a.dims, b.dims)
        except tp.ShapeError:
            continue
        op = rng.choice(BIN)
        try:
            getattr(tp, op)(a, b)
        except (tp.TidepoolError, ZeroDivisionError, OverflowError, ValueError):
            pass
        cases += 1
    # same-dtype binary for every dtype and op (no implicit copy)
    for d in ALL:
        for op in BIN:
            a = random_tensor(rng, tp, d, max_axes=2, max_extent=5, min_axes=1)
            b = random_tensor(rng, tp, d, max_axes=2, max_extent=5, min_axes=1)
            b = tp.tensor_create(a.dims, d)
            fill_tensor(b, rng, tp)
            try:
                getattr(tp, op)(a, b)
            except (tp.TidepoolError, ZeroDivisionError, OverflowError, ValueError):
                pass
    # scalars (materialized 0-dim operands) and mixed-precision promotion
    for _ in range(60):
        a = random_tensor(rng, tp, max_axes=2, max_extent=5, min_axes=1)
        s = rng.choice([2, -3, 1.5, -0.25, 2.0 + 1.0j, True, 1e10])
        op = rng.choice(BIN)
        try:
            getattr(tp, op)(a, s) if rng.random() < 0.5 else getattr(tp, op)(s, a)
        except (tp.TidepoolError, ZeroDivisionError, OverflowError, ValueError):
            pass
    # integer division by zero and INT_MIN / -1
    for d in (dt.INT8, dt.INT32, dt.INT64, dt.UINT64, dt.BOOL):
        lo, hi = dt.int_range(d) if d is not dt.BOOL else (0, 1)
        a = tp.from_nested([lo, hi, 7, -7 if lo < 0 else 7, 0], d)
        b = tp.from_nested([-1 if lo < 0 else 1, 0, 2, -2 if lo < 0 else 3, 0], d)
        tp.divide(a, b)
    # cast-on-write destinations (f32 + f32 into int32 etc.)
    for _ in range(40):
        a = random_tensor(rng, tp, dt.FLOAT, max_axes=1, max_extent=6, min_axes=1)
        dst = tp.tensor_create(a.dims, rng.choice(ALL))
        try:
            tp.add(a, a, dest=dst)
        except tp.TidepoolError:
            pass

    # 3. unary: every op x dtype, standard mode; a few warning / complex mode
    for op in UN:
        for d in ALL:
            a = random_tensor(rng, tp, d, max_axes=2, max_extent=5, min_axes=1)
            if op in ("sine", "cosine") and d.is_float and not d.is_complex:
                # math.sin(inf) raises ValueError in the reference; keep finite
                a = tp.tensor_create(a.dims, d)
                for off in tp.tensors.iter_offsets(a):
                    _, pack = dt.codec(d, a.byteorder)
                    pack(a.storage.view(), off, dt.cast_scalar(rng.uniform(-50, 50), d))
            try:
                getattr(tp, op)(a)
            except (tp.TidepoolError, ValueError, OverflowError, ZeroDivisionError):
                pass
    for op in ("square_root", "logarithm", "arcsine", "arccosine"):
        for d in (dt.FLOAT, dt.DOUBLE, dt.HALF):
            a = tp.from_nested([-2.0, -0.5, 0.0, 0.25, 4.0], d)
            getattr(tp, op)(a, mode="complex")

    # 4. reductions: every op x dtype x axes choice
    RED = ("sum", "product", "minimum", "maximum", "any", "all", "norm")
    for op in RED:
        for d in ALL:
            for _ in range(3):
                a = random_tensor(rng, tp, d, max_axes=3, max_extent=5, min_axes=1)
                if op in ("minimum", "maximum") and d.is_complex:
                    pass
                axes = None if rng.random() < 0.3 else tuple(
                    sorted(rng.sample(range(a.ndim), rng.randint(1, a.ndim))))
                p = rng.choice([2.0, 1.0, 3.0]) if op == "norm" else 2.0
                try:
                    tp.reduce(op, a, axes=axes, p=p)
                except (tp.TidepoolError, TypeError, ValueError, OverflowError):
                    pass
    # longer sums (compensation matters) and NaN-first min/max
    for d in (dt.FLOAT, dt.DOUBLE, dt.HALF):
        base = tp.tensor_create((1000,), d)
        _, pack = dt.codec(d, "little")
        for off in tp.tensors.iter_offsets(base):
            pack(base.storage.view(), off, dt.cast_scalar(rng.uniform(-1, 1) * 10 ** rng.randint(-3, 3), d))
        tp.reduce("sum", base)
        tp.reduce("norm", base)
    for d in (dt.FLOAT, dt.DOUBLE):
        tp.reduce("minimum", tp.from_nested([math.nan, 1.0, -2.0], d))
        tp.reduce("maximum", tp.from_nested([1.0, math.nan, -2.0], d))
        tp.reduce("maximum", tp.from_nested([0.0, -0.0], d))
        tp.reduce("minimum", tp.from_nested([-0.0, 0.0], d))
    tp.reduce("sum", tp.from_nested([16777216.0, 1.0, 1.0], dt.FLOAT))

    # 5. matmul: every dtype, transposed / strided operands
    for d in ALL:
        for _ in range(3):
            m, n, k = rng.randint(1, 7), rng.randint(1, 7), rng.randint(0, 9)
            A = tp.tensor_create((k, m) if rng.random() < 0.5 else (m, k), d)
            fill_tensor(A, rng, tp)
            if A.dims != (m, k):
                A = tp.transpose(A)
            B = tp.tensor_create((k, n), d)
            fill_tensor(B, rng, tp)
            try:
                tp.matmul(A, B)
            except (tp.TidepoolError, OverflowError, ValueError):
                pass
    for _ in range(20):
        da, db = rng.choice(ALL), rng.choice(ALL)
        A = tp.tensor_create((3, 4), da)
        B = tp.tensor_create((4, 2), db)
        fill_tensor(A, rng, tp)
        fill_tensor(B, rng, tp)
        try:
            tp.matmul(A, B)
        except (tp.TidepoolError, OverflowError, ValueError):
            pass

    # 6. fill / arange / byteswap / gather / scatter
    for d in ALL:
        t = tp.tensor_create((3, 4), d)
        tp.fill(random_view(rng, t, tp), edge_value(rng, d, tp))
        tp.arange(rng.randint(0, 40), d)
        v = random_tensor(rng, tp, d, max_axes=2, max_extent=5, min_axes=1)
        tp.byteswap(v)
        tp.tensors.contiguous_clone(v)
        # advanced assignment -> scatter / scatter_fill
        t2 = tp.tensor_create((6,), d)
        tp.fill(t2, 0)
        src = tp.tensor_create((3,), rng.choice(ALL))
        fill_tensor(src, rng, tp)
        try:
            tp.assign_index(t2, ([0, 2, 2],), src)
            tp.assign_index(t2, ([1, 3],), edge_value(rng, d, tp))
        except (tp.TidepoolError, OverflowError, ValueError):
            pass


def save(rec: Recorder, path: Path):
    lens = [len(b) for b in rec.blobs]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    blob = np.frombuffer(b"".join(rec.blobs), dtype=np.uint8)
    meta = json.dumps(rec.records, separators=(",", ":"))
    np.savez_compressed(path, meta=np.frombuffer(meta.encode(), dtype=np.uint8),
                        blob=blob, offs=offs)


def host_semantics(tp) -> dict:
    """Promotion lattice, compute/container dtypes, scalar casts and
    canonical plans as the reference computes them (host-side logic)."""
    dt = tp.dtypes
    rng = random.Random(SEED + 1)
    out = {"promote": {}, "widen": {}, "float_container": {}, "cast": [], "plans": []}
    for a in dt.ALL_DTYPES:
        out["widen"][a.name] = dt.widen_for_compute(a).name
        out["float_container"][a.name] = dt.float_container(a).name
        for b in dt.ALL_DTYPES:
            out["promote"][f"{a.name},{b.name}"] = dt.promote(a, b).name
    vals = [0, 1, -1, 255, 256, 130, -300, 2 ** 40 + 3, -(2 ** 63), 2 ** 64 - 1, 2 ** 70,
            1.9, -1.9, -300.7, 2049.0, 65520.0, 65504.0, 1e20, -1e20, 3.5e38, 16777217.0,
            1152921573326323713, True, False, 1.5 + 2j, 3 + 0j, 0.1]
    for v in vals:
        for d in dt.ALL_DTYPES:
            try:
                r = dt.cast_scalar(v, d)
            except (tp.TidepoolError, OverflowError) as exc:
                r = f"error:{type(exc).__name__}"
            out["cast"].append([repr(v), d.name, repr(r)])
    for _ in range(300):
        nd = rng.randint(0, 5)
        dims = [rng.choice([0, 1, 1, 2, 3, 4, 5]) if rng.random() < 0.1 else rng.randint(1, 5)
                for _ in range(nd)]
        nv = rng.randint(1, 3)
        views = []
        for _ in range(nv):
            if rng.random() < 0.5:
                st, step = [], rng.choice([1, 2, 4, 8])
                order = list(range(nd))
                rng.shuffle(order)
                strides = [0] * nd
                for k in order:
                    strides[k] = step * rng.choice([1, 1, 1, -1]) * (0 if rng.random() < 0.1 else 1)
                    step *= max(dims[k], 1)
                views.append(strides)
            else:
                views.append([rng.choice([-16, -8, -4, 0, 2, 4, 8, 24, 64]) for _ in range(nd)])
        plan = tp.tensors.build_plan(tuple(dims), [tuple(v) for v in views])
        out["plans"].append([dims, views, list(plan.extents), [list(s) for s in plan.strides]])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default=os.environ.get("TIDEPOOL_REF_PATH", "/root/reference/pkg/src"))
    ap.add_argument("--out", default=str(HERE / "golden_table_calls.npz"))
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import tidepool as tp
    rec = Recorder(tp)
    rec.install()
    generate(tp, rec)
    rec.enabled = False
    save(rec, Path(args.out))
    (HERE / "host_semantics.json").write_text(json.dumps(host_semantics(tp), indent=0))
    from collections import Counter
    print(len(rec.records), "records;", sum(len(b) for b in rec.blobs), "bytes")
    print(Counter(r["entry"] for r in rec.records))


if __name__ == "__main__":
    main()
