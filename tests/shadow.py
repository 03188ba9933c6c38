"""Shadow oracle: check every ("core","gpu") table call made by the gpu
pipeline against the C oracle on host copies of the same buffers.

Inside `with ShadowOracle() as so:` each table entry call snapshots its
input storages, runs on the GPU, snapshots the destination, replays the
same descriptors through oracle/tp_oracle.c and records mismatches.
"""

from __future__ import annotations

from paper_1810_08723_b200 import dispatch

from golden_replay import HostBackend, compare


class ShadowOracle:
    def __init__(self, tol=None, max_bytes=1 << 28):
        self.tol = tol
        self.max_bytes = max_bytes
        self.failures = []
        self.calls = 0
        self._restore = []
        self.host = HostBackend()

    def __enter__(self):
        for op in dispatch.table_ops("core", "gpu"):
            self._restore.append(dispatch.override_op("core", "gpu", op, self._wrap(op)))
        return self

    def __exit__(self, *exc):
        for r in reversed(self._restore):
            r()
        return False

    def _wrap(self, op):
        def wrapper(orig):
            def call(*args):
                rec, blobs, dkey = self._capture(op, args)
                out = orig(*args)
                if rec is not None:
                    d_buf = self._dbuf(op, args)
                    d_buf.stream.sync()
                    got = d_buf.snapshot()
                    want, _ = self.host.run(rec, blobs)
                    bad = compare(rec, got, want, self.tol)
                    self.calls += 1
                    if bad:
                        self.failures.append((op, rec.get("d"), rec.get("a"), rec.get("b"),
                                              bad[:3]))
                return out
            return call
        return wrapper

    @staticmethod
    def _dbuf(op, args):
        if op in ("matmul", "byteswap"):
            return args[0]
        if op in ("sum", "product", "reduce_minimum", "reduce_maximum", "any", "all", "norm"):
            return args[2]
        return args[1]

    def _capture(self, op, args):
        blobs, bufs, ids = [], {}, {}

        def add(role, buf, imm=None):
            if buf is None:
                blobs.append(bytes(imm).ljust(16, b"\0"))
                key = f"buf{len(ids)}"
                ids[("imm", role)] = key
                bufs[key] = len(blobs) - 1
                bufs[role] = key
                return
            if buf.nbytes > self.max_bytes:
                raise OverflowError
            k = id(buf)
            if k not in ids:
                buf.stream.sync()
                blobs.append(buf.snapshot())
                ids[k] = f"buf{len(ids)}"
                bufs[ids[k]] = len(blobs) - 1
            bufs[role] = ids[k]

        try:
            if op in ("add", "subtract", "multiply", "divide", "minimum", "maximum"):
                plan, d_buf, store, a_buf, ac, b_buf, bc, fn, bases = args
                add("d", d_buf)
                add("a", a_buf, ac.imm)
                add("b", b_buf, bc.imm)
                rec = dict(entry="binary", op=op, ext=list(plan.extents),
                           str=[list(s) for s in plan.strides],
                           bases=[bases[0], bases[1] if a_buf else 0, bases[2] if b_buf else 0],
                           d=[store.dtype.name, store.byteorder], a=[ac.dtype.name, ac.byteorder],
                           b=[bc.dtype.name, bc.byteorder], mode=store.mode,
                           compute=fn.compute.name, bufs=bufs)
            elif op in ("negate", "absolute", "square_root", "exponential", "logarithm", "sine",
                        "cosine", "arcsine", "arccosine", "conjugate", "copy"):
                plan, d_buf, store, a_buf, ac, fn, bases = args
                add("d", d_buf)
                add("a", a_buf, ac.imm)
                rec = dict(entry="copy" if op == "copy" else "unary", op=op,
                           ext=list(plan.extents), str=[list(s) for s in plan.strides],
                           bases=list(bases), d=[store.dtype.name, store.byteorder],
                           a=[ac.dtype.name, ac.byteorder], mode=store.mode,
                           compute=(ac.dtype.name if fn is None else fn.compute.name),
                           force_complex=bool(fn is not None and fn.force_complex), bufs=bufs)
            elif op in ("sum", "product", "reduce_minimum", "reduce_maximum", "any", "all",
                        "norm"):
                outer, inner, d_buf, store, a_buf, ac, acc, _, _, bases = args
                add("d", d_buf)
                add("a", a_buf)
                rec = dict(entry="reduce", op=op, oext=list(outer.extents),
                           ostr=[list(s) for s in outer.strides], iext=list(inner.extents),
                           istr=[list(s) for s in inner.strides], bases=list(bases),
                           d=[store.dtype.name, store.byteorder], a=[ac.dtype.name, ac.byteorder],
                           mode=store.mode, p=acc.p, bufs=bufs)
            elif op == "matmul":
                (d_buf, d_base, d_str, store, a_buf, a_base, a_str, ac, b_buf, b_base, b_str, bc,
                 m, n, k, mul, *_r) = args
                add("d", d_buf)
                add("a", a_buf)
                add("b", b_buf)
                rec = dict(entry="matmul", op=op, d=[store.dtype.name, store.byteorder],
                           a=[ac.dtype.name, ac.byteorder], b=[bc.dtype.name, bc.byteorder],
                           mode=store.mode, bases=[d_base, a_base, b_base], dstr=list(d_str),
                           astr=list(a_str), bstr=list(b_str), m=m, n=n, k=k,
                           compute=mul.compute.name, bufs=bufs)
            elif op == "fill":
                plan, buf, pack, value, base = args
                add("d", buf)
                from paper_1810_08723_b200 import dtypes as D
                rec = dict(entry="fill", op=op, ext=list(plan.extents),
                           str=[list(s) for s in plan.strides], bases=[base],
                           d=[pack.dtype.name, pack.byteorder],
                           value=D.pack_value(pack.dtype, value, pack.byteorder).hex(), bufs=bufs)
            elif op == "arange":
                plan, buf, pack, _c, base = args
                add("d", buf)
                rec = dict(entry="arange", op=op, ext=list(plan.extents),
                           str=[list(s) for s in plan.strides], bases=[base],
                           d=[pack.dtype.name, pack.byteorder], bufs=bufs)
            elif op == "byteswap":
                buf, base, plan, dtype = args[:4]
                add("d", buf)
                rec = dict(entry="byteswap", op=op, ext=list(plan.extents),
                           str=[list(s) for s in plan.strides], bases=[base],
                           d=[dtype.name, "little"], bufs=bufs)
            else:
                return None, None, None
        except OverflowError:
            return None, None, None
        return rec, blobs, None
