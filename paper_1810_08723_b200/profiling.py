"""Per-op device timing through the function table (SURVEY.md §5 tracing).

The reference's tracing hook is `override_op` wrappers "that record
runtime or accumulate call statistics" (PAPER.md:107-109,
dispatch.py:51-62) plus the OpHandle call counters.  `profile()` wraps
every ("core", "gpu") entry with a pair of CUDA events recorded on the
stream the entry launches on, so the numbers are device time, not host
time; results are collected when the block exits.

    with tp.profiling.profile() as prof:
        tp.add(V, R)
        tp.reduce("sum", X)
    print(prof.table())          # op, calls, total / mean device us
"""

from __future__ import annotations

import ctypes as C
from collections import defaultdict

from . import _native, dispatch
from . import table as tb


class Profile:
    def __init__(self, module="core", device_type="gpu"):
        self.module, self.device_type = module, device_type
        self._restore = []
        self._pending = []  # (op, start event, end event)
        self.stats = defaultdict(lambda: [0, 0.0])  # op -> [calls, total ms]

    def _wrap(self, op):
        L = _native.lib()

        def wrapper(orig):
            def call(*args, **kw):
                st = tb.current_stream()
                h = st.handle if st is not None else None
                a, b = C.c_void_p(), C.c_void_p()
                _native.check(L.tpg_event_create(C.byref(a)), "event")
                _native.check(L.tpg_event_create(C.byref(b)), "event")
                L.tpg_event_record(a.value, h)
                try:
                    return orig(*args, **kw)
                finally:
                    L.tpg_event_record(b.value, h)
                    self._pending.append((op, a.value, b.value))
            return call
        return wrapper

    def __enter__(self):
        for op in dispatch.table_ops(self.module, self.device_type):
            self._restore.append(dispatch.override_op(self.module, self.device_type, op,
                                                      self._wrap(op)))
        return self

    def __exit__(self, *exc):
        for r in reversed(self._restore):
            r()
        self._restore.clear()
        self.collect()
        return False

    def collect(self):
        L = _native.lib()
        ms = C.c_float()
        for op, a, b in self._pending:
            _native.check(L.tpg_event_sync(b), "event sync")
            _native.check(L.tpg_event_elapsed(a, b, C.byref(ms)), "event elapsed")
            s = self.stats[op]
            s[0] += 1
            s[1] += ms.value
            L.tpg_event_destroy(a)
            L.tpg_event_destroy(b)
        self._pending.clear()

    def table(self) -> str:
        lines = [f"{'op':<16}{'calls':>8}{'total us':>14}{'mean us':>12}"]
        for op, (n, t) in sorted(self.stats.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"{op:<16}{n:>8}{t * 1e3:>14.1f}{t * 1e3 / n:>12.2f}")
        return "\n".join(lines)


def profile(module="core", device_type="gpu") -> Profile:
    return Profile(module, device_type)
