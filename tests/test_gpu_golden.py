"""GPU parity gate: every captured reference table call replayed through
libtidepool_gpu's C ABI must reproduce the reference's destination bytes.

Tolerances (golden_replay.tolerance_class): bit-exact for copy/astype,
fill, arange, byteswap, gather/scatter and all binary ops (NaN payloads
compared as NaN, the reference's own rule, tests/conftest.py:86-92); real
transcendentals <= 2 ulp (CUDA libdevice vs glibc); reductions and matmul
on floats rel 1e-12 (f64; f16/f32 results within 1 ulp); complex
transcendentals rel 1e-12.  Status flags must match exactly.
"""

import pytest

from golden_replay import GpuBackend, compare, load_records

ENTRIES = ["binary", "unary", "copy", "reduce", "matmul", "fill", "arange", "byteswap",
           "gather", "scatter", "scatter_fill"]


@pytest.mark.gpu
@pytest.mark.parametrize("entry", ENTRIES)
def test_gpu_reproduces_reference(entry):
    meta, blobs = load_records()
    be = GpuBackend()
    failures = []
    for i, r in enumerate(meta):
        if r["entry"] != entry:
            continue
        got, status = be.run(r, blobs)
        bad = compare(r, got, blobs[r["after"]])
        if bad:
            failures.append((i, r["op"], r.get("d"), r.get("a"), r.get("b"), bad[:3]))
        want = set(r.get("status", []))
        have = {n for b, n in ((1, "domain-violation"), (2, "integer-division-by-zero"))
                if status & b}
        if want != have:
            failures.append((i, r["op"], "flags", sorted(have), sorted(want)))
    assert not failures, f"{len(failures)} mismatches: {failures[:8]}"
