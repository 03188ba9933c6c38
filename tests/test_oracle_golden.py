"""Pin the C oracle against the reference: every captured reference table
call (tests/golden/golden_table_calls.npz, made by make_golden.py from the
unmodified reference cpu table) replayed through oracle/tp_oracle.c must
reproduce the reference's destination bytes."""

from collections import Counter

import pytest

from golden_replay import HostBackend, compare, load_records


def _oracle_tol(r):
    # the oracle restates the reference loops with the same libm: exact,
    # except complex transcendentals (C99 <complex.h> vs CPython cmath)
    if r["entry"] == "unary" and r["op"] not in ("negate", "conjugate", "absolute") and (
            r["compute"].startswith("complex") or r.get("force_complex")):
        return ("rel", 1e-12)
    if r["entry"] == "unary" and r["op"] == "absolute" and r["compute"].startswith("complex"):
        return ("ulp", 1)
    return "exact"


def test_golden_file_covers_every_entry():
    meta, _ = load_records()
    kinds = Counter(r["entry"] for r in meta)
    for e in ("binary", "unary", "copy", "reduce", "matmul", "fill", "arange", "byteswap",
              "gather", "scatter", "scatter_fill"):
        assert kinds[e] > 0, e
    ops = {r["op"] for r in meta}
    assert len(ops) == 31  # every table key was exercised


@pytest.mark.parametrize("entry", ["binary", "unary", "copy", "reduce", "matmul", "fill",
                                   "arange", "byteswap", "gather", "scatter", "scatter_fill"])
def test_oracle_reproduces_reference(entry):
    meta, blobs = load_records()
    be = HostBackend()
    failures = []
    for i, r in enumerate(meta):
        if r["entry"] != entry:
            continue
        got, status = be.run(r, blobs)
        bad = compare(r, got, blobs[r["after"]], _oracle_tol(r))
        if bad:
            failures.append((i, r["op"], r.get("d"), r.get("a"), bad[:3]))
        want_flags = set(r.get("status", []))
        got_flags = {n for b, n in ((1, "domain-violation"), (2, "integer-division-by-zero"))
                     if status & b}
        if want_flags != got_flags:
            failures.append((i, r["op"], "flags", sorted(got_flags), sorted(want_flags)))
    assert not failures, failures[:10]
