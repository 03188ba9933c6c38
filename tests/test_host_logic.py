"""CPU checks of the host-side mirror against reference-generated fixtures
(tests/golden/host_semantics.json): promotion lattice, compute dtypes,
scalar casts and canonical plans, plus registry / dispatch behaviour."""

import json
import math
from pathlib import Path

import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200 import dispatch, dtypes as D
from paper_1810_08723_b200.errors import (ImplNotLoadedError, ModuleRegistryError,
                                          OpNotProvidedError)
from paper_1810_08723_b200.plan import build_plan

SEM = json.loads((Path(__file__).parent / "golden" / "host_semantics.json").read_text())


def test_promotion_table_matches_reference():
    for key, want in SEM["promote"].items():
        a, b = key.split(",")
        assert D.promote(D.by_name(a), D.by_name(b)).name == want, key


def test_widen_and_float_container_match_reference():
    for a, want in SEM["widen"].items():
        assert D.widen_for_compute(D.by_name(a)).name == want
    for a, want in SEM["float_container"].items():
        assert D.float_container(D.by_name(a)).name == want


def _same(x, y):
    if isinstance(x, float) and isinstance(y, float):
        return (math.isnan(x) and math.isnan(y)) or (x == y and math.copysign(1, x) == math.copysign(1, y))
    if isinstance(x, complex) and isinstance(y, complex):
        return _same(x.real, y.real) and _same(x.imag, y.imag)
    return x == y and type(x) is type(y)


def test_cast_scalar_matches_reference():
    inf, nan = math.inf, math.nan  # noqa: F841 (eval namespace)
    for v, d, want in SEM["cast"]:
        value = eval(v)
        if want.startswith("error:"):
            with pytest.raises(Exception):
                D.cast_scalar(value, D.by_name(d))
            continue
        got = D.cast_scalar(value, D.by_name(d))
        assert _same(got, eval(want)), (v, d, got, want)


def test_build_plan_matches_reference():
    for dims, views, ext, strides in SEM["plans"]:
        p = build_plan(tuple(dims), [tuple(v) for v in views])
        assert list(p.extents) == ext and [list(s) for s in p.strides] == strides, (dims, views)


def test_core_table_has_all_31_reference_keys():
    ops = dispatch.table_ops("core", "gpu")
    assert len(set(ops) - {"ewise_chain", "matmul_batched"}) == 31   # + 2 extension entries
    for k in ("add", "copy", "sum", "reduce_minimum", "reduce_maximum", "norm", "matmul",
              "fill", "arange", "byteswap", "gather", "scatter", "scatter_fill"):
        assert k in ops


def test_lookup_error_codes():
    with pytest.raises(ImplNotLoadedError) as e:
        dispatch.lookup("core", "tpu", "add")
    assert e.value.code == "impl-not-loaded"
    with pytest.raises(OpNotProvidedError) as e:
        dispatch.lookup("core", "gpu", "fft")
    assert e.value.code == "op-not-provided"
    with pytest.raises(ModuleRegistryError):
        dispatch.register_device_impl("core", "gpu", {})


def test_override_counts_and_restores():
    h = dispatch.lookup("core", "gpu", "add")
    fn0 = h.fn
    calls = []
    restore = dispatch.override_op("core", "gpu", "add",
                                   lambda orig: (lambda *a: calls.append(len(a))))
    before = h.call_count
    h(1, 2, 3)
    assert calls == [3] and h.call_count == before + 1
    restore()
    assert h.fn is fn0


def test_scalar_packing_roundtrip():
    for d in D.ALL_DTYPES:
        for v in (0, 1, 3):
            c = D.cast_scalar(v, d)
            raw = D.pack_value(d, c, "big")
            assert _same(D.unpack_value(d, raw, 0, "big"), c)
