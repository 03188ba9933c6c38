"""Drop-in check: the UNMODIFIED reference `tidepool` (installed into
baseline/_ref by `pip install --target`) runs on the B200 through
tidepool_plugin.register(); programs on gpu0 must match the same programs
on the reference's own cpu device (the pattern of the reference's
tests/test_device_parity.py:17-57).  Skipped when baseline/_ref is absent."""

import math
import random
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def tp():
    if not (REF / "tidepool").exists():
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    import tidepool
    from paper_1810_08723_b200 import tidepool_plugin
    if not any(d.type.name == "gpu" for d in tidepool.devices.list_devices()):
        tidepool_plugin.register(tidepool, count=1)
    return tidepool


def _eq(x, y, rel=0.0):
    if isinstance(x, complex) or isinstance(y, complex):
        return _eq(complex(x).real, complex(y).real, rel) and _eq(complex(x).imag, complex(y).imag, rel)
    if isinstance(x, float) and isinstance(y, float):
        return (math.isnan(x) and math.isnan(y)) or x == y or abs(x - y) <= rel * abs(y)
    return x == y


def _program(tp, seed, device):
    tz = tp.tensors
    a = tp.tensor_create((4, 3), tp.double, device)
    b = tp.tensor_create((4, 3), tp.double, device)
    st = random.Random(seed)
    for t in (a, b):
        _, pack = tp.dtypes.codec(t.dtype, t.byteorder)
        buf = t.storage.view()
        for off in tz.iter_offsets(t):
            pack(buf, off, round(st.uniform(-4, 4), 3) or 1.0)
    trace = []
    c = tp.add(a, b)
    trace.append(c)
    tp.multiply(c, 2.0, dest=c)
    d = tp.subtract(c, tp.apply_index(c, (slice(None, None, -1), slice(None))))
    trace.append(d)
    e = tp.square_root(tp.absolute(d))
    trace.append(e)
    f = tp.reduce("sum", e, axes=(1,))
    trace.append(f)
    g = tp.matmul(tp.transpose(a), b)
    trace.append(g)
    h = tp.cast(g, tp.int16)
    trace.append(h)
    i = tp.reduce("maximum", tp.cast(a, tp.float))
    trace.append(i)
    # elementwise / cast / min-max results are bit-exact; compensated sums
    # and matmul accumulate in a different order (rel 1e-12)
    tol = [0.0, 0.0, 0.0, 1e-12, 1e-12, 0.0, 0.0]
    return [(t.dims, t.dtype.name, tz.read_values(t), r) for t, r in zip(trace, tol)]


def test_reference_programs_match_on_gpu(tp):
    gpu = tp.devices.by_name("gpu0")
    for seed in range(10):
        cpu_run = _program(tp, seed, tp.cpu())
        gpu_run = _program(tp, seed, gpu)
        for (cd, ct, cv, rel), (gd, gt, gv, _) in zip(cpu_run, gpu_run):
            assert cd == gd and ct == gt
            assert all(_eq(x, y, rel) for x, y in zip(cv, gv)), (seed, ct, cv, gv)


def test_cross_device_round_trip_and_table_counts(tp):
    gpu = tp.devices.by_name("gpu0")
    t = tp.from_nested([[1, 2], [3, 4]], tp.int32)
    there = tp.cast(t, device=gpu)
    assert there.device is gpu
    back = tp.cast(there, device=tp.cpu())
    assert tp.tensors.read_values(back) == [1, 3, 2, 4]
    stats = tp.dispatch.table_stats("core", "gpu")
    assert len(stats) == 31 and stats["copy"] >= 1


def test_descriptor_gather_replaces_pair_lists(tp):
    """gpu -> same-gpu raw gathers (clones, reshape copies) run through
    tpg_gather_plan instead of the reference's pair list, byte-exact."""
    gpu = tp.devices.by_name("gpu0")
    tz = tp.tensors
    assert getattr(tz._raw_gather, "reference", None) is not None
    t = tp.cast(tp.arange(24, tp.int16), device=gpu)
    v = tp.apply_index(tz.reshape(t, (4, 6)), (slice(None, None, -1), slice(1, None, 2)))
    before = tp.dispatch.table_stats("core", "gpu").get("gather", 0)
    c = tz.contiguous_clone(v)
    assert tp.dispatch.table_stats("core", "gpu").get("gather", 0) == before
    cpu_v = tp.apply_index(tz.reshape(tp.arange(24, tp.int16), (4, 6)),
                           (slice(None, None, -1), slice(1, None, 2)))
    assert tz.read_values(c) == tz.read_values(cpu_v)
    tp.byteswap(c)
    c2 = tz.contiguous_clone(c)
    assert c2.byteorder == "big" and tz.read_values(c2) == tz.read_values(cpu_v)


def _program2(tp, seed, device):
    """Mixed dtypes, byte order, reductions over each axis, casts: the
    reference's own pipeline (promotion, implicit casts, aliasing clones)
    with the gpu table underneath."""
    tz = tp.tensors
    st = random.Random(1000 + seed)
    dts = [tp.int8, tp.int16, tp.int32, tp.uint8, tp.float, tp.double, tp.half]
    out = []
    a = tp.tensor_create((5, 4), st.choice(dts), device)
    b = tp.tensor_create((5, 4), st.choice(dts), device)
    for t in (a, b):
        _, pack = tp.dtypes.codec(t.dtype, t.byteorder)
        buf = t.storage.view()
        for off in tz.iter_offsets(t):
            v = st.randint(-20, 20)
            if t.dtype is tp.uint8:
                v = abs(v)
            pack(buf, off, float(v) if t.dtype in (tp.float, tp.double, tp.half) else v)
    if st.random() < 0.5:
        tp.byteswap(b)
    out.append(tp.add(a, b))
    out.append(tp.multiply(tp.transpose(a), tp.transpose(b)))
    out.append(tp.maximum(a, tp.apply_index(b, (slice(None, None, -1), slice(None)))))
    out.append(tp.cast(tp.subtract(a, b), tp.int16))
    for op in ("sum", "minimum", "maximum"):
        for axes in ((0,), (1,), None):
            out.append(tp.reduce(op, a, axes=axes))
    out.append(tp.cast(a, tp.double))
    return [(t.dims, t.dtype.name, tz.read_values(t)) for t in out]


def test_reference_mixed_dtype_programs_match_on_gpu(tp):
    gpu = tp.devices.by_name("gpu0")
    for seed in range(15):
        for (cd, ct, cv), (gd, gt, gv) in zip(_program2(tp, seed, tp.cpu()),
                                              _program2(tp, seed, gpu)):
            assert cd == gd and ct == gt, (seed, ct, gt)
            assert all(_eq(x, y, 1e-12) for x, y in zip(cv, gv)), (seed, ct, cv, gv)
