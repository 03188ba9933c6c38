"""The drop-in: the UNMODIFIED reference `tidepool` with
tidepool_plugin.register() attached, on two backends:

* "fake" (CPU suite): a test double of the C ABI (tests/fake_native.py: host
  "device" memory, kernels run by the C oracle) - pins closure decoding,
  status / cast-loss / error routing into the reference's own state and
  exception classes, lazy casts, staging and descriptor transfers;
* "gpu" (-m gpu): libtidepool_gpu.so on the B200.

The reference is loaded from $TIDEPOOL_REF_PATH, baseline/_ref (travels to
the GPU box) or /root/reference/pkg/src; skipped when none exists."""

import gc
import math
import random

import pytest

import ref_loader
from fake_native import FakeNative


_ENVS = {}


@pytest.fixture(scope="module", params=["fake", pytest.param("gpu", marks=pytest.mark.gpu)])
def env(request):
    return _ENVS.get(request.param) or _make_env(request.param)


def _fill(tp, t, values):
    _, pack = tp.dtypes.codec(t.dtype, t.byteorder)
    buf = t.storage.view()
    for v, off in zip(values, tp.tensors.iter_offsets(t)):
        pack(buf, off, tp.dtypes.cast_scalar(v, t.dtype))


def _on(tp, gpu, nested, dtype):
    return tp.cast(tp.from_nested(nested, dtype), device=gpu)


def test_registration_shape(env):
    tp, gpu, fake, rt = env
    assert gpu.name == "gpu0" and tp.devices.by_name("gpu0") is gpu
    stats = tp.dispatch.table_stats("core", "gpu")
    assert len(set(stats) - {"ewise_chain", "matmul_batched"}) == 31   # + 2 extension entries
    assert gpu.properties["device-type"] == "gpu"


def test_int_division_by_zero_reaches_reference_status(env):
    """reference tests/test_ops.py:122-128 on gpu0."""
    tp, gpu, fake, rt = env
    tp.clear_status()
    out = tp.divide(_on(tp, gpu, [1, 7], tp.int32), _on(tp, gpu, [0, 2], tp.int32))
    assert tp.tensors.read_values(out) == [0, 3]
    assert tp.kernels.STATUS_INT_DIV_ZERO in tp.get_status()
    assert tp.kernels.STATUS_INT_DIV_ZERO in tp.ops._status  # the reference's own set
    tp.clear_status()
    assert tp.get_status() == frozenset()


def test_status_visible_without_an_explicit_sync(env):
    tp, gpu, fake, rt = env
    tp.clear_status()
    tp.square_root(_on(tp, gpu, [-1.0], tp.double))
    assert tp.kernels.STATUS_DOMAIN in tp.get_status()   # get_status drains gpu streams
    tp.clear_status()


def test_int_division_error_mode_raises_reference_class(env):
    """reference tests/test_ops.py:130-133."""
    tp, gpu, fake, rt = env
    with pytest.raises(tp.errors.DomainError):
        tp.divide(_on(tp, gpu, [1], tp.int32), _on(tp, gpu, [0], tp.int32), mode="error")


def test_cast_loss_error_mode_raises_before_writing(env):
    tp, gpu, fake, rt = env
    src = _on(tp, gpu, [1.0, 300.0, 2.0], tp.double)
    dst = tp.tensor_create((3,), tp.int8, gpu)
    tp.fill(dst, 5)
    with pytest.raises(tp.errors.DomainError):
        tp.copy(src, dst, mode="error")
    assert tp.tensors.read_values(dst) == [5, 5, 5]
    # the reference's own class: `except tidepool.DomainError` catches it
    with pytest.raises(tp.DomainError):
        tp.cast(src, tp.int8, mode="error")


def test_cast_loss_warning_mode_warns_once_through_reference_handler(env):
    tp, gpu, fake, rt = env
    seen = []
    prev = tp.set_warning_handler(seen.append)
    try:
        out = tp.cast(_on(tp, gpu, [1.0, 300.0, 400.0], tp.double), tp.int8, mode="warning")
        assert tp.tensors.read_values(out) == [1, 44, -112]
        assert len(seen) == 1
        tp.square_root(_on(tp, gpu, [-1.0, -2.0], tp.double), mode="warning")
        assert len(seen) == 2
    finally:
        tp.set_warning_handler(prev)


def test_reduce_and_matmul_error_mode(env):
    tp, gpu, fake, rt = env
    x = _on(tp, gpu, [100, 100, 100], tp.int8)
    with pytest.raises(tp.errors.DomainError):
        tp.reduce("sum", x, mode="error")
    assert tp.tensors.read_values(tp.reduce("sum", x)) == [44]
    m = _on(tp, gpu, [[100, 100], [100, 100]], tp.int8)
    with pytest.raises(tp.errors.DomainError):
        tp.matmul(m, m, mode="error")


def test_lazy_cast_fuses_into_the_binary_entry(env):
    """cfg2 shape family through the unmodified reference: the int16 ->
    float conversion of ops._dtype_convert is consumed by the add entry
    (one launch reading int16), and the result equals the cpu device's."""
    tp, gpu, fake, rt = env
    n = 24
    rng = random.Random(3)
    xs = [[rng.randint(-1000, 1000) for _ in range(n)] for _ in range(n)]
    row = [[rng.uniform(-1, 1) for _ in range(n)]]
    X = tp.from_nested(xs, tp.int16)
    R = tp.from_nested(row, tp.float)
    want = tp.add(tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None))), R)
    Xg, Rg = tp.cast(X, device=gpu), tp.cast(R, device=gpu)
    V = tp.apply_index(tp.transpose(Xg), (slice(None, None, -1), slice(None)))
    before = dict(rt.stats)
    out = tp.add(V, Rg)
    assert rt.stats["lazy"] == before.get("lazy", 0) + 1
    assert rt.stats["fused"] == before.get("fused", 0) + 1     # converted on load
    assert rt.stats["materialized"] == before.get("materialized", 0)
    if fake is not None:
        assert [c[0] for c in fake.calls[-1:]] == ["binary"]
        assert fake.calls[-1][2] == tp.int16.wire_code
    gc.collect()   # a record lives no longer than the reference's temporary
    assert all(p in rt.blocks for p in rt.lazy)
    assert tp.tensors.read_values(out) == tp.tensors.read_values(want)
    assert out.storage.snapshot() == want.storage.snapshot()


def test_lazy_cast_materialises_for_other_consumers_and_writers(env):
    tp, gpu, fake, rt = env
    x = _on(tp, gpu, [1, 2, 3, 4], tp.int16)
    y = tp.cast(x, tp.float)                  # recorded, not launched
    assert rt.lazy
    tp.fill(x, 9)                             # writing the source materialises first
    assert not rt.lazy
    assert tp.tensors.read_values(y) == [1.0, 2.0, 3.0, 4.0]
    y2 = tp.cast(x, tp.double)
    assert tp.reduce("sum", y2).item() == 36.0  # reduction consumer materialises
    y3 = tp.cast(x, tp.int32)
    assert tp.tensors.read_values(y3) == [9, 9, 9, 9]  # host read: sync materialises


def test_destination_aliasing_inplace_equals_copy_first(env):
    """reference tests/test_ops.py:177-219 on gpu0."""
    tp, gpu, fake, rt = env
    rng = random.Random(223)
    for _ in range(5):
        vals = [round(rng.uniform(-8, 8), 3) for _ in range(16)]
        base = tp.tensor_create((4, 4), tp.double, gpu)
        _fill(tp, base, vals)
        a = tp.apply_index(base, (slice(None, None, -1), slice(None)))
        b = tp.apply_index(base, (slice(0, 4), slice(None)))
        want = [x + y for x, y in zip(tp.tensors.read_values(a), tp.tensors.read_values(b))]
        tp.add(a, b, dest=a)
        assert tp.tensors.read_values(a) == want
    m = tp.cast(tp.reshape(tp.arange(4), (2, 2)), device=gpu)
    tp.matmul(m, m, dest=m)
    assert tp.tensors.read_values(m) == [2.0, 3.0, 6.0, 11.0]


def test_transfers_are_descriptor_based_and_byte_exact(env):
    tp, gpu, fake, rt = env
    t = tp.from_nested([[1.5, -2.25, 3.0], [4.0, 5.5, -6.0]], tp.double)
    tp.byteswap(t)
    s0 = dict(rt.stats)
    g = tp.cast(t, device=gpu)                   # host source staged for the copy entry
    assert g.byteorder == "little"
    assert rt.stats["staged"] == s0.get("staged", 0) + 1
    back = tp.cast(g, tp.float, device=tp.cpu())  # cpu `copy` override: GPU convert + one D2H
    assert rt.stats["cpu_copy_from_gpu"] == s0.get("cpu_copy_from_gpu", 0) + 1
    assert tp.tensors.read_values(back) == [1.5, 4.0, -2.25, 5.5, 3.0, -6.0]
    # byte-order-preserving transfers ride _raw_gather (tensors.py:686-699)
    moved = tp.ops._device_transfer(t, gpu)
    assert moved.byteorder == "big"
    assert rt.stats["gather_plan"] == s0.get("gather_plan", 0) + 1
    home = tp.ops._device_transfer(moved, tp.cpu())
    assert rt.stats["gather_to_host"] == s0.get("gather_to_host", 0) + 1
    assert home.storage.snapshot() == t.storage.snapshot()


def _program(tp, seed, device):
    st = random.Random(seed)
    dts = [tp.int8, tp.int16, tp.int32, tp.uint8, tp.float, tp.double, tp.half]
    a = tp.tensor_create((5, 4), st.choice(dts), device)
    b = tp.tensor_create((5, 4), st.choice(dts), device)
    for t in (a, b):
        _fill(tp, t, [abs(v) if t.dtype is tp.uint8 else v
                      for v in (st.randint(-20, 20) for _ in range(20))])
    if st.random() < 0.5:
        tp.byteswap(b)
    out = [tp.add(a, b), tp.multiply(tp.transpose(a), tp.transpose(b)),
           tp.maximum(a, tp.apply_index(b, (slice(None, None, -1), slice(None)))),
           tp.cast(tp.subtract(a, b), tp.int16), tp.divide(a, tp.add(b, 1))]
    for op in ("sum", "minimum", "maximum", "norm"):
        for axes in ((0,), (1,), None):
            out.append(tp.reduce(op, a, axes=axes))
    out.append(tp.matmul(tp.cast(a, tp.double), tp.transpose(tp.cast(b, tp.double))))
    return [(t.dims, t.dtype.name, tp.tensors.read_values(t)) for t in out]


def _eq(x, y, rel):
    if isinstance(x, float) and isinstance(y, float):
        return (math.isnan(x) and math.isnan(y)) or x == y or abs(x - y) <= rel * abs(y)
    return x == y


def test_mixed_dtype_programs_match_cpu_device(env):
    tp, gpu, fake, rt = env
    for seed in range(12):
        for (cd, ct, cv), (gd, gt, gv) in zip(_program(tp, seed, tp.cpu()),
                                              _program(tp, seed, gpu)):
            assert cd == gd and ct == gt, (seed, ct, gt)
            assert all(_eq(x, y, 1e-12) for x, y in zip(cv, gv)), (seed, ct, cv, gv)
    gc.collect()
    assert all(p in rt.blocks for p in rt.lazy)


def test_fuse_strides_mapping():
    from paper_1810_08723_b200.tidepool_plugin import _fuse_strides, _is_dense

    class P:
        def __init__(self, e, s):
            self.extents, self.strides = e, s
    copy = P((4096, 4096), [(4, 16384), (-8192, 2)])
    assert _fuse_strides(copy, (4096, 4096), (4, 16384), 0, 4) == ([-8192, 2], 0)
    assert _fuse_strides(copy, (4096, 4096), (16384, 4), 0, 4) == ([2, -8192], 0)
    assert _fuse_strides(copy, (4096,), (0,), 0, 4) == ([0], 0)
    assert _fuse_strides(copy, (2048, 4096), (8, 16384), 0, 4) is None   # split axis
    assert _fuse_strides(copy, (4096,), (4,), 16384, 4) == ([-8192], 2)  # column 1
    assert _fuse_strides(copy, (4096,), (16384,), 4, 4) == ([2], -8192)  # row 1
    assert _is_dense((4, 3), (8, 32), 8) and not _is_dense((4, 3), (8, 40), 8)


def _from_numpy(tp, arr, device):
    """Column-major numpy array -> reference tensor on `device` (bytes
    written straight into the storage, as the reference's own raw_write)."""
    dt = {"int16": tp.int16, "float32": tp.float, "float64": tp.double}[arr.dtype.name]
    t = tp.tensor_create(arr.shape, dt, device)
    t.storage.stream.sync()
    t.storage.view()[:] = arr.tobytes(order="F")
    return t


@pytest.mark.gpu
def test_cfg2_full_size_through_the_unmodified_reference():
    """BASELINE cfg2 at its stated size through `tidepool.add` on gpu0: one
    fused launch (lazy int16 -> float cast consumed on load), bit-exact."""
    import numpy as np
    tp, gpu, fake, rt = _gpu_env()
    rng = np.random.default_rng(3)
    x16 = rng.integers(-1000, 1001, (4096, 4096)).astype(np.int16)
    r = np.random.default_rng(4).standard_normal((1, 4096)).astype(np.float32)
    X, R = _from_numpy(tp, x16, gpu), _from_numpy(tp, r, gpu)
    V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
    s0 = dict(rt.stats)
    out = tp.add(V, R)
    assert rt.stats["fused"] == s0.get("fused", 0) + 1
    got = np.frombuffer(out.storage.snapshot(), dtype=np.float32).reshape((4096, 4096), order="F")
    want = x16.T[::-1, :].astype(np.float32) + r
    assert np.array_equal(got, want)


def _gpu_env():
    return _ENVS.get("gpu") or _make_env("gpu")


def _make_env(kind):
    tp = ref_loader.load(f"tidepool_{kind}_plugin")
    if tp is None:
        pytest.skip("reference tidepool not found")
    from paper_1810_08723_b200 import tidepool_plugin
    lib = None
    if kind == "fake":
        from oracle import oracle
        lib = FakeNative(oracle.lib())
    devs = tidepool_plugin.register(tp, count=1, lib=lib)
    _ENVS[kind] = (tp, devs[0], lib, tidepool_plugin.register.runtime)
    return _ENVS[kind]


def test_chain_extension_matches_sequential_reference_ops(env):
    """`tidepool_plugin.chain` (the `ewise_chain` extension entry, added with
    the reference's dispatch.add_op) equals the reference's own ops run one
    after another, byte for byte, on the cpu device and on gpu0."""
    tp, gpu, fake, rt = env
    from paper_1810_08723_b200 import tidepool_plugin as plug
    rng = random.Random(17)
    cases = [
        (tp.float, [round(rng.uniform(-1e3, 1e3), 4) for _ in range(257)],
         [("multiply", tp.Scalar(1.5, tp.float)), ("add", tp.Scalar(-2.0, tp.float))]),
        (tp.int16, [rng.randint(-30000, 30000) for _ in range(129)],
         [("multiply", 3), ("subtract", tp.Scalar(7, tp.int16), True)]),
        (tp.double, [rng.uniform(-5, 5) for _ in range(64)],
         [("divide", 3.0), ("maximum", 0.25), ("minimum", 1.0)]),
    ]
    for dt, vals, steps in cases:
        x = tp.from_nested(vals, dt)
        want = x
        for st in steps:
            s = st[1]
            want = getattr(tp, st[0])(s, want) if len(st) > 2 and st[2] else \
                getattr(tp, st[0])(want, s)
        got = plug.chain(tp.cast(x, device=gpu), steps)
        assert got.dtype is want.dtype, (dt, got.dtype, want.dtype)
        assert got.storage.snapshot() == want.storage.snapshot(), dt


def test_matmul_batched_extension_matches_reference_slices(env):
    tp, gpu, fake, rt = env
    from paper_1810_08723_b200 import tidepool_plugin as plug
    rng = random.Random(5)
    m, k, n, nb = 6, 5, 4, 3
    a = tp.tensor_create((m, k, nb), tp.double)
    b = tp.tensor_create((k, n, nb), tp.double)
    _fill(tp, a, [rng.uniform(-1, 1) for _ in range(m * k * nb)])
    _fill(tp, b, [rng.uniform(-1, 1) for _ in range(k * n * nb)])
    got = plug.matmul_batched(tp.cast(a, device=gpu), tp.cast(b, device=gpu))
    assert got.dims == (m, n, nb) and got.device is gpu
    for q in range(nb):
        want = tp.matmul(tp.apply_index(a, (slice(None), slice(None), q)),
                         tp.apply_index(b, (slice(None), slice(None), q)))
        gq = tp.apply_index(got, (slice(None), slice(None), q))
        assert all(_eq(x, y, 1e-12) for x, y in zip(tp.tensors.read_values(gq),
                                                   tp.tensors.read_values(want))), q


def test_c_entry_fast_paths_match_the_python_entries(env):
    """The C fast paths of the binary and lazy-copy entries
    (hostsrc/tpg_pyfast.c) take the standard all-gpu calls and hand every
    other call (error mode, profiling) to the Python entries before any side
    effect; on random mixed-dtype / broadcast / reversed programs both paths
    produce the same bytes as the cpu device."""
    tp, gpu, fake, rt = env
    rng = random.Random(29)
    dts = [tp.int8, tp.int16, tp.uint16, tp.int32, tp.float, tp.double, tp.half]
    ops = ["add", "subtract", "multiply", "minimum", "maximum"]
    c0 = rt.entries.counts()
    for it in range(24):
        da, db = rng.choice(dts), rng.choice(dts)
        r, c = rng.randint(1, 9), rng.randint(1, 9)
        xa = [[rng.randint(-50, 50) for _ in range(c)] for _ in range(r)]
        xb = [[rng.randint(-50, 50) for _ in range(c)]]  # broadcast row
        A, B = tp.from_nested(xa, da), tp.from_nested(xb, db)
        if rng.random() < 0.5:
            A = tp.apply_index(A, (slice(None, None, -1), slice(None)))
        op = getattr(tp, rng.choice(ops))
        want = op(A, B)
        Ag, Bg = tp.cast(A, device=gpu), tp.cast(B, device=gpu)
        got_fast = op(Ag, Bg)
        rt.profile = []          # profiling forces the Python entries
        try:
            got_py = op(Ag, Bg)
        finally:
            rt.profile = None
        assert tp.tensors.read_values(got_fast) == tp.tensors.read_values(want), it
        assert got_fast.storage.snapshot() == want.storage.snapshot(), it
        assert got_py.storage.snapshot() == want.storage.snapshot(), it
    for it in range(12):   # unary entries (kind 2)
        d = rng.choice([tp.float, tp.double, tp.int16, tp.half])
        n = rng.randint(1, 30)
        name = rng.choice(["negate", "absolute", "square_root", "exponential", "sine"])
        lo = 0 if name == "square_root" else -20   # (NaN payloads are not compared bytewise)
        xs = [rng.randint(lo, 20) for _ in range(n)]
        A = tp.from_nested(xs, d)
        op = getattr(tp, name)
        want = op(A)
        Ag = tp.cast(A, device=gpu)
        got_fast = op(Ag)
        rt.profile = []
        try:
            got_py = op(Ag)
        finally:
            rt.profile = None
        assert got_fast.storage.snapshot() == want.storage.snapshot(), (it, op)
        assert got_py.storage.snapshot() == want.storage.snapshot(), (it, op)
    for it in range(10):   # reduction entries (kinds 3 / 4)
        d = rng.choice([tp.float, tp.double, tp.int32])
        r, c = rng.randint(1, 7), rng.randint(1, 7)
        A = tp.from_nested([[rng.randint(-9, 9) for _ in range(c)] for _ in range(r)], d)
        name = rng.choice(["sum", "maximum", "minimum", "norm"])
        axes = rng.choice([None, (0,), (1,)])
        want = tp.reduce(name, A, axes=axes)
        Ag = tp.cast(A, device=gpu)
        f0 = rt.entries.counts()["fast"]
        got_fast = tp.reduce(name, Ag, axes=axes)
        assert rt.entries.counts()["fast"] > f0, (it, name)
        rt.profile = []
        try:
            got_py = tp.reduce(name, Ag, axes=axes)
        finally:
            rt.profile = None
        assert tp.tensors.read_values(got_fast) == tp.tensors.read_values(want), (it, name)
        assert tp.tensors.read_values(got_py) == tp.tensors.read_values(want), (it, name)
    c1 = rt.entries.counts()
    assert c1["fast"] > c0["fast"]
    # error mode goes to the Python entry (CastContext semantics live there)
    x = _on(tp, gpu, [100, 100], tp.int8)
    before = rt.entries.counts()["fallback"]
    with pytest.raises(tp.errors.DomainError):
        tp.add(x, x, mode="error")
    assert rt.entries.counts()["fallback"] > before


def test_threads_share_the_drop_in(env):
    """Several Python threads run reference ops on gpu0 at once (the C entry
    paths, the lazy-cast records and the block pool are shared state under
    the GIL; a recycled block waits for its last GPU use): every result
    equals the cpu device's."""
    import threading
    tp, gpu, fake, rt = env
    errors = []

    def worker(seed):
        try:
            rng = random.Random(seed)
            for it in range(15):
                n = rng.randint(1, 40)
                xs = [[rng.randint(-99, 99) for _ in range(n)] for _ in range(3)]
                row = [[rng.uniform(-2, 2) for _ in range(n)]]
                X, R = tp.from_nested(xs, tp.int16), tp.from_nested(row, tp.float)
                want = tp.multiply(tp.add(X, R), R)
                Xg, Rg = tp.cast(X, device=gpu), tp.cast(R, device=gpu)
                got = tp.multiply(tp.add(Xg, Rg), Rg)
                if got.storage.snapshot() != want.storage.snapshot():
                    errors.append((seed, it))
        except Exception as exc:  # noqa: BLE001 - reported below
            errors.append((seed, repr(exc)))
    ts = [threading.Thread(target=worker, args=(s,)) for s in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:3]


@pytest.mark.gpu
def test_recycled_blocks_wait_for_their_last_gpu_use():
    """The block pool hands a freed block out again only after the GPU work
    that last used it completed (completion words / events): fresh storages
    written by the host right after dropping results of in-flight 64 MiB
    kernels keep exactly the host's bytes."""
    import numpy as np
    tp, gpu, fake, rt = _gpu_env()
    n = 4096
    X = tp.tensor_create((n, n), tp.int16, gpu)
    R = tp.tensor_create((1, n), tp.float, gpu)
    gpu.default_stream().sync()
    X.storage.view()[:] = np.arange(n * n, dtype=np.int16).tobytes()
    R.storage.view()[:] = np.ones(n, dtype=np.float32).tobytes()
    V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))
    stats0 = rt.pool.stats()
    for i in range(24):
        out = tp.add(V, R)          # 64 MiB result written by an in-flight kernel
        del out                     # block back to the pool while the kernel may still run
        fresh = tp.tensor_create((n, n), tp.float, gpu)
        pattern = np.full(n * n, float(i) + 0.5, dtype=np.float32)
        fresh.storage.view()[:] = pattern.tobytes()   # host write, no sync
        gpu.default_stream().sync()
        got = np.frombuffer(fresh.storage.snapshot(), dtype=np.float32)
        assert np.array_equal(got, pattern), i
        del fresh
    assert rt.pool.stats()["reused"] > stats0["reused"]


def test_block_pool_falls_back_to_events_without_stream_memory_ops():
    """Where tpg_stream_mark is unavailable the block pool records CUDA
    events instead of completion words; blocks are still recycled and every
    result equals the cpu device's (CPU test double, marks failing)."""
    tp = ref_loader.load("tidepool_events_plugin")
    if tp is None:
        pytest.skip("reference tidepool not found")
    from oracle import oracle

    from paper_1810_08723_b200 import tidepool_plugin
    fake = FakeNative(oracle.lib())
    fake.fail_marks = True
    records = []
    real_record = fake.tpg_event_record
    fake.tpg_event_record = lambda ev, s: (records.append(ev), real_record(ev, s))[1]
    gpu = tidepool_plugin.register(tp, count=1, lib=fake)[0]
    rt = tidepool_plugin.register.runtime
    rng = random.Random(41)
    for it in range(40):
        xs = [[rng.randint(-50, 50) for _ in range(6)] for _ in range(5)]
        X, R = tp.from_nested(xs, tp.int16), tp.from_nested([[1.5] * 6], tp.float)
        want = tp.add(X, R)
        got = tp.add(tp.cast(X, device=gpu), tp.cast(R, device=gpu))
        assert got.storage.snapshot() == want.storage.snapshot(), it
    st = rt.pool.stats()
    assert st["reused"] > 0 and st["released"] > 0
    assert records   # the markers were CUDA events


def test_c_host_path_does_not_leak(env):
    """Reference counts of the C entries (hostsrc/tpg_pyfast.c): repeated
    cfg2-shaped adds (lazy cast fused), unaries, reductions and lazy casts
    leave the interpreter's allocated-block count flat
    (scripts/plugin_leak_probe.py is the long version)."""
    import sys
    tp, gpu, fake, rt = env
    X = _on(tp, gpu, [[i - 8 for i in range(16)] for _ in range(16)], tp.int16)
    R = _on(tp, gpu, [[0.5 * i for i in range(16)]], tp.float)
    V = tp.apply_index(tp.transpose(X), (slice(None, None, -1), slice(None)))

    def rounds(n):
        for _ in range(n):
            tp.add(V, R)
            tp.negate(R)
            tp.reduce("sum", R)
            tp.cast(V, tp.float)
            if fake is not None:
                fake.calls.clear()  # the test double's own launch log
        gpu.default_stream().sync()
        gc.collect()
        return sys.getallocatedblocks()
    rounds(300)
    b0 = rounds(1000)
    b1 = rounds(3000)
    assert b1 - b0 < 100, (b0, b1)
