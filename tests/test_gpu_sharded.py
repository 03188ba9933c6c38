"""Sharded full reductions on the device: local kernel partials + NCCL
all-reduce (world 1 on the test box; the multi-rank host logic is covered
with gloo in test_sharded_gloo.py)."""

import math

import numpy as np
import pytest

import paper_1810_08723_b200 as tp
from paper_1810_08723_b200.sharded import NcclComm, Sharded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = NcclComm(tp.gpu(0), 0, 1, lambda uid: uid)
    yield c
    c.close()


def test_sharded_full_reductions_match_single_device(comm):
    rng = np.random.default_rng(1)
    x = rng.random((512, 256))
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    T = tp.from_numpy(np.asfortranarray(x))
    assert S.reduce_full("sum", comm) == pytest.approx(tp.reduce("sum", T).item(), rel=1e-13)
    assert S.reduce_full("norm", comm) == pytest.approx(tp.reduce("norm", T).item(), rel=1e-13)
    assert S.reduce_full("maximum", comm) == tp.reduce("maximum", T).item()
    assert S.reduce_full("minimum", comm) == tp.reduce("minimum", T).item()


def test_nan_rules(comm):
    x = np.array([1.0, np.nan, 5.0, -2.0])
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    assert S.reduce_full("maximum", comm) == 5.0  # NaN not first: skipped
    y = np.array([np.nan, 1.0, 5.0])
    S2 = Sharded.from_numpy(y, 0, 1, tp.gpu(0))
    assert math.isnan(S2.reduce_full("maximum", comm))  # first element NaN


def test_sharded_map_is_local(comm):
    rng = np.random.default_rng(2)
    x = rng.random(1 << 16).astype(np.float32)
    S = Sharded.from_numpy(x, 0, 1, tp.gpu(0))
    out = S.map(lambda t, s: tp.multiply(t, s), tp.Scalar(1.5, tp.float))
    assert np.array_equal(tp.to_numpy(out.local), (x.astype(np.float64) * 1.5).astype(np.float32))
