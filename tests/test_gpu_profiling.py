"""Per-op device timing through override_op wrappers (the
reference's tracing hook, dispatch.py:51-62 / PAPER.md:107-109)."""

import numpy as np
import pytest

import paper_1810_08723_b200 as tp

pytestmark = pytest.mark.gpu


def test_profile_times_table_entries_on_device():
    X = tp.from_numpy(np.asfortranarray(np.random.default_rng(1).random((2048, 2048))))
    with tp.profiling.profile() as prof:
        Y = tp.add(X, 1.0)
        tp.reduce("sum", Y)
        tp.reduce("sum", Y, axes=(0,))
    assert prof.stats["add"][0] == 1 and prof.stats["sum"][0] == 2
    assert prof.stats["add"][1] > 0.0 and prof.stats["sum"][1] > 0.0
    assert "add" in prof.table()
    # wrappers are removed on exit
    tp.add(X, 1.0)
    assert prof.stats["add"][0] == 1
