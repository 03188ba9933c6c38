"""Public async host <-> device transfer API used by the end-to-end path."""

import numpy as np
import pytest

import paper_1810_08723_b200 as tp

pytestmark = pytest.mark.gpu


def test_pinned_upload_download_slabs():
    n = 512
    x = np.asfortranarray(np.random.default_rng(1).integers(-999, 999, (n, n)).astype(np.int16))
    X = tp.tensor_create((n, n), tp.int16)
    hx = tp.pinned((n, n), np.int16)
    hx[...] = x
    s = tp.gpu(0).create_stream()
    for c0 in range(0, n, 128):                       # column slabs: contiguous runs
        tp.upload(hx[:, c0:c0 + 128], tp.apply_index(X, (slice(None), slice(c0, c0 + 128))), s)
    s.sync()
    assert np.array_equal(tp.to_numpy(X), x)
    out = tp.pinned((n, n), np.int16)
    out[...] = 0
    for r0 in range(0, n, 64):                        # row slabs: pitched on both sides
        tp.download(tp.apply_index(X, (slice(r0, r0 + 64), slice(None))), out[r0:r0 + 64, :], s)
    s.sync()
    assert np.array_equal(out, x)
    with pytest.raises(tp.ShapeError):
        tp.download(tp.transpose(X), out, s)          # neither a run nor a slab
