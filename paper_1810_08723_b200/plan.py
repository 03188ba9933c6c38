"""Stride-descriptor layer: canonical iteration plans.

Restates the reference IterPlan / build_plan / canonicalize
(pkg/src/tidepool/tensors.py:533-604): drop extent-1 axes, order the axes
by |stride| of view 0 (the destination; ties keep axis order), merge axis
k+1 into k when stride[k+1] == stride[k] * extent[k] holds for every view,
and represent an empty iteration as the single axis (0,).  Plans are
handed to the C ABI as a fixed-size `tpg_plan` (abi.Plan).
"""

from __future__ import annotations

import math

from . import abi

MAX_DIMS = 8


class IterPlan:
    __slots__ = ("extents", "strides", "total", "_c")

    def __init__(self, extents, strides):
        self.extents = tuple(extents)
        self.strides = [tuple(s) for s in strides]
        self.total = math.prod(self.extents)
        self._c = None

    def to_c(self) -> abi.Plan:
        if self._c is None:
            self._c = abi.make_plan(self.extents, self.strides)
        return self._c

    def offsets(self, bases):
        """Byte offsets per view in plan order (host-side helper)."""
        nv = len(self.strides)
        offs = list(bases)
        if not self.extents:
            yield tuple(offs)
            return
        idx = [0] * len(self.extents)
        for _ in range(self.total):
            yield tuple(offs)
            for k, e in enumerate(self.extents):
                idx[k] += 1
                for v in range(nv):
                    offs[v] += self.strides[v][k]
                if idx[k] < e:
                    break
                idx[k] = 0
                for v in range(nv):
                    offs[v] -= self.strides[v][k] * e

    def __repr__(self):
        return f"IterPlan({self.extents}, {self.strides})"


def build_plan(dims, strides_per_view) -> IterPlan:
    nviews = len(strides_per_view)
    if math.prod(dims) == 0:
        return IterPlan((0,), [(0,)] * nviews)
    lead = strides_per_view[0]
    axes = sorted((k for k, d in enumerate(dims) if d != 1), key=lambda k: (abs(lead[k]), k))
    ext: list[int] = []
    strd: list[list[int]] = [[] for _ in range(nviews)]
    for k in axes:
        if ext and all(strides_per_view[v][k] == strd[v][-1] * ext[-1] for v in range(nviews)):
            ext[-1] *= dims[k]
            continue
        ext.append(dims[k])
        for v in range(nviews):
            strd[v].append(strides_per_view[v][k])
    return IterPlan(ext, strd)


def canonicalize(*views) -> IterPlan:
    dims = views[0].dims
    for v in views[1:]:
        if v.dims != dims:
            from .errors import ShapeError
            raise ShapeError(f"canonicalize needs equal dims, got {v.dims} vs {dims}")
    return build_plan(dims, [v.strides for v in views])
