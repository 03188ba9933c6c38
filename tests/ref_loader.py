"""Locate and load the UNMODIFIED reference `tidepool` package (test helper).

Search order: $TIDEPOOL_REF_PATH, baseline/_ref (the pip --target install
that travels to the GPU box), /root/reference/pkg/src (this container only).
`load(alias)` imports an independent copy under another top-level name, so
several tests can register devices without sharing the reference's global
registries.
"""

from __future__ import annotations

import importlib.util
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def reference_dir() -> Path | None:
    cands = []
    if os.environ.get("TIDEPOOL_REF_PATH"):
        cands.append(Path(os.environ["TIDEPOOL_REF_PATH"]))
    cands += [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]
    for c in cands:
        if (c / "tidepool" / "__init__.py").exists():
            return c / "tidepool"
    return None


def load(alias: str):
    pkg = reference_dir()
    if pkg is None:
        return None
    if alias in sys.modules:
        return sys.modules[alias]
    spec = importlib.util.spec_from_file_location(alias, pkg / "__init__.py",
                                                  submodule_search_locations=[str(pkg)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[alias] = mod
    spec.loader.exec_module(mod)
    return mod
