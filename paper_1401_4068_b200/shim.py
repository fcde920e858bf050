"""Route an imported reference package `ente` through the B200 path.

The reference binds its engine and estimator by name at import time
(/root/reference/pkg/src/ente/ksg.py:14 `from .engine import batch_search`,
bench.py:20, inference.py:24 `from .ksg import estimate_te_batch`), so
patching `ente.engine` alone would change nothing.  install() rebinds every
call site listed in SURVEY.md 8(b):

    ente.engine.batch_search / knn_kth_distances / radius_counts
    ente.ksg.batch_search, ente.ksg.estimate_te_batch, ente.ksg.estimate_te
    ente.bench.batch_search
    ente.inference.estimate_te_batch

Inputs are the reference's own objects (Chunk, PointSetBundle, numpy seeds);
the replacements read only their public attributes (`points`, `joint`,
`n_rows`, `dims`), so they take reference objects as they are.  Results come
back as this package's NeighborCounts (same fields, same dtypes) and plain
floats, which the reference code consumes unchanged.
"""

from __future__ import annotations

import importlib

from . import engine as _engine
from . import ksg as _ksg

_PATCHES = {
    "ente.engine": {"batch_search": _engine.batch_search,
                    "knn_kth_distances": _engine.knn_kth_distances,
                    "radius_counts": _engine.radius_counts},
    "ente.ksg": {"batch_search": _engine.batch_search,
                 "estimate_te_batch": _ksg.estimate_te_batch,
                 "estimate_te": _ksg.estimate_te},
    "ente.bench": {"batch_search": _engine.batch_search},
    "ente.inference": {"estimate_te_batch": _ksg.estimate_te_batch},
}


def install() -> dict:
    """Patch the imported `ente` modules; returns the originals for uninstall()."""
    saved = {}
    for modname, names in _PATCHES.items():
        mod = importlib.import_module(modname)
        for name, fn in names.items():
            if hasattr(mod, name):
                saved[(modname, name)] = getattr(mod, name)
                setattr(mod, name, fn)
    return saved


def uninstall(saved: dict) -> None:
    for (modname, name), fn in saved.items():
        setattr(importlib.import_module(modname), name, fn)
