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
floats, which the reference code consumes unchanged; errors (raised, or
returned per slot by batch_search) are re-issued as the reference's own
exception classes (ente.exceptions) with the same messages.
"""

from __future__ import annotations

import importlib

from . import engine as _engine
from . import ksg as _ksg

def _translate(exc):
    """The reference's exception of the same name (ente.exceptions), same message:
    callers of the reference test `isinstance(e, ente.exceptions.KTooLarge)`."""
    from . import exceptions as ours
    if isinstance(exc, ours.EnteError):
        ref = importlib.import_module("ente.exceptions")
        cls = getattr(ref, type(exc).__name__, None)
        if cls is not None:
            out = cls(*exc.args)
            out.__cause__ = exc
            return out
    return exc


def _wrap(fn, slots=False):
    """Call fn; translate raised errors (and, for batch_search, per-slot ones)."""
    import functools

    @functools.wraps(fn)
    def call(*args, **kwargs):
        try:
            out = fn(*args, **kwargs)
        except Exception as exc:  # noqa: BLE001 - re-raised as the reference's type
            tr = _translate(exc)
            if tr is exc:
                raise
            raise tr from exc
        if slots:
            out = [_translate(r) if isinstance(r, Exception) else r for r in out]
        return out
    return call


_PATCHES = {
    "ente.engine": {"batch_search": _wrap(_engine.batch_search, slots=True),
                    "knn_kth_distances": _wrap(_engine.knn_kth_distances),
                    "radius_counts": _wrap(_engine.radius_counts)},
    "ente.ksg": {"batch_search": _wrap(_engine.batch_search, slots=True),
                 "estimate_te_batch": _wrap(_ksg.estimate_te_batch),
                 "estimate_te": _wrap(_ksg.estimate_te)},
    "ente.bench": {"batch_search": _wrap(_engine.batch_search, slots=True)},
    "ente.inference": {"estimate_te_batch": _wrap(_ksg.estimate_te_batch)},
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
