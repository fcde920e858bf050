"""Stage the reference package for the GPU box (test infrastructure only).

The reference (`ente`, /root/reference/pkg) is pure Python + numba, so there
is nothing to compile into oracle/_ref; what travels is the package source
and its test suite, zipped from where they lie by stage() (run by
__graft_entry__.build() in the container that has /root/reference; the zip
is git-ignored and never committed).  On the GPU box extract() unpacks it to
a scratch directory for

  * tests/test_reference_suite.py: the reference's own fast tests run
    against this package through paper_1401_4068_b200.shim.install();
  * bench.py --impl reference and the cpu_baseline leg: the unmodified
    reference CPU path (numba, all host threads) timed beside ours.

Nothing on the product path imports this module.
"""

from __future__ import annotations

import json
import os
import tempfile
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
ZIP = os.path.join(HERE, "_ref", "ente_ref.zip")


def stage(ref_pkg: str = REF_PKG, out: str = ZIP) -> str | None:
    """Zip <ref_pkg>/src/ente and <ref_pkg>/tests into oracle/_ref/ente_ref.zip."""
    if not os.path.isdir(os.path.join(ref_pkg, "src", "ente")):
        return None
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + ".tmp"
    meta = {"source": ref_pkg}
    try:
        import numba
        import numpy
        import scipy
        meta.update(numpy=numpy.__version__, scipy=scipy.__version__, numba=numba.__version__)
    except ImportError:  # pragma: no cover
        pass
    with zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as z:
        for sub in ("src/ente", "tests"):
            base = os.path.join(ref_pkg, sub)
            for name in sorted(os.listdir(base)):
                if name.endswith(".py"):
                    with open(os.path.join(base, name), "rb") as f:  # (source mtimes predate 1980)
                        z.writestr(zipfile.ZipInfo(f"{sub}/{name}", (1980, 1, 1, 0, 0, 0)),
                                   f.read(), zipfile.ZIP_DEFLATED)
        z.writestr("STAGED.json", json.dumps(meta))
    os.replace(tmp, out)
    return out


def available() -> bool:
    return os.path.exists(ZIP)


def extract(dest: str | None = None) -> str | None:
    """Unpack the staged reference; returns the root holding src/ and tests/."""
    if not available():
        return None
    root = dest or tempfile.mkdtemp(prefix="ente_ref_")
    with zipfile.ZipFile(ZIP) as z:
        z.extractall(root)
    return root


def import_reference(dest: str | None = None):
    """Import the staged reference package `ente` (numba cache in the scratch dir)."""
    import sys
    root = extract(dest)
    if root is None:
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(root, "numba_cache"))
    src = os.path.join(root, "src")
    if src not in sys.path:
        sys.path.insert(0, src)
    import ente
    return ente


if __name__ == "__main__":
    print(stage())
