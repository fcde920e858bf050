"""shim.install() rebinds the reference's call sites and speaks its exception types.

CPU-only: the checks below stop at argument validation, before any device
work (the full reference suite through the shim runs on the GPU in
tests/test_reference_suite.py).  The reference package comes from
oracle/_ref (staged by __graft_entry__.build(), oracle/ref_stage.py).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref_stage  # noqa: E402


@pytest.fixture(scope="module")
def ente(tmp_path_factory):
    if not ref_stage.available():
        pytest.skip("reference not staged (oracle/_ref/ente_ref.zip)")
    mod = ref_stage.import_reference(str(tmp_path_factory.mktemp("ref")))
    from paper_1401_4068_b200 import shim
    saved = shim.install()
    yield mod
    shim.uninstall(saved)


def test_install_rebinds_every_call_site(ente):
    import ente.bench
    import ente.engine
    import ente.inference
    import ente.ksg
    for mod, name in [(ente.engine, "batch_search"), (ente.engine, "knn_kth_distances"),
                      (ente.engine, "radius_counts"), (ente.ksg, "batch_search"),
                      (ente.ksg, "estimate_te_batch"), (ente.ksg, "estimate_te"),
                      (ente.bench, "batch_search"), (ente.inference, "estimate_te_batch")]:
        fn = getattr(mod, name)
        assert fn.__wrapped__.__module__.startswith("paper_1401_4068_b200"), (mod, name)


def test_errors_are_the_references_types(ente):
    import ente.engine
    import ente.exceptions as ex
    pts = np.zeros((5, 2)) + np.arange(5)[:, None]
    with pytest.raises(ex.KTooLarge, match="k=5"):
        ente.engine.knn_kth_distances(ente.engine.Chunk(pts), 5)
    with pytest.raises(ex.ShapeMismatch):
        ente.engine.radius_counts(ente.engine.Chunk(np.arange(6.0).reshape(3, 2)),
                                  np.array([1.0, 2.0]))


def test_uninstall_restores(ente):
    import ente.ksg
    from paper_1401_4068_b200 import shim
    patched = ente.ksg.estimate_te_batch
    saved = shim.install()
    shim.uninstall(saved)
    assert ente.ksg.estimate_te_batch is patched
