"""Shared-y TE batches (ente_search_te_shared) equal the per-chunk search bit for bit.

Every chunk of one analyze_pair window pools the same target rows, so the
two y marginals are counted once per original point (csrc/shared_y.cuh).
The counts and eps must equal ente_search's on the same jittered chunks --
including jitter amplitude 0 and rounded (tied) ensembles, where many pairs
sit exactly on the radius and the exact settlement decides -- and the TE of
whole pipelines must not change.
"""

import numpy as np
import pytest
import torch

from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.engine import search_device, search_te_shared_device
from paper_1401_4068_b200.inference import PairPipeline, surrogate_perms
from paper_1401_4068_b200.ksg import jitter_device, te_masks

pytestmark = pytest.mark.gpu


def _batch(x, y, dy, dx, us, s, window, amp, seed=0):
    spec_x, spec_y = EmbeddingSpec(dx, 1), EmbeddingSpec(dy, 1)
    cfg = AnalysisConfig(u_candidates=tuple(us), window=window, k=4, n_surrogates=s, seed=seed,
                         jitter_amplitude=amp)
    pipe = PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec_x, spec_y, cfg)
    pipe.set_perms(surrogate_perms(seed, s, x.shape[0], True))
    items = pipe._items([(u, -1) for u in us] + [(u, i) for u in us for i in range(s)])
    from paper_1401_4068_b200 import _native as nat
    n = len(items)
    pts = torch.empty((n * pipe.m, pipe.dim), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().ente_pack_te_items(
        nat.ptr(pipe.x), nat.ptr(pipe.y), pipe.reps, pipe.n_samples, dx, 1, dy, 1, pipe.w,
        items.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int32)), n, nat.ptr(pipe.perm_dev),
        nat.ptr(pts), nat.stream_handle()), "pack")
    rows0 = np.arange(n, dtype=np.int64) * pipe.m
    ns = np.full(n, pipe.m, dtype=np.int64)
    st = jitter_device(pts, rows0, ns, amp, pipe._states(items))
    assert not st.cpu().numpy().any()
    return pipe, items, pts, rows0, ns


@pytest.mark.parametrize("kind,amp", [("lorenz", 1e-8), ("ar", 1e-8), ("ar_round", 1e-8),
                                      ("ar_round", 0.0), ("ar", 0.0)])
def test_shared_y_counts_equal_per_chunk_search(kind, amp):
    if kind == "lorenz":
        x, y = workloads.lorenz_pair(5, 60, 200, gamma_schedule=lambda t: 0.3, seed=1)
        dy = dx = 3
        window = (121, 200)
    else:
        x, y = workloads.ar_pair("bidirectional", 40, 400, seed=2)
        if kind == "ar_round":
            x, y = np.round(x, 1), np.round(y, 1)
        dy, dx = 2, 3
        window = (201, 300)
    pipe, items, pts, rows0, ns = _batch(x, y, dy, dx, (2, 5), 30, window, amp)
    eps_a, cnt_a, st_a = search_device(pts, rows0, ns, te_masks(dy, dx), 4)
    eps_a, cnt_a = eps_a.clone(), cnt_a.clone()
    shared = pipe.shared_y(int(items[0, 2]), items[:, 1])
    eps_b, cnt_b, st_b = search_te_shared_device(pts, rows0, ns, dy, 4, shared)
    assert torch.equal(st_a, st_b) and not st_b.cpu().numpy().any()
    assert torch.equal(eps_a, eps_b)
    assert torch.equal(cnt_a, cnt_b)


@pytest.mark.parametrize("name", ["C1", "C2", "C5"])
def test_pipeline_te_unchanged_by_shared_y(name, monkeypatch):
    from paper_1401_4068_b200 import inference
    wl = workloads.CONFIGS[name]
    x, y = wl.ensembles()
    spec = EmbeddingSpec(*wl.spec)
    s = 40
    cfg = AnalysisConfig(u_candidates=wl.u_candidates[:3], window=wl.window, k=4, n_surrogates=s,
                         seed=0)
    pipe = PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec, spec, cfg)
    pipe.set_perms(surrogate_perms(0, s, x.shape[0], True))
    items = [(u, -1) for u in cfg.u_candidates] + [(u, i) for u in cfg.u_candidates for i in range(s)]
    monkeypatch.setattr(inference, "SHARED_Y", True)
    monkeypatch.setattr(PairPipeline, "shared_pays", lambda self, t, u: True)  # AR data too
    te_shared = pipe.run(items)
    monkeypatch.setattr(inference, "SHARED_Y", False)
    te_sweep = pipe.run(items)
    assert np.array_equal(te_shared, te_sweep)


def test_shared_y_is_chosen_for_embedded_dynamics_only():
    wl = workloads.CONFIGS["C2"]
    x, y = wl.ensembles()
    spec = EmbeddingSpec(*wl.spec)
    cfg = AnalysisConfig(u_candidates=(1,), window=wl.window, k=4, n_surrogates=2, seed=0)
    assert PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec, spec,
                        cfg).shared_pays(wl.window[0], 1)
    wl = workloads.CONFIGS["C5"]
    x, y = wl.ensembles()
    spec = EmbeddingSpec(*wl.spec)
    cfg = AnalysisConfig(u_candidates=(5,), window=wl.window, k=4, n_surrogates=2, seed=0)
    assert not PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec, spec,
                            cfg).shared_pays(wl.window[0], 5)


@pytest.mark.parametrize("dy,dx,k", [(1, 4, 4), (4, 2, 7), (3, 3, 20)])
def test_shared_y_other_layouts_and_k(dy, dx, k):
    """d_y = 1 and 4, k = 7, and k = 20 (beyond the shared-y sweep's register
    lists: the call falls back to the general search) -- always the same counts."""
    x, y = workloads.lorenz_pair(5, 50, 200, gamma_schedule=lambda t: 0.3, seed=3)
    spec_x, spec_y = EmbeddingSpec(dx, 1), EmbeddingSpec(dy, 1)
    cfg = AnalysisConfig(u_candidates=(3,), window=(121, 200), k=k, n_surrogates=12, seed=4)
    pipe = PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec_x, spec_y, cfg)
    pipe.set_perms(surrogate_perms(4, 12, x.shape[0], True))
    items = pipe._items([(3, -1)] + [(3, i) for i in range(12)])
    from paper_1401_4068_b200 import _native as nat
    n = len(items)
    pts = torch.empty((n * pipe.m, pipe.dim), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().ente_pack_te_items(
        nat.ptr(pipe.x), nat.ptr(pipe.y), pipe.reps, pipe.n_samples, dx, 1, dy, 1, pipe.w,
        items.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int32)), n, nat.ptr(pipe.perm_dev),
        nat.ptr(pts), nat.stream_handle()), "pack")
    rows0 = np.arange(n, dtype=np.int64) * pipe.m
    ns = np.full(n, pipe.m, dtype=np.int64)
    jitter_device(pts, rows0, ns, 1e-8, pipe._states(items))
    eps_a, cnt_a, _ = search_device(pts, rows0, ns, te_masks(dy, dx), k)
    eps_a, cnt_a = eps_a.clone(), cnt_a.clone()
    eps_b, cnt_b, st = search_te_shared_device(pts, rows0, ns, dy, k, pipe.shared_y(121, items[:, 1]))
    assert not st.cpu().numpy().any()
    assert torch.equal(eps_a, eps_b) and torch.equal(cnt_a, cnt_b)
