"""GPU parity of the estimator: jitter, digamma reduction, estimate_te_batch, analyze_pair.

Reference tests mirrored: pkg/tests/test_ksg.py (te_from_counts goldens,
batch == singles, jitter determinism, degenerate / k errors) and
test_inference.py (pipeline determinism and the coupled-pair detection).
"""

import numpy as np
import pytest
import torch

import cases
import oracle
from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.embedding import assemble_pointsets
from paper_1401_4068_b200.exceptions import DegenerateData, KTooLarge
from paper_1401_4068_b200.inference import analyze_pair
from paper_1401_4068_b200.ksg import (TermCounts, estimate_te, estimate_te_batch, jitter_device,
                                      te_from_counts)

pytestmark = pytest.mark.gpu


def bundle_of(row):
    seed, reps, n, sx, sy, u, win = row
    xv, yv = cases.ensemble(seed, reps, n)
    return assemble_pointsets(EnsembleSeries("X", xv), EnsembleSeries("Y", yv),
                              EmbeddingSpec(*sx), EmbeddingSpec(*sy), u, win)


def test_te_from_counts_goldens(golden):
    g = golden("te.npz")
    vals = []
    for i, m in enumerate(cases.TE_COUNT_SIZES):
        a, b, c = cases.count_triples(i, m)
        for k in (1, 4):
            vals.append(te_from_counts(TermCounts(k, a, b, c)))
    assert np.array_equal(vals, g["counts_te"])  # bit-exact, incl. pairwise-sum splits
    v = te_from_counts(TermCounts(4, np.array([10, 12, 8]), np.array([5, 6, 4]),
                                  np.array([7, 9, 6])))
    assert v == pytest.approx(-0.146151996151996152, abs=1e-12)


def test_device_jitter_bit_exact(golden):
    g = golden("te.npz")
    shas = []
    for bi, row in enumerate(cases.TE_BUNDLES):
        joint = bundle_of(row).joint
        for amp in (1e-8, 1e-6, 0.0):
            dev = torch.from_numpy(joint.copy()).cuda()
            st = jitter_device(dev, [0], [joint.shape[0]], amp,
                               [np.random.SeedSequence((bi, row[5], 7))])
            assert int(st.cpu()[0]) == 0
            shas.append(cases.sha(dev.cpu().numpy()))
    assert shas == list(g["bundle_jitter_sha"])


def test_estimate_te_goldens(golden):
    g = golden("te.npz")
    vals = []
    for bi, row in enumerate(cases.TE_BUNDLES):
        b = bundle_of(row)
        for amp in (1e-8, 1e-6, 0.0):
            vals.append(estimate_te(b, 4, amp, np.random.SeedSequence((bi, row[5], 7))))
    assert np.array_equal(vals, g["bundle_te"])
    batch = estimate_te_batch([bundle_of(r) for r in cases.TE_BUNDLES], 4)
    assert np.array_equal(batch, g["batch_default_seeds"])


def test_errors():
    src = EnsembleSeries("X", np.zeros((2, 50)))
    tgt = EnsembleSeries("Y", np.zeros((2, 50)))
    spec = EmbeddingSpec(1, 1)
    b = assemble_pointsets(src, tgt, spec, spec, 1, (2, 50))
    with pytest.raises(DegenerateData):
        estimate_te(b, 4, 0.0, np.random.SeedSequence(0))
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(12), rng.standard_normal(12)
    b = assemble_pointsets(EnsembleSeries("X", x[None]), EnsembleSeries("Y", y[None]), spec, spec,
                           1, (2, 12))
    with pytest.raises(KTooLarge):
        estimate_te(b, 11, 0.0, np.random.SeedSequence(0))


def test_gaussian_channel_close_to_analytic():
    # y_t = 0.5 x_{t-1} + eta: TE = 0.5 ln 1.25 (test_ksg.py:79-88)
    vals = []
    for seed in range(3):
        r = np.random.default_rng(seed)
        m = 10_000
        x = r.standard_normal(m + 1)
        y = np.empty(m + 1)
        y[0] = r.standard_normal()
        eta = r.standard_normal(m + 1)
        y[1:] = 0.5 * x[:-1] + eta[1:]
        spec = EmbeddingSpec(1, 1)
        b = assemble_pointsets(EnsembleSeries("X", x[None]), EnsembleSeries("Y", y[None]), spec,
                               spec, 1, (2, m + 1))
        vals.append(estimate_te(b, 4, 1e-8, np.random.SeedSequence(seed)))
        assert vals[-1] == oracle.estimate_te(b.joint, 1, 1, 4, 1e-8, np.random.SeedSequence(seed))
    assert np.mean(vals) == pytest.approx(0.111571775657104878, abs=0.03)


def test_analyze_pair_matches_reference(golden):
    P = golden("pipeline.json")
    for run in P["runs"]:
        xv, yv = cases.coupled_pair(run["pair_seed"])
        cfg = AnalysisConfig(**{k: tuple(v) if isinstance(v, list) else v
                                for k, v in run["config"].items()})
        res = analyze_pair(EnsembleSeries("X", xv), EnsembleSeries("Y", yv), EmbeddingSpec(1, 1),
                           EmbeddingSpec(1, 1), cfg)
        ref = run["result"]
        assert res.u_selected == ref["u_selected"], run["name"]
        assert res.te_value == ref["te_value"], run["name"]
        assert res.p_value == ref["p_value"], run["name"]
        assert [[u, t] for u, t in res.te_curve] == ref["te_curve"], run["name"]
        assert res.surrogate_values.tolist() == ref["surrogate_values"], run["name"]


@pytest.mark.parametrize("name,key,u,idx", [
    ("C1", "c1_te", 1, [None, 0, 1]),
    ("C2", "c2_te_u1", 1, [None, 0, 1]),
    ("C2", "c2_te_u5", 5, [None, 199]),
    ("C4", "c4_te_t501", 10, [None, 0, 1, 2]),
    ("C5", "c5_te_u5", 5, [None, 0]),
])
def test_config_chunks_match_reference(golden, name, key, u, idx):
    """Original and surrogate chunks of the BASELINE configs, built on the device."""
    from paper_1401_4068_b200.inference import PairPipeline, cached_permutation
    g = golden("workloads.npz")
    wl = workloads.CONFIGS[name]
    xv, yv = wl.ensembles()
    spec = EmbeddingSpec(*wl.spec)
    cfg = AnalysisConfig(u_candidates=(u,), window=wl.window, k=4, n_surrogates=200, seed=0)
    pipe = PairPipeline(EnsembleSeries("X", xv), EnsembleSeries("Y", yv), spec, spec, cfg)
    perm_ids = [i for i in idx if i is not None]
    if perm_ids:
        perms = [cached_permutation(0, i, xv.shape[0], True) for i in range(max(perm_ids) + 1)]
        pipe.set_perms(perms)
    te = pipe.run([(u, -1 if i is None else i) for i in idx])
    assert np.array_equal(te, g[key])


def test_analyze_windows_equals_per_window_analyze_pair():
    """One device batch over many windows == one analyze_pair call per window."""
    import dataclasses
    from paper_1401_4068_b200 import analyze_windows
    wl = workloads.CONFIGS["C4"]
    xv, yv = wl.ensembles()
    xv, yv = xv[:60], yv[:60]  # 60 trials keep the per-window calls quick
    spec = EmbeddingSpec(*wl.spec)
    cfg = AnalysisConfig(u_candidates=(8, 10), window=(501, 501), k=4, n_surrogates=20, seed=3)
    X, Y = EnsembleSeries("X", xv), EnsembleSeries("Y", yv)
    starts = [501, 777, 1200]
    batch = analyze_windows(X, Y, spec, spec, cfg, starts)
    for t, res in zip(starts, batch):
        one = analyze_pair(X, Y, spec, spec, dataclasses.replace(cfg, window=(t, t)))
        assert res.window == one.window == (t, t)
        assert res.te_curve == one.te_curve
        assert res.surrogate_values.tolist() == one.surrogate_values.tolist()
        assert (res.u_selected, res.te_value, res.p_value) == (one.u_selected, one.te_value,
                                                               one.p_value)
    # and the batch agrees with the CPU oracle's analyze_pair on one window
    ref = oracle.analyze_pair(xv, yv, wl.spec, wl.spec, (8, 10), (777, 777), k=4,
                              n_surrogates=20, seed=3)
    assert batch[1].te_value == ref["te_value"]
    assert batch[1].surrogate_values.tolist() == list(ref["surrogate_values"])


def test_te_reduce_runs_of_equal_high_key_bits():
    """Brackets that agree in their top 32 bits but differ below (the sort's
    fix-up path) still reduce to numpy's exact sorted pairwise mean."""
    import torch
    from paper_1401_4068_b200 import _native as nat
    rng = np.random.default_rng(9)
    m = 3000
    table = 1.0 + np.arange(64) * 2.0 ** -44           # values 1 ulp-ish apart at 2^-44
    table[::7] = -0.5 - np.arange(10) * 2.0 ** -41     # and a few negative clusters
    a, b, c = (rng.integers(0, 64, m).astype(np.int32) for _ in range(3))
    vals = (table[a] - table[b]) - table[c]
    ref = np.float64(0.25) + np.sort(vals).sum() / m    # numpy pairwise sum of the sorted terms
    dev = nat.device()
    counts = torch.from_numpy(np.stack([a, b, c])).to(dev)
    psi = torch.from_numpy(table).to(dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    L = nat.lib()
    tab = nat.chunk_table([0], [m])
    ws = nat.workspace(L.ente_te_reduce_workspace_size(tab, 1))
    nat.check(L.ente_te_reduce(nat.ptr(counts), m, tab, 1, nat.ptr(psi), psi.numel(), 0.25,
                               nat.ptr(out), nat.ptr(ws), ws.numel(), nat.stream_handle()), "reduce")
    assert float(out.cpu()[0]) == float(ref)


def test_uniform_batch_tables_built_on_device():
    """>= 4096 equal chunks take the device-built chunk tables (search, jitter
    from pinned states, reduction): the same TE as per-window calls on the
    host-table path and as the CPU oracle."""
    import dataclasses
    from paper_1401_4068_b200 import analyze_windows
    wl = workloads.CONFIGS["C4"]
    xv, yv = wl.ensembles()
    xv, yv = xv[:60], yv[:60]
    spec = EmbeddingSpec(*wl.spec)
    cfg = AnalysisConfig(u_candidates=(8, 10), window=(501, 501), k=4, n_surrogates=20, seed=5)
    X, Y = EnsembleSeries("X", xv), EnsembleSeries("Y", yv)
    starts = list(range(501, 501 + 110))  # 110 windows x 42 chunks = 4620 chunks in one wave
    batch = analyze_windows(X, Y, spec, spec, cfg, starts)
    for i in (0, 57, 109):
        one = analyze_pair(X, Y, spec, spec, dataclasses.replace(cfg, window=(starts[i], starts[i])))
        assert batch[i].te_curve == one.te_curve
        assert batch[i].surrogate_values.tolist() == one.surrogate_values.tolist()
    ref = oracle.analyze_pair(xv, yv, wl.spec, wl.spec, (8, 10), (starts[57], starts[57]), k=4,
                              n_surrogates=20, seed=5)
    assert batch[57].te_value == ref["te_value"]
    assert batch[57].surrogate_values.tolist() == list(ref["surrogate_values"])
