"""Host-side logic of the drop-in API (no GPU): data model, assembly, inference
statistics, seeding, workload generators.  Mirrors the reference's unit tests
(pkg/tests/test_data.py, test_embedding.py, test_inference.py)."""

import numpy as np
import pytest

import cases
import oracle
from paper_1401_4068_b200 import _native as nat
from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.data import (AnalysisConfig, EmbeddingSpec, EnsembleSeries,
                                       ensemble_from_rows, validate_ensemble)
from paper_1401_4068_b200.embedding import assemble_pointsets, embed_past_state
from paper_1401_4068_b200.engine import Chunk, column_mask, max_workers, set_workers
from paper_1401_4068_b200.exceptions import (EmptyEnsemble, EnteError, IndexUnderflow,
                                             InvalidPermutation, KTooLarge, NonFiniteValue,
                                             RaggedRepetitions, ShapeMismatch, UnknownMethod)
from paper_1401_4068_b200.inference import (SurrogateSpec, _permuted_bundle, correct_multiple,
                                            draw_permutation, jitter_state, permutation_pvalue,
                                            shuffle_target)
from paper_1401_4068_b200.ksg import te_masks


def test_exception_tree():
    assert issubclass(KTooLarge, EnteError) and issubclass(ShapeMismatch, EnteError)
    e = NonFiniteValue(2, 5)
    assert (e.rep, e.t) == (2, 5) and "repetition 2" in str(e)


def test_ensemble_validation():
    with pytest.raises(EmptyEnsemble):
        validate_ensemble(EnsembleSeries("a", np.zeros((0, 4))))
    with pytest.raises(RaggedRepetitions):
        validate_ensemble(EnsembleSeries("a", np.zeros(4)))
    v = np.zeros((3, 5))
    v[1, 3] = np.nan
    with pytest.raises(NonFiniteValue) as ei:
        validate_ensemble(EnsembleSeries("a", v))
    assert (ei.value.rep, ei.value.t) == (1, 3)
    with pytest.raises(RaggedRepetitions):
        ensemble_from_rows("a", [[1, 2], [1]])
    s = EnsembleSeries("a", [[1, 2, 3]])
    assert not s.values.flags.writeable and s.n_repetitions == 1 and s.n_samples == 3


def test_config_validation():
    AnalysisConfig(u_candidates=(1, 2), window=(5, 10))
    bad = [dict(u_candidates=()), dict(u_candidates=(2, 1)), dict(u_candidates=(0,)),
           dict(window=(10, 5)), dict(k=0), dict(n_surrogates=0), dict(alpha=1.0),
           dict(correction="holm"), dict(jitter_amplitude=-1.0), dict(scan_statistic="x"),
           dict(test_grid=()), dict(test_grid=(3,)), dict(test_grid=(2, 1))]
    for kw in bad:
        base = dict(u_candidates=(1, 2), window=(5, 10))
        base.update(kw)
        with pytest.raises(ValueError):
            AnalysisConfig(**base)
    with pytest.raises(ValueError):
        EmbeddingSpec(0, 1)
    assert EmbeddingSpec(3, 2).span == 5


def test_assembly_matches_oracle_restatement():
    for seed, reps, n, sx, sy, u, win in cases.TE_BUNDLES:
        xv, yv = cases.ensemble(seed, reps, n)
        b = assemble_pointsets(EnsembleSeries("X", xv), EnsembleSeries("Y", yv),
                               EmbeddingSpec(*sx), EmbeddingSpec(*sy), u, win)
        assert np.array_equal(b.joint, oracle.assemble(xv, yv, sx, sy, u, win))
        assert b.row_origin[0].tolist() == [1, win[0]]


def test_assembly_layout_and_errors():
    rng = np.random.default_rng(3)
    src = EnsembleSeries("X", rng.standard_normal((4, 30)))
    tgt = EnsembleSeries("Y", rng.standard_normal((4, 30)))
    sx, sy = EmbeddingSpec(2, 3), EmbeddingSpec(3, 1)
    b = assemble_pointsets(src, tgt, sx, sy, 5, (12, 20))
    for row in (0, 7, 13, 35):
        r, t = b.row_origin[row]
        assert b.joint[row, 0] == tgt.values[r - 1, t - 1]
        assert np.array_equal(b.joint[row, 1:4], embed_past_state(tgt, sy, int(r), int(t) - 1))
        assert np.array_equal(b.joint[row, 4:], embed_past_state(src, sx, int(r), int(t) - 5))
    assert np.array_equal(b.marg_ypast_xpast, b.joint[:, 1:6])
    with pytest.raises(IndexUnderflow):
        assemble_pointsets(src, tgt, sx, sy, 5, (5, 20))
    with pytest.raises(IndexUnderflow):
        assemble_pointsets(src, tgt, sx, sy, 1, (12, 31))
    with pytest.raises(ShapeMismatch):
        assemble_pointsets(src, EnsembleSeries("Y", np.zeros((3, 30))), sx, sy, 1, (12, 20))


def test_permuted_bundle_and_shuffle():
    rng = np.random.default_rng(0)
    src = EnsembleSeries("X", rng.standard_normal((7, 80)))
    tgt = EnsembleSeries("Y", rng.standard_normal((7, 80)))
    sx, sy = EmbeddingSpec(2, 2), EmbeddingSpec(2, 1)
    b = assemble_pointsets(src, tgt, sx, sy, 4, (20, 60))
    perm = draw_permutation(7, 9)
    fast = _permuted_bundle(b, perm.permutation, 41)
    slow = assemble_pointsets(src, shuffle_target(tgt, perm), sx, sy, 4, (20, 60))
    assert np.array_equal(fast.joint, slow.joint)
    assert np.array_equal(_permuted_bundle(b, np.arange(7), 41).joint, b.joint)
    with pytest.raises(InvalidPermutation):
        SurrogateSpec(np.array([0, 0, 1]))
    with pytest.raises(InvalidPermutation):
        draw_permutation(1, 0)


def test_permutations_match_reference(golden):
    P = golden("pipeline.json")
    for key, perm in P["permutations"].items():
        r, s, strict = (int(v) for v in key.split("_"))
        got = draw_permutation(r, np.random.SeedSequence((s, 3)), bool(strict)).permutation
        assert got.tolist() == perm


def test_pvalue_and_corrections():
    assert permutation_pvalue(0.5, [0.1, 0.5, 0.7, 0.2]) == 0.5
    assert permutation_pvalue(0.8, [0.1, 0.5, 0.7, 0.2], conservative=True) == 0.2
    with pytest.raises(ValueError):
        permutation_pvalue(0.5, [])
    assert correct_multiple([0.01, 0.02, 0.04, 0.5], 0.05, "bonferroni") == [True, False, False, False]
    assert correct_multiple([0.01, 0.02, 0.04, 0.5], 0.05, "fdr") == [True, True, False, False]
    assert correct_multiple([0.04, 0.03, 0.02, 0.05], 0.05, "fdr") == [True] * 4
    assert correct_multiple([0.01, 0.2], 0.05, "none") == [True, False]
    with pytest.raises(UnknownMethod):
        correct_multiple([0.01], 0.05, "holm")


def test_chunk_and_masks():
    with pytest.raises(ShapeMismatch):
        Chunk(np.zeros((1, 3)))
    with pytest.raises(ShapeMismatch):
        Chunk(np.array([[0.0, np.nan], [1.0, 2.0]]))
    assert column_mask([0, 2, 2], 3) == 0b101
    with pytest.raises(ShapeMismatch):
        column_mask([0, 7], 3)
    with pytest.raises(ShapeMismatch):
        column_mask([], 3)
    assert te_masks(2, 2) == [0b110, 0b111, 0b11110]
    assert set_workers(10 ** 6) == max_workers()
    assert set_workers(-3) == 1
    set_workers(max_workers())


def test_pcg_state_extraction_matches_numpy():
    st = nat.pcg_states([np.random.SeedSequence((1, 2, 3)), 5], [10, 10])
    for row, seed in zip(st, [np.random.SeedSequence((1, 2, 3)), 5]):
        s = np.random.default_rng(seed).bit_generator.state["state"]
        assert (int(row[0]) << 64 | int(row[1])) == s["state"]
        assert (int(row[2]) << 64 | int(row[3])) == s["inc"]
    assert tuple(int(v) for v in st[0]) == jitter_state((1, 2, 3))
    gen = np.random.default_rng(7)
    nat.pcg_states([gen], [12])
    ref = np.random.default_rng(7)
    ref.uniform(-1, 1, size=12)
    assert gen.bit_generator.state == ref.bit_generator.state


def test_workloads_match_reference_simulators(golden):
    g = golden("workloads.npz")
    x, y = workloads.lorenz_pair(45, 3, 400, gamma_schedule=lambda t: 0.3 if 100 <= t <= 300 else 0.0,
                                 seed=2)
    assert cases.sha(x, y) == str(g["lorenz_small_sha"])
    for name in ("C1", "C2"):
        x, y = workloads.CONFIGS[name].ensembles()
        assert cases.sha(x, y) == str(g[f"{name.lower()}_sha"])


def test_window_statistics_batch_matches_per_window():
    """analyze_windows' array statistics equal analyze_pair's per-window host
    statistics (inference.py:153-193), NaN surrogates and both p-value forms."""
    import dataclasses

    import numpy as np

    from paper_1401_4068_b200.data import AnalysisConfig, EnsembleSeries
    from paper_1401_4068_b200.inference import _assemble_result, _assemble_results

    rng = np.random.default_rng(5)
    X = EnsembleSeries("X", rng.standard_normal((4, 60)))
    Y = EnsembleSeries("Y", rng.standard_normal((4, 60)))
    for cons in (False, True):
        cfg = AnalysisConfig(u_candidates=(3, 5, 7), window=(20, 20), k=4, n_surrogates=40,
                             seed=0, conservative_pvalue=cons, test_grid=(5, 7))
        us, grid = list(cfg.u_candidates), list(cfg.test_grid)
        te_o = np.round(rng.random((25, len(us))), 1)           # ties in the delay scan
        te_s = np.round(rng.random((25, len(grid), 40)), 1)
        te_s[3, 0, 5] = np.nan
        windows = [(20 + i, 20 + i) for i in range(25)]
        one = [_assemble_result(X, Y, dataclasses.replace(cfg, window=w), us, grid, te_o[i], te_s[i])
               for i, w in enumerate(windows)]
        batch = _assemble_results(X, Y, cfg, windows, us, grid, te_o, te_s)
        for a, b in zip(one, batch):
            da, db = dataclasses.asdict(a), dataclasses.asdict(b)
            assert np.array_equal(da.pop("surrogate_values"), db.pop("surrogate_values"), equal_nan=True)
            ma, mb = da.pop("te_minus_median_surrogate"), db.pop("te_minus_median_surrogate")
            assert ma == mb or (np.isnan(ma) and np.isnan(mb))
            assert da == db
