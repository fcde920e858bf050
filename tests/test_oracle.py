"""The CPU oracle is pinned to outputs of the reference itself (tests/golden/)."""

import numpy as np
import pytest

import cases
import oracle

ENGINE_GROUPS = [("hand", cases.hand_cases), ("random", cases.engine_random_chunks),
                 ("tie", cases.engine_tie_chunk), ("c6", cases.criterion6_chunks),
                 ("telayout", cases.te_layout_chunks)]


@pytest.mark.parametrize("name,gen", ENGINE_GROUPS)
def test_oracle_engine_matches_reference(golden, name, gen):
    g = golden("engine.npz")
    cl = gen()
    assert cases.sha(*[p for p, _, _ in cl]) == str(g[f"{name}_sha"]), "input drift"
    eps, cnt = [], []
    for p, m, k in cl:
        e, c = oracle.search(p, m, k)
        eps.append(e)
        cnt += c
    assert np.array_equal(np.concatenate(eps), g[f"{name}_eps"])
    assert np.array_equal(np.concatenate(cnt), g[f"{name}_counts"])


def test_oracle_sweep_equals_brute_force():
    for p, m, k in cases.engine_random_chunks() + cases.criterion6_chunks()[:30]:
        e1, c1 = oracle.search(p, m, k)
        e2, c2 = oracle.search(p, m, k, brute=True)
        assert np.array_equal(e1, e2)
        assert all(np.array_equal(a, b) for a, b in zip(c1, c2))


def test_oracle_hand_examples(golden):
    g = golden("engine.npz")
    eps = oracle.kth_distances(np.array([[0.0], [0.3], [1.0], [2.0]]), 2)
    assert np.allclose(eps, [1.0, 0.7, 1.0, 1.7])
    pts = np.array([[0.0], [1.0], [2.0]])
    assert oracle.radius_counts(pts, [0], [1.0] * 3).tolist() == g["strict_r1"].tolist() == [0, 0, 0]
    assert oracle.radius_counts(pts, [0], [1.5] * 3).tolist() == g["strict_r15"].tolist() == [1, 2, 1]


def test_oracle_te_from_counts(golden):
    g = golden("te.npz")
    vals = []
    for i, m in enumerate(cases.TE_COUNT_SIZES):
        a, b, c = cases.count_triples(i, m)
        for k in (1, 4):
            vals.append(oracle.te_from_counts(k, a, b, c))
    assert np.array_equal(vals, g["counts_te"])
    gold = oracle.te_from_counts(4, [10, 12, 8], [5, 6, 4], [7, 9, 6])
    assert gold == float(g["golden_te_146"])
    assert gold == pytest.approx(-0.146151996151996152, abs=1e-12)  # test_ksg.py:38-46


def test_oracle_estimate_and_jitter(golden):
    g = golden("te.npz")
    tes, shas = [], []
    for bi, (seed, reps, n, sx, sy, u, win) in enumerate(cases.TE_BUNDLES):
        xv, yv = cases.ensemble(seed, reps, n)
        joint = oracle.assemble(xv, yv, sx, sy, u, win)
        for amp in (1e-8, 1e-6, 0.0):
            tes.append(oracle.estimate_te(joint, sy[0], sx[0], 4, amp,
                                          np.random.SeedSequence((bi, u, 7))))
            shas.append(cases.sha(oracle.jittered_joint(joint, amp,
                                                        np.random.SeedSequence((bi, u, 7)))))
    assert np.array_equal(tes, g["bundle_te"])
    assert shas == list(g["bundle_jitter_sha"])


def test_oracle_analyze_pair(golden):
    P = golden("pipeline.json")
    for run in P["runs"][:3]:
        xv, yv = cases.coupled_pair(run["pair_seed"])
        c = run["config"]
        r = oracle.analyze_pair(xv, yv, (1, 1), (1, 1), tuple(c["u_candidates"]),
                                tuple(c["window"]), c["k"], c["n_surrogates"], c.get("seed", 0),
                                c.get("jitter_amplitude", 1e-8), c.get("strict_permutation", True),
                                c.get("test_grid"), c.get("scan_statistic", "max"),
                                c.get("conservative_pvalue", False))
        ref = run["result"]
        assert r["u_selected"] == ref["u_selected"]
        assert r["te_value"] == ref["te_value"]
        assert r["p_value"] == ref["p_value"]
        assert list(r["surrogate_values"]) == ref["surrogate_values"]


def test_oracle_permutations(golden):
    P = golden("pipeline.json")
    for key, perm in P["permutations"].items():
        r, s, strict = (int(v) for v in key.split("_"))
        assert oracle.draw_permutation(r, np.random.SeedSequence((s, 3)), bool(strict)).tolist() == perm
