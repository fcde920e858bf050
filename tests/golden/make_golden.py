"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package ``ente`` in place from
/root/reference/pkg/src (read-only; nothing is copied) and records, for the
inputs produced by tests/golden/cases.py:

* engine.npz    - kth_distance / radius_counts of ente.engine.batch_search
                  (pkg/src/ente/engine.py:203-216) for every engine case group
* te.npz        - te_from_counts (pkg/src/ente/ksg.py:39-49) on count triples,
                  estimate_te_batch (ksg.py:66-90) on assembled bundles, the
                  jittered joints (ksg.py:52-59) as hashes + leading rows
* pipeline.json - analyze_pair (pkg/src/ente/inference.py:120-193) results
* workloads.npz - simulator output hashes (simulators.py:100-231) and TE
                  values of original/surrogate chunks of configs C1, C2, C4, C5

Versions of numpy/scipy/numba are recorded in every file: RNG streams
(PCG64, SeedSequence) are pinned against this container's numpy.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numba  # noqa: E402
import scipy  # noqa: E402

import cases  # noqa: E402
from ente import engine, inference, ksg, simulators  # noqa: E402
from ente.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries  # noqa: E402
from ente.embedding import assemble_pointsets  # noqa: E402

VERSIONS = {"numpy": np.__version__, "scipy": scipy.__version__, "numba": numba.__version__}


def engine_group(case_list):
    items = [(engine.Chunk(p), m) for p, m, _ in case_list]
    eps_all, cnt_all = [], []
    for (p, m, k), item in zip(case_list, items):
        (res,) = engine.batch_search([item], k)
        assert not isinstance(res, Exception), res
        eps_all.append(res.kth_distance)
        for c in res.radius_counts:
            cnt_all.append(c.astype(np.int64))
    sha_in = cases.sha(*[p for p, _, _ in case_list])
    return np.concatenate(eps_all), np.concatenate(cnt_all), sha_in


def make_engine():
    out = {}
    groups = {
        "hand": cases.hand_cases() and [(p, m, k) for p, m, k in cases.hand_cases()],
        "random": cases.engine_random_chunks(),
        "tie": cases.engine_tie_chunk(),
        "c6": cases.criterion6_chunks(),
        "telayout": cases.te_layout_chunks(),
    }
    for name, cl in groups.items():
        t0 = time.time()
        eps, cnt, sha_in = engine_group(cl)
        out[f"{name}_eps"] = eps
        out[f"{name}_counts"] = cnt.astype(np.int32)
        out[f"{name}_sha"] = np.array(sha_in)
        print(f"engine {name}: {len(cl)} chunks, {time.time() - t0:.1f}s")
    # strict-boundary known answers (pkg/tests/test_engine.py:62-68)
    pts = np.array([[0.0], [1.0], [2.0]])
    out["strict_r1"] = engine.radius_counts(engine.Chunk(pts), np.array([1.0, 1.0, 1.0]))
    out["strict_r15"] = engine.radius_counts(engine.Chunk(pts), np.array([1.5, 1.5, 1.5]))
    np.savez_compressed(os.path.join(HERE, "engine.npz"), versions=json.dumps(VERSIONS), **out)


def bundle_of(spec_row):
    seed, reps, n, sx, sy, u, window = spec_row
    xv, yv = cases.ensemble(seed, reps, n)
    return assemble_pointsets(EnsembleSeries("X", xv), EnsembleSeries("Y", yv),
                              EmbeddingSpec(*sx), EmbeddingSpec(*sy), u, window)


def make_te():
    out = {}
    vals = []
    for i, m in enumerate(cases.TE_COUNT_SIZES):
        a, b, c = cases.count_triples(i, m)
        for k in (1, 4):
            vals.append(ksg.te_from_counts(ksg.TermCounts(k, a, b, c)))
    out["counts_te"] = np.array(vals)
    out["golden_te_146"] = np.array(ksg.te_from_counts(ksg.TermCounts(
        4, np.array([10, 12, 8]), np.array([5, 6, 4]), np.array([7, 9, 6]))))
    # psi table check values used by the device reduction
    out["psi_1_64"] = ksg.digamma(np.arange(1, 65, dtype=np.float64))

    te_vals, jit_sha, jit_head, eps_sha, cnt_sha = [], [], [], [], []
    for bi, row in enumerate(cases.TE_BUNDLES):
        bundle = bundle_of(row)
        for amp in (1e-8, 1e-6, 0.0):
            seed = np.random.SeedSequence((bi, row[5], 7))
            te = ksg.estimate_te(bundle, 4, amp, seed)
            te_vals.append(te)
            joint = ksg._jittered_joint(bundle, amp, np.random.SeedSequence((bi, row[5], 7)))
            jit_sha.append(cases.sha(joint))
            jit_head.append(joint[:8].ravel())
            (res,) = engine.batch_search([(engine.Chunk(joint), ksg._marginal_cols(bundle))], 4)
            eps_sha.append(cases.sha(res.kth_distance))
            cnt_sha.append(cases.sha(*[c.astype(np.int64) for c in res.radius_counts]))
    out["bundle_te"] = np.array(te_vals)
    out["bundle_jitter_sha"] = np.array(jit_sha)
    out["bundle_jitter_head"] = np.concatenate(jit_head)
    out["bundle_eps_sha"] = np.array(eps_sha)
    out["bundle_counts_sha"] = np.array(cnt_sha)
    # batch call with default integer seeds (ksg.py:72-73: seeds=range(len))
    bundles = [bundle_of(r) for r in cases.TE_BUNDLES]
    out["batch_default_seeds"] = np.array(ksg.estimate_te_batch(bundles, 4))
    np.savez_compressed(os.path.join(HERE, "te.npz"), versions=json.dumps(VERSIONS), **out)
    print("te fixtures done")


def result_dict(res):
    return {"u_selected": int(res.u_selected), "te_value": float(res.te_value),
            "p_value": float(res.p_value), "significant": bool(res.significant),
            "te_curve": [[int(u), float(t)] for u, t in res.te_curve],
            "surrogate_values": [float(v) for v in res.surrogate_values],
            "te_minus_median_surrogate": float(res.te_minus_median_surrogate)}


def make_pipeline():
    runs = []
    base = dict(u_candidates=(1, 2, 3, 4, 5), window=(40, 200), k=4,
                n_surrogates=20, alpha=0.1, seed=0)
    for name, seed, kw in [("detect", 2, {}), ("selected", 5, {"scan_statistic": "selected"}),
                           ("seed11", 4, {"seed": 11}), ("nojitter", 7, {"jitter_amplitude": 0.0,
                                                                         "n_surrogates": 5}),
                           ("grid", 3, {"test_grid": (2, 4), "conservative_pvalue": True}),
                           ("nonstrict", 6, {"strict_permutation": False, "n_surrogates": 8})]:
        xv, yv = cases.coupled_pair(seed)
        cfg = AnalysisConfig(**{**base, **kw})
        res = inference.analyze_pair(EnsembleSeries("X", xv), EnsembleSeries("Y", yv),
                                     EmbeddingSpec(1, 1), EmbeddingSpec(1, 1), cfg)
        runs.append({"name": name, "pair_seed": seed, "config": {**base, **kw},
                     "result": result_dict(res)})
    # permutations drawn by draw_permutation (inference.py:41-49)
    perms = {f"{r}_{s}_{int(strict)}": inference.draw_permutation(
        r, np.random.SeedSequence((s, 3)), strict).permutation.tolist()
        for r in (2, 5, 50, 250) for s in (0, 1, 9) for strict in (True, False)}
    with open(os.path.join(HERE, "pipeline.json"), "w") as f:
        json.dump({"versions": VERSIONS, "runs": runs, "permutations": perms}, f, indent=1)
    print("pipeline fixtures done")


def config_chunks(x, y, spec, u, window, seed, idx_list):
    """Original (idx=None) and surrogate chunks exactly as analyze_pair builds them."""
    bundle = assemble_pointsets(x, y, spec, spec, u, window)
    w = window[1] - window[0] + 1
    out = []
    for idx in idx_list:
        if idx is None:
            out.append((bundle, np.random.SeedSequence((seed, u, 0))))
        else:
            perm = inference.draw_permutation(x.n_repetitions,
                                              inference._surrogate_seed(seed, idx), True)
            out.append((inference._permuted_bundle(bundle, perm.permutation, w),
                        np.random.SeedSequence((seed, u, idx + 1))))
    return out


def make_workloads():
    out = {}
    t0 = time.time()
    x1, y1 = simulators.simulate_ar_pair(simulators.table1_params("unidirectional", 50, 3000, seed=0))
    out["c1_sha"] = np.array(cases.sha(x1.values, y1.values))
    lor = simulators.LorenzParams(delta_xy=5, n_repetitions=500, n_samples=200,
                                  gamma_schedule=lambda t: 0.3, seed=0)
    x2, y2 = simulators.simulate_lorenz_pair(lor)
    out["c2_sha"] = np.array(cases.sha(x2.values, y2.values))
    out["c2_head"] = np.concatenate([x2.values[:2, :16].ravel(), y2.values[:2, :16].ravel()])
    x4, y4 = simulators.simulate_ar_pair(simulators.table1_params("unidirectional", 500, 1600, seed=0))
    out["c4_sha"] = np.array(cases.sha(x4.values, y4.values))
    x5, y5 = simulators.simulate_ar_pair(simulators.table1_params("bidirectional", 250, 1000, seed=0))
    out["c5_sha"] = np.array(cases.sha(x5.values, y5.values))
    # small Lorenz for a fast exact-simulator check (criterion-1 style params)
    lsmall = simulators.LorenzParams(delta_xy=45, n_repetitions=3, n_samples=400,
                                     gamma_schedule=lambda t: 0.3 if 100 <= t <= 300 else 0.0, seed=2)
    xs, ys = simulators.simulate_lorenz_pair(lsmall)
    out["lorenz_small_sha"] = np.array(cases.sha(xs.values, ys.values))
    out["lorenz_small"] = np.stack([xs.values, ys.values])
    print(f"simulators {time.time() - t0:.1f}s")

    def te_of(chunks):
        return [ksg.estimate_te(b, 4, 1e-8, s) for b, s in chunks]

    t0 = time.time()
    out["c1_te"] = np.array(te_of(config_chunks(x1, y1, EmbeddingSpec(2, 1), 1, (1101, 1400), 0,
                                                [None, 0, 1])))
    out["c2_te_u1"] = np.array(te_of(config_chunks(x2, y2, EmbeddingSpec(3, 1), 1, (121, 180), 0,
                                                   [None, 0, 1])))
    out["c2_te_u5"] = np.array(te_of(config_chunks(x2, y2, EmbeddingSpec(3, 1), 5, (121, 180), 0,
                                                   [None, 199])))
    out["c4_te_t501"] = np.array(te_of(config_chunks(x4, y4, EmbeddingSpec(2, 1), 10, (501, 501), 0,
                                                     [None, 0, 1, 2])))
    out["c5_te_u5"] = np.array(te_of(config_chunks(x5, y5, EmbeddingSpec(3, 1), 5, (801, 890), 0,
                                                   [None, 0])))
    print(f"config TE {time.time() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, "workloads.npz"), versions=json.dumps(VERSIONS), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["engine", "te", "pipeline", "workloads"]
    for w in which:
        globals()[f"make_{w}"]()
