"""N>1 logic of the chunk scheduler on CPU (gloo, world_size 2), and on the GPU.

CPU tests: the per-chunk compute is the CPU oracle (test infrastructure),
standing in for the device pipeline through a PairPipeline stand-in; what
is tested is the planning in the reference's order, the LPT sharding, the
single fixed-size exchange, the error propagation (every rank raises the
reference's first error, no rank blocks) and the reassembly.

GPU test: two ranks (gloo) both drive the real device pipeline on cuda:0
and must reproduce the single-process analyze_pairs / analyze_windows bit
for bit (reference counterpart: the analyze_pairs loop,
/root/reference/pkg/src/ente/inference.py:203-216).
"""

import os
import socket
import sys
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_4068_b200.scheduler import (chunk_cost, exchange, lpt_partition, raise_first,
                                            sharded_run)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_lpt_partition_balances_and_covers():
    costs = [9, 7, 6, 5, 5, 4, 3, 3, 1]
    bins = lpt_partition(costs, 3)
    assert sorted(i for b in bins for i in b) == list(range(len(costs)))
    loads = [sum(costs[i] for i in b) for b in bins]
    assert max(loads) - min(loads) <= max(costs)
    assert lpt_partition(costs, 3) == bins  # deterministic
    assert lpt_partition([1, 1], 4)[2:] == [[], []]
    assert chunk_cost(10, 3) == 2 * 3 * 10 * 9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# sharded_run / exchange
# ---------------------------------------------------------------------------
def _items():
    rng = np.random.default_rng(11)
    return [rng.standard_normal((int(rng.integers(20, 120)), 5)) for _ in range(9)]


def _te_of(batch):
    import oracle
    te = np.array([oracle.te_from_counts(4, *oracle.search(p, oracle.te_margs(2, 2), 4)[1])
                   for p in batch])
    return te, np.zeros(len(batch), dtype=np.int32)


def _w_sharded(rank, world, out_path):
    items = _items()
    costs = [chunk_cost(p.shape[0], p.shape[1]) for p in items]
    te, st = sharded_run(_te_of, items, costs, dist)
    bins = [[0], [1, 2], [3]][:world] if world == 3 else [[0, 2], [1]]
    v, s = exchange(np.arange(len(bins[rank])) + 10.0 * rank, [rank] * len(bins[rank]), bins,
                    dist)
    if rank == 0:
        np.savez(out_path, te=te, st=st, v=v, s=s)


def test_sharded_run_gloo_world2(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    out = str(tmp_path / "res.npz")
    _spawn(_w_sharded, 2, out)
    res = np.load(out)
    assert np.array_equal(res["te"], _te_of(_items())[0])
    assert not res["st"].any()
    assert res["v"].tolist() == [0.0, 10.0, 1.0] and res["s"].tolist() == [0, 1, 0]


def _w_errors(rank, world, out_path):
    from paper_1401_4068_b200.exceptions import DegenerateData, ShapeMismatch
    items = list(range(12))
    costs = [1.0] * 12

    def run(mine):  # item 9 degenerate, item 5 non-finite: the lowest (5) wins on every rank
        st = np.array([3 if i == 9 else 2 if i == 5 else 0 for i in mine], dtype=np.int32)
        return np.asarray(mine, dtype=np.float64), st

    got = []
    vals, st = sharded_run(run, items, costs, dist)
    try:
        raise_first(st)
    except ShapeMismatch as exc:
        got.append(type(exc).__name__)
    assert vals.tolist() == list(map(float, items))

    def boom(mine):  # rank 1's share fails outside the chunk checks: nobody blocks
        if rank == 1:
            raise DegenerateData("rank-local failure")
        return np.zeros(len(mine)), np.zeros(len(mine), dtype=np.int32)

    try:
        sharded_run(boom, items, costs, dist)
    except (DegenerateData, RuntimeError) as exc:
        got.append(type(exc).__name__)
    with open(out_path + f".{rank}", "w") as f:
        f.write(",".join(got))


def test_sharded_errors_raise_in_reference_order_gloo_world2(tmp_path):
    out = str(tmp_path / "err")
    _spawn(_w_errors, 2, out)
    assert open(out + ".0").read() == "ShapeMismatch,RuntimeError"
    assert open(out + ".1").read() == "ShapeMismatch,DegenerateData"


# ---------------------------------------------------------------------------
# the analyses, with an oracle stand-in for the device pipeline
# ---------------------------------------------------------------------------
class _OraclePipeline:
    """PairPipeline stand-in computing every chunk with the CPU oracle."""

    def __init__(self, source, target, spec_x, spec_y, config, *a):
        self.x, self.y = source.values, target.values
        self.sx, self.sy, self.cfg = (spec_x.dim, spec_x.delay), (spec_y.dim, spec_y.delay), config
        self.w = config.window[1] - config.window[0] + 1
        self.perms = None

    def set_perms(self, perms):
        self.perms = np.asarray(perms)

    def run_status(self, items):
        import oracle
        te, st = [], []
        for u, i, t_lo in items:
            joint = oracle.assemble(self.x, self.y, self.sx, self.sy, u, (t_lo, t_lo + self.w - 1))
            if i >= 0:
                joint = oracle.permuted_joint(joint, self.perms[i], self.w, self.sy[0])
            seed = np.random.SeedSequence((self.cfg.seed, u, 0 if i < 0 else i + 1))
            try:
                te.append(oracle.estimate_te(joint, self.sy[0], self.sx[0], self.cfg.k,
                                             self.cfg.jitter_amplitude, seed))
                st.append(0)
            except ValueError:  # DegenerateData in the oracle's spelling
                te.append(0.0)
                st.append(3)
        return np.array(te), np.array(st, dtype=np.int32)


def _series(n_pairs, reps=12, n=160):
    from paper_1401_4068_b200 import workloads
    from paper_1401_4068_b200.data import EnsembleSeries
    series = {}
    for p in range(n_pairs):
        x, y = workloads.ar_pair("bidirectional", reps, n, seed=p)
        series[f"X{p}"] = EnsembleSeries(f"X{p}", x)
        series[f"Y{p}"] = EnsembleSeries(f"Y{p}", y)
    return series


def _cfg(**kw):
    from paper_1401_4068_b200.data import AnalysisConfig
    base = dict(u_candidates=(3, 5), window=(60, 75), k=4, n_surrogates=7, seed=3,
                correction="fdr")
    base.update(kw)
    return AnalysisConfig(**base)


def _oracle_result(series, a, b, cfg):
    import oracle
    return oracle.analyze_pair(series[a].values, series[b].values, (2, 1), (2, 1),
                               cfg.u_candidates, cfg.window, cfg.k, cfg.n_surrogates, cfg.seed,
                               cfg.jitter_amplitude, cfg.strict_permutation, cfg.test_grid,
                               cfg.scan_statistic)


def _w_pairs(rank, world, out_path, statistic):
    from paper_1401_4068_b200 import inference
    from paper_1401_4068_b200.data import EmbeddingSpec
    from paper_1401_4068_b200.scheduler import (analyze_pair_distributed,
                                                analyze_pairs_distributed,
                                                analyze_windows_distributed)
    inference.PairPipeline = _OraclePipeline
    series = _series(3)
    specs = {k: EmbeddingSpec(2, 1) for k in series}
    cfg = _cfg(scan_statistic=statistic)
    pairs = [("X0", "Y0"), ("X1", "Y1"), ("Y2", "X2")]
    res = analyze_pairs_distributed(series, pairs, specs, cfg, dist)
    one = analyze_pair_distributed(series["X1"], series["Y1"], specs["X1"], specs["Y1"], cfg, dist)
    wins = analyze_windows_distributed(series["X0"], series["Y0"], specs["X0"], specs["Y0"], cfg,
                                       [60, 64, 70], dist)
    if rank == 0:
        np.save(out_path, np.array([[r.te_value, r.p_value, r.u_selected, *r.surrogate_values]
                                    for r in res + [one] + wins]))


@pytest.mark.parametrize("statistic", ["max", "selected"])
def test_distributed_analyses_equal_oracle_gloo_world2(tmp_path, statistic):
    import dataclasses
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    out = str(tmp_path / "pairs.npy")
    _spawn(_w_pairs, 2, out, statistic)
    got = np.load(out)
    series = _series(3)
    cfg = _cfg(scan_statistic=statistic)
    want = [_oracle_result(series, a, b, cfg) for a, b in [("X0", "Y0"), ("X1", "Y1"), ("Y2", "X2")]]
    want.append(_oracle_result(series, "X1", "Y1", cfg))
    for t in (60, 64, 70):
        want.append(_oracle_result(series, "X0", "Y0",
                                   dataclasses.replace(cfg, window=(t, t + 15))))
    for row, w in zip(got, want):
        assert row[0] == w["te_value"] and row[1] == w["p_value"] and row[2] == w["u_selected"]
        assert row[3:].tolist() == list(w["surrogate_values"])


def _w_order(rank, world, out_path):
    from paper_1401_4068_b200 import inference
    from paper_1401_4068_b200.data import EmbeddingSpec, EnsembleSeries
    from paper_1401_4068_b200.exceptions import EnteError
    from paper_1401_4068_b200.scheduler import (analyze_pairs_distributed,
                                                analyze_windows_distributed)
    inference.PairPipeline = _OraclePipeline
    series = _series(2)
    specs = {k: EmbeddingSpec(2, 1) for k in series}
    flat = np.zeros((12, 160))
    series["F"] = EnsembleSeries("F", flat)
    specs["F"] = EmbeddingSpec(2, 1)
    got = []
    cases = [
        # pair 1 degenerate (constant source and target) -> DegenerateData
        lambda: analyze_pairs_distributed(series, [("X0", "Y0"), ("F", "F"), ("X1", "Y1")],
                                          specs, _cfg(), dist),
        # u=70 underflows: the pair's u=3 original runs first, then IndexUnderflow
        lambda: analyze_pairs_distributed(series, [("X0", "Y0")], specs,
                                          _cfg(u_candidates=(3, 70)), dist),
        # R < 2 strict: InvalidPermutation after the originals
        lambda: analyze_pairs_distributed({"A": EnsembleSeries("A", series["X0"].values[:1]),
                                           "B": EnsembleSeries("B", series["Y0"].values[:1])},
                                          [("A", "B")], {"A": specs["X0"], "B": specs["Y0"]},
                                          _cfg(window=(60, 75)), dist),
        # a later window underflows: earlier windows compute, then IndexUnderflow
        lambda: analyze_windows_distributed(series["X0"], series["Y0"], specs["X0"], specs["Y0"],
                                            _cfg(), [60, 2], dist),
        # source/target shape mismatch -> ShapeMismatch on every rank (no out-of-bounds pack)
        lambda: analyze_pairs_distributed({"A": EnsembleSeries("A", series["X0"].values[:6]),
                                           "B": series["Y0"]}, [("A", "B")],
                                          {"A": specs["X0"], "B": specs["Y0"]}, _cfg(), dist),
    ]
    for case in cases:
        try:
            case()
            got.append("none")
        except EnteError as exc:
            got.append(type(exc).__name__)
        except Exception:  # pragma: no cover
            got.append("other:" + traceback.format_exc(limit=1).replace("\n", " "))
    with open(out_path + f".{rank}", "w") as f:
        f.write(",".join(got))


def test_distributed_errors_in_reference_order_gloo_world2(tmp_path):
    out = str(tmp_path / "order")
    _spawn(_w_order, 2, out)
    want = "DegenerateData,IndexUnderflow,InvalidPermutation,IndexUnderflow,ShapeMismatch"
    assert open(out + ".0").read() == want
    assert open(out + ".1").read() == want


# ---------------------------------------------------------------------------
# GPU: two ranks, real device pipeline on cuda:0
# ---------------------------------------------------------------------------
def _w_gpu(rank, world, out_path):
    from paper_1401_4068_b200 import workloads
    from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
    from paper_1401_4068_b200.scheduler import (analyze_pairs_distributed,
                                                analyze_windows_distributed)
    torch.cuda.set_device(0)
    series = {}
    for p in range(3):
        x, y = workloads.ar_pair("bidirectional", 30, 300, seed=p)
        series[f"X{p}"] = EnsembleSeries(f"X{p}", x)
        series[f"Y{p}"] = EnsembleSeries(f"Y{p}", y)
    pairs = [(f"X{p}", f"Y{p}") for p in range(3)] + [("Y0", "X0")]
    specs = {k: EmbeddingSpec(2, 1) for k in series}
    cfg = AnalysisConfig(u_candidates=(5, 7), window=(200, 230), k=4, n_surrogates=15, seed=2,
                         correction="fdr")
    res = analyze_pairs_distributed(series, pairs, specs, cfg, dist)
    wins = analyze_windows_distributed(series["X1"], series["Y1"], specs["X1"], specs["Y1"], cfg,
                                       [200, 210, 240], dist)
    if rank == 0:
        np.save(out_path, np.array([[r.te_value, r.p_value, r.u_selected, r.significant_corrected,
                                     *r.surrogate_values] for r in res + wins]))


@pytest.mark.gpu
def test_distributed_device_pipeline_world2_on_one_gpu(tmp_path):
    """Both ranks run the real device pipeline on cuda:0 (gloo exchange): the
    sharded analyses equal the single-process analyze_pairs / analyze_windows."""
    import dataclasses

    from paper_1401_4068_b200 import workloads
    from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
    from paper_1401_4068_b200.inference import analyze_pair, analyze_pairs
    out = str(tmp_path / "gpu.npy")
    _spawn(_w_gpu, 2, out)
    got = np.load(out)
    series = {}
    for p in range(3):
        x, y = workloads.ar_pair("bidirectional", 30, 300, seed=p)
        series[f"X{p}"] = EnsembleSeries(f"X{p}", x)
        series[f"Y{p}"] = EnsembleSeries(f"Y{p}", y)
    pairs = [(f"X{p}", f"Y{p}") for p in range(3)] + [("Y0", "X0")]
    specs = {k: EmbeddingSpec(2, 1) for k in series}
    cfg = AnalysisConfig(u_candidates=(5, 7), window=(200, 230), k=4, n_surrogates=15, seed=2,
                         correction="fdr")
    ref = analyze_pairs(series, pairs, specs, cfg)
    ref += [analyze_pair(series["X1"], series["Y1"], specs["X1"], specs["Y1"],
                         dataclasses.replace(cfg, window=(t, t + 30))) for t in (200, 210, 240)]
    for row, r in zip(got, ref):
        assert (row[0], row[1], row[2]) == (r.te_value, r.p_value, r.u_selected)
        assert row[4:].tolist() == r.surrogate_values.tolist()
    assert [bool(r[3]) for r in got[:4]] == [r.significant_corrected for r in ref[:4]]
