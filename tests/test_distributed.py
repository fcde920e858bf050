"""N>1 host logic of the chunk scheduler on CPU: gloo, world_size 2.

The per-chunk compute here is the CPU oracle (test infrastructure), standing
in for the device pipeline; what is tested is the sharding, the single
all_gather exchange and the reassembly into input order.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1401_4068_b200.scheduler import chunk_cost, gather_te, lpt_partition, sharded_run


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


def _items():
    rng = np.random.default_rng(11)
    return [rng.standard_normal((int(rng.integers(20, 120)), 5)) for _ in range(9)]


def _te_of(batch):
    import oracle
    return np.array([oracle.te_from_counts(4, *oracle.search(p, oracle.te_margs(2, 2), 4)[1])
                     for p in batch])


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        items = _items()
        costs = [chunk_cost(p.shape[0], p.shape[1]) for p in items]
        te = sharded_run(_te_of, items, costs, dist)
        v = gather_te(torch.arange(rank + 1, dtype=torch.float64), dist)
        if rank == 0:
            np.savez(out_path, te=te, gathered=v.numpy())
    finally:
        dist.destroy_process_group()


def test_sharded_run_gloo_world2(tmp_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = np.load(out)
    assert np.array_equal(res["te"], _te_of(_items()))
    assert res["gathered"].tolist() == [0.0, 0.0, 1.0]


@pytest.mark.gpu
def test_analyze_pairs_distributed_equals_analyze_pairs(tmp_path):
    """Single-rank process group on the GPU: the sharded multi-pair analysis
    reproduces analyze_pairs bit for bit (placement never changes a TE)."""
    from paper_1401_4068_b200 import workloads
    from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
    from paper_1401_4068_b200.inference import analyze_pairs
    from paper_1401_4068_b200.scheduler import analyze_pairs_distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        series = {}
        for p in range(3):
            x, y = workloads.ar_pair("bidirectional", 30, 300, seed=p)
            series[f"X{p}"] = EnsembleSeries(f"X{p}", x)
            series[f"Y{p}"] = EnsembleSeries(f"Y{p}", y)
        pairs = [(f"X{p}", f"Y{p}") for p in range(3)] + [("Y0", "X0")]
        specs = {k: EmbeddingSpec(2, 1) for k in series}
        cfg = AnalysisConfig(u_candidates=(5, 7), window=(200, 230), k=4, n_surrogates=15,
                             seed=2, correction="fdr")
        ref = analyze_pairs(series, pairs, specs, cfg)
        got = analyze_pairs_distributed(series, pairs, specs, cfg, dist)
        for a, b in zip(ref, got):
            assert (a.te_value, a.p_value, a.u_selected) == (b.te_value, b.p_value, b.u_selected)
            assert a.surrogate_values.tolist() == b.surrogate_values.tolist()
            assert a.significant_corrected == b.significant_corrected
    finally:
        dist.destroy_process_group()
