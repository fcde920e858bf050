"""The run_bench harness (mirror of /root/reference/pkg/src/ente/bench.py and
pkg/tests/test_bench.py) and the C3 workload generator."""

import numpy as np
import pytest

import oracle
from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.bench import BenchReport, _counts_equal, run_bench
from paper_1401_4068_b200.engine import NeighborCounts


def test_rejects_unsorted_chunk_list():
    with pytest.raises(ValueError):
        run_bench(50, 3, 1, 4, [4, 2], repeats=1)


def test_csv_layout():
    r = BenchReport(10, 3, 1, 4, 1, "hw")
    r.rows.append({"n_chunks": 2, "seconds_parallel": 0.5, "seconds_sequential": 1.0,
                   "speedup": 2.0, "searches_per_s": 40.0})
    assert r.to_csv() == "n_chunks,seconds_parallel,seconds_sequential,speedup\n2,0.5,1.0,2.0\n"


def test_counts_equal_is_bitwise():
    a = NeighborCounts(np.array([1.0, 2.0]), (np.array([1, 2]),))
    b = NeighborCounts(np.array([1.0, np.nextafter(2.0, 3.0)]), (np.array([1, 2]),))
    c = NeighborCounts(np.array([1.0, 2.0]), (np.array([1, 3]),))
    assert _counts_equal(a, a) and not _counts_equal(a, b) and not _counts_equal(a, c)


def test_c3_generator_and_layouts():
    a = workloads.c3_chunk(100, 5, 3)
    b = np.random.default_rng(np.random.SeedSequence((0, 100, 5, 3))).standard_normal((100, 5))
    assert np.array_equal(a, b)
    assert np.array_equal(workloads.c3_chunk(100, 5, 3, tied=True), np.round(b, 1))
    assert workloads.c3_marginals(17, "te") == oracle.te_margs(8, 8)
    assert workloads.c3_marginals(17, "bench") == [list(range(8))]
    assert workloads.c3_marginals(7, "knn") == []
    with pytest.raises(ValueError):
        workloads.c3_marginals(6, "te")


@pytest.mark.gpu
def test_run_bench_gate_and_rows():
    rep = run_bench(600, 5, 2, 4, [1, 3], repeats=1)
    assert [r["n_chunks"] for r in rep.rows] == [1, 3]
    for r in rep.rows:
        assert r["seconds_parallel"] > 0 and r["speedup"] > 0 and r["searches_per_s"] > 0
    rep2 = run_bench(600, 5, 2, 4, [4], repeats=1, sequential=False)
    assert rep2.rows[0]["speedup"] is None


@pytest.mark.gpu
@pytest.mark.parametrize("dim,layout,tied", [(7, "te", False), (17, "bench", False),
                                             (5, "te", True), (9, "knn", False)])
def test_c3_cells_bit_exact_vs_oracle(dim, layout, tied):
    from paper_1401_4068_b200.engine import Chunk, batch_search
    margs = workloads.c3_marginals(dim, layout)
    pts = [workloads.c3_chunk(1024, dim, c, tied) for c in range(2)]
    res = batch_search([(Chunk(p), margs) for p in pts], 4)
    for p, r in zip(pts, res):
        eps, cnt = oracle.search(p, margs, 4)
        assert np.array_equal(r.kth_distance, eps)
        assert all(np.array_equal(a, b) for a, b in zip(r.radius_counts, cnt))
