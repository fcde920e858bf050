"""GPU parity of the neighbour engine: bit-exact vs the reference goldens and the oracle.

Reference tests mirrored: pkg/tests/test_engine.py (hand examples, random and
tied chunks vs O(n^2), validation, error slots, worker invariance) and the
engine-oracle acceptance criterion (test_acceptance.py:198-247).
"""

import numpy as np
import pytest

import cases
import oracle
from paper_1401_4068_b200.engine import (Chunk, batch_search, knn_kth_distances,
                                         radius_counts)
from paper_1401_4068_b200.exceptions import KTooLarge, ShapeMismatch

pytestmark = pytest.mark.gpu

GROUPS = [("hand", cases.hand_cases), ("random", cases.engine_random_chunks),
          ("tie", cases.engine_tie_chunk), ("c6", cases.criterion6_chunks),
          ("telayout", cases.te_layout_chunks)]


def run_group(cl):
    eps, cnt = [], []
    by_k = {}
    for i, (p, m, k) in enumerate(cl):
        by_k.setdefault(k, []).append(i)
    res = [None] * len(cl)
    for k, idx in by_k.items():
        out = batch_search([(Chunk(cl[i][0]), cl[i][1]) for i in idx], k)
        for i, r in zip(idx, out):
            res[i] = r
    for r in res:
        assert not isinstance(r, Exception), r
        eps.append(r.kth_distance)
        cnt += list(r.radius_counts)
    return np.concatenate(eps), np.concatenate(cnt)


@pytest.mark.parametrize("name,gen", GROUPS)
def test_engine_bit_exact_vs_reference_goldens(golden, name, gen):
    g = golden("engine.npz")
    cl = gen()
    assert cases.sha(*[p for p, _, _ in cl]) == str(g[f"{name}_sha"])
    eps, cnt = run_group(cl)
    assert eps.dtype == np.float64
    assert np.array_equal(eps, g[f"{name}_eps"])
    assert np.array_equal(cnt, g[f"{name}_counts"])


def test_hand_examples():
    eps = knn_kth_distances(Chunk(np.array([[0.0], [0.3], [1.0], [2.0]])), 2)
    assert np.allclose(eps, [1.0, 0.7, 1.0, 1.7])
    pts = Chunk(np.array([[0.0], [1.0], [2.0]]))
    assert radius_counts(pts, np.array([1.0, 1.0, 1.0])).tolist() == [0, 0, 0]
    assert radius_counts(pts, np.array([1.5, 1.5, 1.5])).tolist() == [1, 2, 1]


def _te_case(rng, n, d_y, d_x, kind):
    d = 1 + d_y + d_x
    pts = rng.standard_normal((n, d))
    if kind == "round":
        pts = np.round(pts, 1)
    elif kind == "offset":
        pts = pts * 1e-4 + 5e3
    elif kind == "dup":
        pts[n // 2:] = pts[: n - n // 2]
    elif kind == "lowdim":
        t = rng.standard_normal((n, 1))
        pts = np.concatenate([t + 1e-3 * rng.standard_normal((n, 1)) for _ in range(d)], axis=1)
    return pts, cases.te_margs(d_y, d_x)


@pytest.mark.parametrize("kind", ["normal", "round", "offset", "dup", "lowdim"])
def test_fast_path_vs_oracle_multi_chunk(kind):
    rng = np.random.default_rng(hash(kind) % 2 ** 32)
    for d_y, d_x in [(1, 1), (2, 2), (3, 3), (2, 3), (8, 8)]:
        items, ref = [], []
        for n in (5, 129, 700, 1500):
            pts, margs = _te_case(rng, n, d_y, d_x, kind)
            items.append((Chunk(pts), margs))
            ref.append(oracle.search(pts, margs, 4))
        for (e, c), r in zip(ref, batch_search(items, 4)):
            assert np.array_equal(r.kth_distance, e)
            for a, b in zip(r.radius_counts, c):
                assert np.array_equal(a, b)


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 15, 16, 20])
def test_all_k_vs_oracle(k):
    rng = np.random.default_rng(k)
    pts = np.round(rng.standard_normal((900, 5)), 2)
    margs = cases.te_margs(2, 2) + [[0], [4, 1]]
    (r,) = batch_search([(Chunk(pts), margs)], k)
    e, c = oracle.search(pts, margs, k)
    assert np.array_equal(r.kth_distance, e)
    for a, b in zip(r.radius_counts, c):
        assert np.array_equal(a, b)


def test_bench_layout_paper_geometry_sample():
    # paper geometry columns: joint 17, marginal = first 8 (bench.py:56)
    rng = np.random.default_rng(0)
    pts = rng.standard_normal((3000, 17))
    (r,) = batch_search([(Chunk(pts), [list(range(8))])], 4)
    e, (c,) = oracle.search(pts, [list(range(8))], 4)
    assert np.array_equal(r.kth_distance, e) and np.array_equal(r.radius_counts[0], c)


def test_errors_are_isolated_per_slot():
    rng = np.random.default_rng(0)
    good = Chunk(rng.standard_normal((20, 3)))
    res = batch_search([(good, [[0], [0, 1]]), (good, [[0, 7]]), (good, [[2]]),
                        (Chunk(rng.standard_normal((3, 3))), [[0]])], k=3)
    assert not isinstance(res[0], Exception)
    assert isinstance(res[1], ShapeMismatch)
    assert not isinstance(res[2], Exception)
    assert isinstance(res[3], KTooLarge)
    assert np.array_equal(res[0].kth_distance, res[2].kth_distance)
    with pytest.raises(KTooLarge):
        knn_kth_distances(Chunk(np.arange(10.0).reshape(5, 2)), 5)
    with pytest.raises(ShapeMismatch):
        radius_counts(Chunk(np.arange(6.0).reshape(3, 2)), np.array([1.0, -1.0, 2.0]))


def test_strict_count_bound_and_monotone_k():
    rng = np.random.default_rng(4)
    pts = rng.standard_normal((400, 3))
    ch = Chunk(pts)
    prev = None
    for k in (1, 2, 3, 4):
        (r,) = batch_search([(ch, [[0, 1, 2]])], k)
        assert np.all(r.radius_counts[0] <= k - 1)
        if prev is not None:
            assert np.all(r.kth_distance >= prev)
        prev = r.kth_distance


def test_translation_and_scale():
    rng = np.random.default_rng(9)
    pts = rng.standard_normal((600, 5))
    e = knn_kth_distances(Chunk(pts), 4)
    assert np.allclose(knn_kth_distances(Chunk(pts + 7.25), 4), e, rtol=0, atol=1e-9)
    assert np.allclose(knn_kth_distances(Chunk(pts * 2.0), 4), 2.0 * e, rtol=1e-12, atol=0)


def test_batch_equals_singles():
    rng = np.random.default_rng(5)
    chunks = [Chunk(rng.standard_normal((n, 7))) for n in (300, 1000, 2048)]
    margs = cases.te_margs(3, 3)
    batch = batch_search([(c, margs) for c in chunks], 4)
    for c, b in zip(chunks, batch):
        (s,) = batch_search([(c, margs)], 4)
        assert np.array_equal(s.kth_distance, b.kth_distance)
        assert all(np.array_equal(x, y) for x, y in zip(s.radius_counts, b.radius_counts))


@pytest.mark.parametrize("uniform", [True, False])
def test_pipelined_parts_equal_one_wave(monkeypatch, uniform):
    """batch_search waves are uploaded / searched / read back in parts of
    PIPE_BYTES on two streams; tiny parts must give the one-part results,
    slot for slot, with the per-slot errors of mixed batches in place."""
    from paper_1401_4068_b200 import engine

    rng = np.random.default_rng(11)
    sizes = [700] * 40 if uniform else rng.integers(20, 1500, 40).tolist()
    chunks = [Chunk(rng.standard_normal((int(n), 7))) for n in sizes]
    margs = cases.te_margs(3, 3)
    items = [(c, margs) for c in chunks]
    if not uniform:  # per-slot errors in the middle of the batch
        items[5] = (chunks[5], [[0, 9]])
        items[17] = (Chunk(rng.standard_normal((3, 7))), margs)
    whole = batch_search(items, 4)
    monkeypatch.setattr(engine, "PIPE_BYTES", 64 << 10)  # ~ 1 to 3 chunks per part
    parts = batch_search(items, 4)
    for a, b in zip(whole, parts):
        if isinstance(a, Exception):
            assert type(a) is type(b)
            continue
        assert np.array_equal(a.kth_distance, b.kth_distance)
        assert all(np.array_equal(x, y) for x, y in zip(a.radius_counts, b.radius_counts))
    for i in (0, 13, 39):
        eps, cnts = oracle.search(chunks[i].points, margs, 4)
        assert np.array_equal(parts[i].kth_distance, eps)
        assert all(np.array_equal(x, y) for x, y in zip(parts[i].radius_counts, cnts))
    if not uniform:
        assert isinstance(parts[5], ShapeMismatch) and isinstance(parts[17], KTooLarge)


@pytest.mark.parametrize("subset", [(0,), (1,), (2,), (1, 2), (2, 0), ()])
def test_marginal_subsets_choose_exact_filter(subset):
    # every subset of the TE marginals selects its own pruning columns
    rng = np.random.default_rng(len(subset) * 7 + sum(subset))
    d_y, d_x = 3, 3
    full = cases.te_margs(d_y, d_x)
    margs = [full[s] for s in subset]
    t = np.cumsum(rng.standard_normal((4000, 1)), axis=0) * 0.05
    pts = np.concatenate([np.sin(t * (c + 1)) + 1e-3 * rng.standard_normal((4000, 1))
                          for c in range(1 + d_y + d_x)], axis=1)
    (r,) = batch_search([(Chunk(pts), margs)], 4)
    e, c = oracle.search(pts, margs, 4)
    assert np.array_equal(r.kth_distance, e)
    for a, b in zip(r.radius_counts, c):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["clustered", "lorenz_like", "round"])
def test_pruned_sweep_large_chunks(kind):
    # multi-stage traversal with heavy pruning: clustered / attractor-like data
    rng = np.random.default_rng(11)
    n = 9000
    if kind == "clustered":
        centres = rng.standard_normal((12, 7)) * 10
        pts = centres[rng.integers(0, 12, n)] + 0.1 * rng.standard_normal((n, 7))
    elif kind == "lorenz_like":
        s = np.cumsum(rng.standard_normal(n + 10)) * 0.1
        pts = np.stack([np.sin(s[i:i + n] * 0.7 + i) for i in range(7)], axis=1)
    else:
        pts = np.round(rng.standard_normal((n, 7)), 1)
    margs = cases.te_margs(3, 3)
    (r,) = batch_search([(Chunk(pts), margs)], 4)
    e, c = oracle.search(pts, margs, 4)
    assert np.array_equal(r.kth_distance, e)
    for a, b in zip(r.radius_counts, c):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["random", "rounded", "duplicates", "lorenz_like", "lowdim"])
@pytest.mark.parametrize("k", [1, 4, 9])
def test_knn_indices_canonical_order(kind, k):
    """Neighbour indices bit-exact vs the O(n^2) oracle: ascending (fp64 distance, index)."""
    from paper_1401_4068_b200.engine import knn_indices
    rng = np.random.default_rng(5 + k)
    n = 1500
    if kind == "random":
        pts = rng.standard_normal((n, 7))
    elif kind == "rounded":
        pts = np.round(rng.standard_normal((n, 5)), 1)
    elif kind == "duplicates":
        pts = rng.standard_normal((n // 3, 3)).repeat(3, axis=0)
    elif kind == "lorenz_like":
        s = np.cumsum(rng.standard_normal(n + 10)) * 0.05
        pts = np.stack([np.sin(s[i:i + n] * 0.7 + i) for i in range(7)], axis=1)
    else:
        pts = rng.standard_normal((n, 1))
    got = knn_indices(Chunk(pts), k)
    assert np.array_equal(got, oracle.knn_indices(pts, k))
    # the k-th entry sits at exactly the k-th distance
    eps = knn_kth_distances(Chunk(pts), k)
    assert np.array_equal(np.abs(pts - pts[got[:, -1]]).max(axis=1), eps)


def test_knn_indices_large_pruned_chunk():
    from paper_1401_4068_b200.engine import knn_indices
    rng = np.random.default_rng(2)
    n = 12000
    s = np.cumsum(rng.standard_normal(n + 10)) * 0.05
    pts = np.stack([np.sin(s[i:i + n] * 0.7 + i) for i in range(7)], axis=1)
    got = knn_indices(Chunk(pts), 4)
    sel = rng.choice(n, 300, replace=False)
    d = np.abs(pts[sel][:, None, :] - pts[None, :, :]).max(axis=2)
    d[np.arange(300), sel] = np.inf
    for row, i in enumerate(sel):
        order = np.lexsort((np.arange(n), d[row]))[:4]
        assert np.array_equal(got[i], order)


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_split_search_parts_cover_every_row_once(parts):
    """ente_search_split: the parts' outputs are disjoint and sum to the full search."""
    import torch
    from paper_1401_4068_b200.engine import search_device
    rng = np.random.default_rng(parts)
    dup = np.repeat(rng.standard_normal((40, 7)), 6, axis=0)  # >= k+1 copies: eps == 0
    chunks = [rng.standard_normal((7000, 7)), np.round(rng.standard_normal((3000, 7)), 1),
              rng.standard_normal((200, 7)), dup]
    ns = np.array([len(c) for c in chunks])
    rows0 = np.concatenate([[0], np.cumsum(ns)[:-1]])
    dev = torch.from_numpy(np.concatenate(chunks)).cuda()
    margs = cases.te_margs(3, 3)
    masks = [sum(1 << c for c in m) for m in margs]
    eps_sum = torch.zeros(dev.shape[0], dtype=torch.float64, device=dev.device)
    cnt_sum = torch.zeros((3, dev.shape[0]), dtype=torch.int32, device=dev.device)
    written = torch.zeros(dev.shape[0], dtype=torch.int32, device=dev.device)
    for part in range(parts):
        # rows outside the part keep the fill: NaN / -1 mark them unwritten, so
        # rows with eps == 0 (duplicates) still count as written
        eps, cnt, _ = search_device(dev, rows0, ns, masks, 4, split=(part, parts),
                                    split_fill=(float("nan"), -1))
        mine = ~torch.isnan(eps)
        assert bool((cnt[:, mine] >= 0).all()) and bool((cnt[:, ~mine] == -1).all())
        eps_sum += torch.where(mine, eps, torch.zeros_like(eps))
        cnt_sum += torch.where(mine[None, :], cnt, torch.zeros_like(cnt))
        written += mine.int()
    assert int(written.min()) == 1 and int(written.max()) == 1
    for c, r0, n in zip(chunks, rows0, ns):
        e, cnt = oracle.search(c, margs, 4)
        assert np.array_equal(eps_sum[r0:r0 + n].cpu().numpy(), e)
        for m in range(3):
            assert np.array_equal(cnt_sum[m, r0:r0 + n].cpu().numpy().astype(np.int64), cnt[m])


def test_batch_search_split_single_rank_group():
    import os
    import socket
    import torch.distributed as dist
    from paper_1401_4068_b200.scheduler import batch_search_split
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        pts = np.random.default_rng(4).standard_normal((5000, 5))
        margs = cases.te_margs(2, 2)
        (r,) = batch_search_split([(Chunk(pts), margs)], 4, dist)
        e, c = oracle.search(pts, margs, 4)
        assert np.array_equal(r.kth_distance, e)
        assert all(np.array_equal(a, b) for a, b in zip(r.radius_counts, c))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k", [16, 31, 32, 47, 63])
def test_large_k_shared_memory_lists(k):
    """k + 1 > 16: the kNN pass keeps its sorted lists in shared memory; exact anyway."""
    rng = np.random.default_rng(k)
    for pts in (rng.standard_normal((4500, 7)), np.round(rng.standard_normal((3000, 5)), 1)):
        dim = pts.shape[1]
        dy = 3 if dim == 7 else 2
        margs = [list(range(1, 1 + dy)), list(range(0, 1 + dy)), list(range(1, dim))]
        (r,) = batch_search([(Chunk(pts), margs)], k)
        e, c = oracle.search(pts, margs, k)
        assert np.array_equal(r.kth_distance, e)
        assert all(np.array_equal(a, b) for a, b in zip(r.radius_counts, c))


def test_uniform_batch_search_equals_host_table_path():
    """5000 equal chunks (device-built chunk table) give the results of the
    same chunks with one ragged chunk appended (host-built table)."""
    rng = np.random.default_rng(21)
    chunks = [Chunk(rng.standard_normal((64, 5))) for _ in range(5000)]
    margs = cases.te_margs(2, 2)
    uni = batch_search([(c, margs) for c in chunks], 4)
    mixed = batch_search([(c, margs) for c in chunks] + [(Chunk(rng.standard_normal((65, 5))), margs)], 4)
    for a, b in zip(uni, mixed):
        assert np.array_equal(a.kth_distance, b.kth_distance)
        assert all(np.array_equal(x, y) for x, y in zip(a.radius_counts, b.radius_counts))
    for i in (0, 2500, 4999):
        eps, cnts = oracle.search(chunks[i].points, margs, 4)
        assert np.array_equal(uni[i].kth_distance, eps)
        assert all(np.array_equal(x, y) for x, y in zip(uni[i].radius_counts, cnts))
