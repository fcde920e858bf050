"""Randomised parity sweep of the engine: many small batches with random shapes,
layouts, k, offsets, scales and tie levels, every result bit-exact vs the C oracle
(oracle/ente_oracle.c, the restated reference sweep engine.py:70-160)."""

import os

import numpy as np
import pytest

import oracle
from paper_1401_4068_b200.engine import Chunk, batch_search

pytestmark = pytest.mark.gpu


def _case(rng):
    kind = rng.integers(0, 6)
    dim = int(rng.integers(1, 12))
    n = int(rng.integers(6, 2600))
    k = int(rng.integers(1, min(20, n - 1) + 1))
    pts = rng.standard_normal((n, dim)) * 10.0 ** rng.uniform(-3, 3)
    if kind == 1:
        pts = np.round(pts, int(rng.integers(0, 3)))              # heavy ties
    elif kind == 2:
        pts = pts + 10.0 ** rng.uniform(0, 6)                      # large offset
    elif kind == 3:
        pts[: n // 2] = pts[0]                                     # duplicate block
    elif kind == 4:
        s = np.cumsum(rng.standard_normal(n + dim))               # smooth, embedded
        pts = np.stack([s[i:i + n] for i in range(dim)], axis=1)
    elif kind == 5:
        pts = rng.integers(-3, 4, (n, dim)).astype(np.float64)     # tiny integer lattice
    if dim >= 3 and rng.random() < 0.6:                            # TE layout
        dy = int(rng.integers(1, dim - 1))
        margs = [list(range(1, 1 + dy)), list(range(0, 1 + dy)), list(range(1, dim))]
    else:
        margs = [sorted(rng.choice(dim, int(rng.integers(1, dim + 1)), replace=False).tolist())
                 for _ in range(int(rng.integers(0, 3)))]
    return pts, margs, k


@pytest.mark.parametrize("seed", range(int(os.environ.get("ENTE_FUZZ_SEEDS", "12"))))
def test_random_batches_bit_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    cases = [_case(rng) for _ in range(6)]
    for pts, margs, k in cases:
        (res,) = batch_search([(Chunk(pts), margs)], k)
        assert not isinstance(res, Exception), res
        eps, cnt = oracle.search(pts, margs, k)
        assert np.array_equal(res.kth_distance, eps), (pts.shape, k, margs)
        for a, b in zip(res.radius_counts, cnt):
            assert np.array_equal(a, b), (pts.shape, k, margs)


@pytest.mark.parametrize("seed", range(3))
def test_mixed_batch_one_call(seed):
    """Many chunks of one layout in one launch sequence (different n, data kinds)."""
    rng = np.random.default_rng(77 + seed)
    dim, dy = 7, 3
    margs = [list(range(1, 1 + dy)), list(range(0, 1 + dy)), list(range(1, dim))]
    chunks = []
    for _ in range(9):
        n = int(rng.integers(50, 6000))
        p = rng.standard_normal((n, dim))
        if rng.random() < 0.4:
            p = np.round(p, 1)
        chunks.append(p)
    res = batch_search([(Chunk(p), margs) for p in chunks], 4)
    for p, r in zip(chunks, res):
        eps, cnt = oracle.search(p, margs, 4)
        assert np.array_equal(r.kth_distance, eps)
        assert all(np.array_equal(a, b) for a, b in zip(r.radius_counts, cnt))


@pytest.mark.parametrize("seed", range(8))
def test_compacted_sweeps_bit_exact(seed):
    """Batches whose largest chunk has >= 4096 rows take the compacted kNN and
    count sweeps (grouped rounds); random k over all three register-list
    widths (k + 1 <= 5, 8, 16), ties, smooth embedded data and clusters."""
    rng = np.random.default_rng(500 + seed)
    dim = int(rng.choice([3, 5, 7, 9]))
    dy = int(rng.integers(1, dim - 1))
    margs = [list(range(1, 1 + dy)), list(range(0, 1 + dy)), list(range(1, dim))]
    k = int(rng.choice([1, 4, 6, 11, 15]))
    chunks = []
    for kind in range(4):
        n = int(rng.integers(4096, 9000)) if kind == 0 else int(rng.integers(300, 7000))
        if kind == 1:
            p = np.round(rng.standard_normal((n, dim)), 1)
        elif kind == 2:
            s = np.cumsum(rng.standard_normal(n + dim))
            p = np.stack([s[i:i + n] for i in range(dim)], axis=1)
        elif kind == 3:
            c = rng.standard_normal((8, dim)) * 5.0
            p = c[rng.integers(0, 8, n)] + 0.05 * rng.standard_normal((n, dim))
        else:
            p = rng.standard_normal((n, dim))
        chunks.append(p)
    res = batch_search([(Chunk(p), margs) for p in chunks], k)
    for p, r in zip(chunks, res):
        assert not isinstance(r, Exception), r
        eps, cnt = oracle.search(p, margs, k)
        assert np.array_equal(r.kth_distance, eps), (p.shape, k)
        assert all(np.array_equal(a, b) for a, b in zip(r.radius_counts, cnt)), (p.shape, k)
