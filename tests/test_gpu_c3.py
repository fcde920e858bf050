"""Parity at the sizes the C3 bench reports (1k-64k points/chunk,
joint dims 3-17, TE and bench layouts, tied variant).

The full O(n^2) oracle is too slow at 64k points, so every cell checks a
sample of references exactly: for 256-2048 sampled rows (first, last and random)
the fp64 k-th max-norm distance (self excluded, engine.py:70-123) and the
strict marginal counts (engine.py:126-160) are recomputed by brute force in
numpy -- |a - b| and max are exact in any order, so this is the reference's
value bit for bit -- and compared with the GPU's.  All rows are checked
against size-independent properties: 0 <= count <= n - 1, counts monotone
in the marginal inclusion order of the TE layout, and eps > 0 on
continuous data.
"""

import numpy as np
import pytest

from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.engine import Chunk, batch_search

pytestmark = pytest.mark.gpu

K = 4


def brute_rows(pts, rows, margs, k):
    """Exact eps and marginal counts of the given reference rows (numpy, fp64)."""
    eps = np.empty(len(rows))
    cnt = np.empty((len(margs), len(rows)), dtype=np.int64)
    for i, r in enumerate(rows):
        diff = np.abs(pts - pts[r])
        d = diff.max(axis=1)
        d[r] = np.inf
        eps[i] = np.partition(d, k - 1)[k - 1]
        for m, cols in enumerate(margs):
            dm = diff[:, cols].max(axis=1)
            dm[r] = np.inf
            cnt[m, i] = int(np.count_nonzero(dm < eps[i]))
    return eps, cnt


def sample_rows(n, count=1024, seed=0):
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([[0, 1, n - 2, n - 1],
                                     rng.choice(n, min(count, n), replace=False)]))
    return rows


CELLS = [
    # (n, dim, layout, tied, chunks)
    (65536, 3, "te", False, 1),
    (65536, 7, "te", False, 1),
    (65536, 17, "te", False, 1),
    (16384, 11, "te", False, 2),
    (16384, 13, "te", False, 2),
    (30094, 17, "bench", False, 2),
    (30094, 7, "te", True, 1),
    (30094, 7, "bench", True, 1),
    (1024, 5, "te", True, 8),
]


@pytest.mark.parametrize("n,dim,layout,tied,chunks", CELLS)
def test_c3_cell_exact_on_sampled_rows(n, dim, layout, tied, chunks):
    margs = workloads.c3_marginals(dim, layout)
    pts = [workloads.c3_chunk(n, dim, c, tied) for c in range(chunks)]
    res = batch_search([(Chunk(p), margs) for p in pts], K)
    for c, (p, r) in enumerate(zip(pts, res)):
        assert not isinstance(r, Exception), r
        eps, counts = r.kth_distance, np.stack(r.radius_counts)
        assert eps.shape == (n,) and eps.dtype == np.float64 and counts.dtype == np.int64
        assert (counts >= 0).all() and (counts <= n - 1).all()
        if not tied:
            assert (eps > 0).all()
        if layout == "te":  # ypast subset of y_ypast, ypast subset of ypast_xpast
            assert (counts[1] <= counts[0]).all() and (counts[2] <= counts[0]).all()
        budget = 2048 if n * dim <= 200_000 else (512 if n * dim <= 1_000_000 else 256)
        rows = sample_rows(n, budget if c == 0 else budget // 4, seed=c)
        e_ref, c_ref = brute_rows(p, rows, margs, K)
        assert np.array_equal(eps[rows], e_ref), (n, dim, layout, tied, c)
        assert np.array_equal(counts[:, rows], c_ref), (n, dim, layout, tied, c)
