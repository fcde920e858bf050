"""Generic marginals and caller radii on the fp32-filter sweeps (bit-exact).

Reference functions: radius_counts (engine.py:179-188, strict counts for
caller radii) and _search_one's arbitrary marginal column lists
(engine.py:191-200; criterion 6 draws random subsets,
test_acceptance.py:212-225).  These no longer fall back to the fp64 scan:
ente_search_path says which engine a layout takes, and the counts must equal
the C oracle's (a restatement of _count_sweep) bit for bit, including radii
that equal pairwise distances exactly (the strict boundary), zero and
huge radii, and tied data.
"""

import warnings

import numpy as np
import pytest

import oracle
from paper_1401_4068_b200.engine import (Chunk, SlowPathWarning, batch_search, column_mask,
                                         radius_counts, search_path)

pytestmark = pytest.mark.gpu


def _radii(rng, pts, kind):
    n = len(pts)
    if kind == "pairwise":  # radii equal to an actual max-norm distance: strict boundary
        j = rng.integers(0, n, n)
        r = np.abs(pts - pts[j]).max(axis=1)
        r[j == np.arange(n)] = 0.0
        return r
    if kind == "mixed":
        r = rng.uniform(0.0, 1.5, n)
        r[::7] = 0.0
        r[1::11] = 1e30
        r[2::13] = np.inf
        return r
    return np.full(n, 0.4)


@pytest.mark.parametrize("n,dim,tied", [(5000, 7, False), (3000, 3, True), (4000, 12, False),
                                        (2000, 16, True), (3000, 17, False), (600, 1, False)])
@pytest.mark.parametrize("kind", ["pairwise", "mixed", "const"])
def test_radius_counts_caller_radii_vs_oracle(n, dim, tied, kind):
    rng = np.random.default_rng(n + dim)
    pts = rng.standard_normal((n, dim))
    if tied:
        pts = np.round(pts, 1)
    radii = _radii(rng, pts, kind)
    with warnings.catch_warnings():
        warnings.simplefilter("error", SlowPathWarning)  # <= 17 columns: never the fp64 scan
        got = radius_counts(Chunk(pts), radii)
    want = oracle.radius_counts(pts, list(range(dim)), radii)
    assert got.dtype == np.int64
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_arbitrary_marginal_subsets_take_the_generic_path(seed):
    rng = np.random.default_rng(100 + seed)
    items, expect = [], []
    for _ in range(6):
        n, dim = int(rng.integers(300, 6000)), int(rng.integers(2, 11))
        pts = rng.standard_normal((n, dim))
        if rng.random() < 0.3:
            pts = np.round(pts, 1)
        margs = [sorted(rng.choice(dim, int(rng.integers(1, dim + 1)), replace=False).tolist())
                 for _ in range(int(rng.integers(1, 4)))]
        items.append((Chunk(pts), margs))
        expect.append(oracle.search(pts, margs, 4))
    for (chunk, margs), (eps, cnts) in zip(items, expect):
        masks = [column_mask(m, chunk.points.shape[1]) for m in margs]
        assert search_path(chunk.points.shape[1], masks, 4) in (1, 2)
        (r,) = batch_search([(chunk, margs)], 4)
        assert np.array_equal(r.kth_distance, eps)
        for a, b in zip(r.radius_counts, cnts):
            assert np.array_equal(a, b)


def test_bench_geometry_radius_counts_fast_and_exact():
    """30094 x 17 paper geometry: radius_counts with the kNN radii of the
    bench marginal equals the oracle on sampled rows and takes the sweep."""
    rng = np.random.default_rng(5)
    pts = rng.standard_normal((30094, 17))
    (r,) = batch_search([(Chunk(pts), [list(range(8))])], 4)
    with warnings.catch_warnings():
        warnings.simplefilter("error", SlowPathWarning)
        got = radius_counts(Chunk(pts[:, :8].copy()), r.kth_distance)
    assert np.array_equal(got, r.radius_counts[0])
    rows = rng.choice(len(pts), 256, replace=False)
    sub = pts[:, :8]
    for i in rows:
        d = np.abs(sub - sub[i]).max(axis=1)
        d[i] = np.inf
        assert got[i] == np.count_nonzero(d < r.kth_distance[i])


def test_slow_path_is_reported():
    rng = np.random.default_rng(0)
    pts = rng.standard_normal((300, 20))
    with pytest.warns(SlowPathWarning):
        (r,) = batch_search([(Chunk(pts), [[0, 1]])], 3)
    eps, cnts = oracle.search(pts, [[0, 1]], 3)
    assert np.array_equal(r.kth_distance, eps) and np.array_equal(r.radius_counts[0], cnts[0])
