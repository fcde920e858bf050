"""Deterministic input generators shared by the golden-fixture script and the tests.

Only numpy is used, so the same inputs can be regenerated on the GPU box
(same image, same numpy) without /root/reference.  Every generator restates
the input-drawing code of a reference test or config so that fixture outputs
computed by the reference can be matched against this repo's outputs:

* ``engine_random_chunks``   -> pkg/tests/test_engine.py:71-80 (rng(0), 25 chunks)
* ``engine_tie_chunk``       -> pkg/tests/test_engine.py:83-89
* ``criterion6_chunks``      -> pkg/tests/test_acceptance.py:212-225
* ``te_layout_chunks``       -> TE-layout joints (SURVEY 8d C1/C2 shapes, smaller n)
* ``coupled_pair``           -> pkg/tests/test_inference.py:108-113
"""

from __future__ import annotations

import hashlib

import numpy as np


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def hand_cases():
    """Hand examples of pkg/tests/test_engine.py:55-68."""
    return [
        (np.array([[0.0], [0.3], [1.0], [2.0]]), [[0]], 2),
        (np.array([[0.0], [1.0], [2.0]]), [[0]], 1),
    ]


def engine_random_chunks():
    """pkg/tests/test_engine.py:71-80 drawing order, plus two marginals per chunk."""
    rng = np.random.default_rng(0)
    out = []
    for _ in range(25):
        n = int(rng.integers(5, 80))
        dim = int(rng.integers(1, 7))
        pts = rng.standard_normal((n, dim))
        k = int(rng.integers(1, min(5, n - 1) + 1))
        out.append((pts, k))
    cases = []
    mrng = np.random.default_rng(1)
    for pts, k in out:
        dim = pts.shape[1]
        margs = [list(range(dim))]
        sub = sorted(mrng.choice(dim, size=int(mrng.integers(1, dim + 1)), replace=False).tolist())
        margs.append(sub)
        cases.append((pts, margs, k))
    return cases


def engine_tie_chunk():
    rng = np.random.default_rng(0)
    pts = np.round(rng.standard_normal((60, 3)), 0)
    return [(pts, [[0], [1, 2], [0, 1, 2]], 3)]


def criterion6_chunks():
    """Restatement of pkg/tests/test_acceptance.py:212-225 (k=4)."""
    rng = np.random.default_rng(2024)
    chunks = []
    for _ in range(100):
        n = int(rng.integers(10, 501))
        dim = int(rng.integers(1, 11))
        pts = rng.standard_normal((n, dim))
        if rng.random() < 0.3:
            pts = np.round(pts, 1)
        n_marg = int(rng.integers(1, 4))
        margs = [sorted(rng.choice(dim, size=int(rng.integers(1, dim + 1)),
                                   replace=False).tolist())
                 for _ in range(n_marg)]
        chunks.append((pts, margs, 4))
    return chunks


def te_margs(d_y: int, d_x: int):
    """Marginal column lists of the TE layout (pkg/src/ente/embedding.py:50-60)."""
    return [list(range(1, 1 + d_y)), list(range(0, 1 + d_y)),
            list(range(1, 1 + d_y + d_x))]


def te_layout_chunks():
    """Medium TE-layout and bench-layout chunks (continuous, tied, offset)."""
    cases = []
    for seed, (n, d_y, d_x, kind) in enumerate([
            (1500, 2, 2, "normal"), (2000, 3, 3, "normal"), (1200, 1, 1, "normal"),
            (900, 2, 2, "round"), (1100, 3, 3, "offset"), (700, 4, 4, "normal"),
            (800, 8, 8, "normal"), (600, 2, 3, "round1")]):
        rng = np.random.default_rng((77, seed))
        d = 1 + d_y + d_x
        pts = rng.standard_normal((n, d))
        if kind == "round":
            pts = np.round(pts, 1)
        elif kind == "round1":
            pts = np.round(pts * 2.0, 0)
        elif kind == "offset":
            pts = pts * 1e-3 + 1e3
        cases.append((pts, te_margs(d_y, d_x), 4))
    # bench layout: one marginal = first m columns (pkg/src/ente/bench.py:56)
    rng = np.random.default_rng((78, 0))
    cases.append((rng.standard_normal((1000, 17)), [list(range(8))], 4))
    rng = np.random.default_rng((78, 1))
    cases.append((rng.standard_normal((700, 9)), [list(range(4))], 4))
    return cases


def ensemble(seed, reps, n):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((reps, n)), rng.standard_normal((reps, n))


def coupled_pair(seed, n_rep=15, n=250, lag=3, gain=0.9):
    """pkg/tests/test_inference.py:108-113."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n_rep, n))
    y = rng.standard_normal((n_rep, n)) * 0.4
    y[:, lag:] += gain * x[:, :-lag]
    return x, y


def count_triples(seed, m, hi=60):
    rng = np.random.default_rng((91, seed))
    a = rng.integers(0, hi, size=m)
    b = np.minimum(a, rng.integers(0, hi, size=m))
    c = np.minimum(a, rng.integers(0, hi, size=m))
    return a.astype(np.int64), b.astype(np.int64), c.astype(np.int64)


TE_COUNT_SIZES = [1, 2, 3, 7, 8, 9, 15, 16, 17, 100, 127, 128, 129, 130, 255, 256,
                  257, 1000, 1023, 4099, 15000, 30000]

# (seed, reps, n_samples, spec_x (dim, delay), spec_y, u, window) for TE-level fixtures
TE_BUNDLES = [
    (0, 10, 120, (1, 1), (1, 1), 1, (5, 110)),
    (1, 7, 80, (2, 2), (2, 1), 4, (20, 60)),
    (2, 20, 200, (2, 1), (2, 1), 3, (10, 160)),
    (3, 12, 300, (3, 1), (3, 1), 2, (20, 280)),
    (4, 30, 100, (1, 1), (2, 1), 5, (11, 100)),
]
