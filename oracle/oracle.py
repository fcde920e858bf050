"""CPU oracle for the ensemble-TE hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker or the CPU
baseline.  The product package (paper_1401_4068_b200) never imports it.

Parity status: PINNED.  Every function below is checked against golden
vectors produced by running the reference itself (tests/golden/make_golden.py,
fixtures in tests/golden/*.npz|json) by tests/test_oracle.py.

Restatements (reference = /root/reference/pkg/src/ente):
  kth_distances / radius_counts / batch_search
        -> engine.py:70-216 via the C sweep in oracle/ente_oracle.c
  jittered_joint   -> ksg.py:52-59   (numpy Generator.uniform, column std)
  te_from_counts   -> ksg.py:39-49   (scipy digamma, sort, numpy mean)
  estimate_te_batch-> ksg.py:66-90
  assemble         -> embedding.py:75-120
  permuted_joint   -> inference.py:105-117
  draw_permutation -> inference.py:41-49
  analyze_pair     -> inference.py:120-193 (+ permutation_pvalue 62-74)
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
from scipy import special

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    path = os.path.join(HERE, "libente_oracle.so")
    src = os.path.join(HERE, "ente_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return path


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.oracle_kth_sweep.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_kth_brute.argtypes = [dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, dp]
        L.oracle_count_sweep.argtypes = [dp, ctypes.c_int64, ctypes.c_int, i32p, ctypes.c_int,
                                         dp, ip]
        L.oracle_count_brute.argtypes = [dp, ctypes.c_int64, ctypes.c_int, i32p, ctypes.c_int,
                                         dp, ip]
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def kth_distances(points, k, brute=False):
    p = np.ascontiguousarray(points, dtype=np.float64)
    n, d = p.shape
    eps = np.empty(n)
    fn = lib().oracle_kth_brute if brute else lib().oracle_kth_sweep
    if fn(_dp(p), n, d, int(k), _dp(eps)) != 0:
        raise ValueError(f"k={k} not in [1, n-1] for n={n}")
    return eps


def radius_counts(points, cols, radii, brute=False):
    p = np.ascontiguousarray(points, dtype=np.float64)
    n, d = p.shape
    c = np.ascontiguousarray(cols, dtype=np.int32)
    r = np.ascontiguousarray(radii, dtype=np.float64)
    out = np.empty(n, dtype=np.int64)
    fn = lib().oracle_count_brute if brute else lib().oracle_count_sweep
    rc = fn(_dp(p), n, d, c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), c.size, _dp(r),
            out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc != 0:
        raise ValueError("bad marginal columns")
    return out


def search(points, marginals, k, brute=False):
    """(kth_distance, [counts per marginal]) -- engine.py:191-200."""
    eps = kth_distances(points, k, brute)
    return eps, [radius_counts(points, m, eps, brute) for m in marginals]


def knn_indices(points, k):
    """O(n^2) canonical k nearest neighbours: ascending (fp64 max-norm, index), self excluded.

    The reference keeps only the k-th distance (engine.py:70-123); the index
    order is this package's contract, stated by brute force."""
    p = np.asarray(points, dtype=np.float64)
    n = len(p)
    out = np.empty((n, k), dtype=np.int64)
    idx = np.arange(n)
    for i in range(n):
        d = np.abs(p - p[i]).max(axis=1)
        d[i] = np.inf
        order = np.lexsort((idx, d))  # primary d, then index
        out[i] = order[:k]
    return out


def jittered_joint(joint, amplitude, seed):
    """ksg.py:52-59: joint + U(-1,1) * (amplitude * std(axis=0))."""
    out = np.array(joint, dtype=np.float64, copy=True)
    if amplitude > 0:
        gen = np.random.default_rng(seed)
        half = amplitude * out.std(axis=0)
        out += gen.uniform(-1.0, 1.0, size=out.shape) * half
    return out


def te_from_counts(k, a, b, c):
    """ksg.py:39-49: psi(k) + mean(sort(psi(a+1) - psi(b+1) - psi(c+1)))."""
    terms = (special.digamma(np.asarray(a) + 1.0) - special.digamma(np.asarray(b) + 1.0)
             - special.digamma(np.asarray(c) + 1.0))
    return float(special.digamma(k) + np.mean(np.sort(terms)))


def te_margs(d_y, d_x):
    return [list(range(1, 1 + d_y)), list(range(0, 1 + d_y)), list(range(1, 1 + d_y + d_x))]


def estimate_te(joint, d_y, d_x, k, amplitude, seed, brute=False):
    """ksg.py:66-90 for one bundle."""
    j = jittered_joint(joint, amplitude, seed)
    if j.shape[0] <= k:
        raise ValueError("KTooLarge")
    if np.ptp(j, axis=0).max() == 0.0:
        raise ValueError("DegenerateData")
    _, (a, b, c) = search(j, te_margs(d_y, d_x), k, brute)
    return te_from_counts(k, a, b, c)


def assemble(xv, yv, spec_x, spec_y, u, window):
    """embedding.py:75-120 joint matrix [y_t | y-past | x-past], rep-outer/time-inner."""
    (dx, tx), (dy, ty) = spec_x, spec_y
    t_lo, t_hi = window
    times = np.arange(t_lo, t_hi + 1)
    reps = yv.shape[0]
    m = reps * times.size
    joint = np.empty((m, 1 + dy + dx))
    joint[:, 0] = yv[:, times - 1].reshape(m)
    for j in range(dy):
        joint[:, 1 + j] = yv[:, times - 2 - j * ty].reshape(m)
    for j in range(dx):
        joint[:, 1 + dy + j] = xv[:, times - 1 - u - j * tx].reshape(m)
    return joint


def permuted_joint(joint, perm, w, d_y):
    """inference.py:105-117: y columns take block rows perm[r]*w + t."""
    rows = (np.asarray(perm)[:, None] * w + np.arange(w)[None, :]).ravel()
    out = joint.copy()
    out[:, :1 + d_y] = joint[rows, :1 + d_y]
    return out


def draw_permutation(reps, seed, strict=True):
    """inference.py:41-49."""
    gen = np.random.default_rng(seed)
    while True:
        perm = gen.permutation(reps)
        if not strict or not np.any(perm == np.arange(reps)):
            return perm


def analyze_pair(xv, yv, spec_x, spec_y, u_candidates, window, k=4, n_surrogates=500,
                 seed=0, amplitude=1e-8, strict=True, test_grid=None, scan_statistic="max",
                 conservative=False):
    """inference.py:120-193 (statistics restated; returns a plain dict)."""
    grid = None if scan_statistic == "selected" else (test_grid or tuple(u_candidates))
    curve, joints = [], {}
    for u in u_candidates:
        joint = assemble(xv, yv, spec_x, spec_y, u, window)
        te = estimate_te(joint, spec_y[0], spec_x[0], k, amplitude,
                         np.random.SeedSequence((seed, u, 0)))
        curve.append((u, te))
        if grid is None or u in grid:
            joints[u] = joint
    u_best, te_best = max(curve, key=lambda ut: (ut[1], -ut[0]))
    if grid is None:
        grid = (u_best,)
        stat = te_best
    else:
        stat = max(te for u, te in curve if u in grid)
    perms = [draw_permutation(yv.shape[0], np.random.SeedSequence((seed, i)), strict)
             for i in range(n_surrogates)]
    w = window[1] - window[0] + 1
    surr = np.full(n_surrogates, -np.inf)
    for u in grid:
        vals = [estimate_te(permuted_joint(joints[u], p, w, spec_y[0]), spec_y[0], spec_x[0], k,
                            amplitude, np.random.SeedSequence((seed, u, i + 1)))
                for i, p in enumerate(perms)]
        np.maximum(surr, vals, out=surr)
    cnt = int(np.sum(surr >= stat))
    p = (cnt + 1) / (n_surrogates + 1) if conservative else cnt / n_surrogates
    return {"u_selected": u_best, "te_value": te_best, "te_curve": curve,
            "surrogate_values": surr, "p_value": p}


def ragwitz_errors(values, d, tau, anchors_r, anchors_t, k_pred):
    """embedding.py:123-165 restated: k_pred nearest cross-repetition embedded points in
    lexicographic (max-norm distance, scan position r2 asc / t2 asc) order; the
    prediction sums their next samples in that order, / k_pred; squared error."""
    v = np.asarray(values, dtype=np.float64)
    n_rep, n_samp = v.shape
    span_lo = (d - 1) * tau
    t2 = np.arange(span_lo, n_samp - 1)
    errs = np.empty(len(anchors_r))
    for a, (r0, t0) in enumerate(zip(anchors_r, anchors_t)):
        ref = v[r0, t0 - tau * np.arange(d)]
        others = [r for r in range(n_rep) if r != r0]
        emb = np.stack([v[others][:, t2 - c * tau] for c in range(d)], axis=-1)  # [R-1, T, d]
        dist = np.abs(emb - ref).max(axis=-1).ravel()
        nxt = v[others][:, t2 + 1].ravel()
        order = np.argsort(dist, kind="stable")[:k_pred]  # stable = scan order on ties
        pred = 0.0
        for q in order:
            pred += nxt[q]
        pred /= k_pred
        diff = pred - v[r0, t0 + 1]
        errs[a] = diff * diff
    return errs
