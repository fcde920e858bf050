"""Ragwitz fixtures from the REFERENCE package (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_ragwitz_golden.py

Calls ente.embedding._local_predictor_sq_errors and optimize_embedding
(/root/reference/pkg/src/ente/embedding.py:123-210) on two small seeded
ensembles (one with heavy ties) and stores the per-anchor squared errors and
the MSE tables in tests/golden/ragwitz.npz.
"""
import os

import numpy as np

from ente.data import EnsembleSeries
from ente.embedding import _local_predictor_sq_errors, optimize_embedding

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}
for name, rounding in (("smooth", None), ("tied", 1)):
    rng = np.random.default_rng(11)
    v = np.cumsum(rng.standard_normal((9, 140)), axis=1) * 0.3
    if rounding is not None:
        v = np.round(v, rounding)
    out[f"{name}_values"] = v
    spec, table = optimize_embedding(EnsembleSeries("Y", v), [1, 2, 3], [1, 2], k_pred=4,
                                     sample_budget=70, seed=5)
    keys = sorted(table)
    out[f"{name}_keys"] = np.array(keys)
    out[f"{name}_mse"] = np.array([table[k] for k in keys])
    out[f"{name}_best"] = np.array([spec.dim, spec.delay])
    # raw errors for one candidate with explicit anchors (every anchor of two repetitions)
    d, tau = 2, 2
    span_lo = (d - 1) * tau
    ar = np.repeat(np.array([0, 4]), 140 - 1 - span_lo).astype(np.int64)
    at = np.tile(np.arange(span_lo, 139), 2).astype(np.int64)
    out[f"{name}_anchors_r"] = ar
    out[f"{name}_anchors_t"] = at
    out[f"{name}_errs"] = _local_predictor_sq_errors(v, d, tau, ar, at, 4)
np.savez(os.path.join(HERE, "ragwitz.npz"), **out)
print("wrote ragwitz.npz")
