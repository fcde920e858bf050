"""Ragwitz embedding optimisation: oracle pinned to the reference's
_local_predictor_sq_errors, GPU errors and MSE tables bit-exact vs both."""

import numpy as np
import pytest

import oracle
from paper_1401_4068_b200.data import EnsembleSeries


@pytest.mark.parametrize("name", ["smooth", "tied"])
def test_oracle_matches_reference_errors(golden, name):
    g = golden("ragwitz.npz")
    errs = oracle.ragwitz_errors(g[f"{name}_values"], 2, 2, g[f"{name}_anchors_r"],
                                 g[f"{name}_anchors_t"], 4)
    assert np.array_equal(errs, g[f"{name}_errs"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["smooth", "tied"])
def test_gpu_errors_and_table_match_reference(golden, name):
    import torch
    from paper_1401_4068_b200 import _native as nat
    from paper_1401_4068_b200.embedding import optimize_embedding
    g = golden("ragwitz.npz")
    v = g[f"{name}_values"]
    dev = nat.device()
    vals = torch.from_numpy(v).to(dev)
    ar = torch.from_numpy(g[f"{name}_anchors_r"].astype(np.int32)).to(dev)
    at = torch.from_numpy(g[f"{name}_anchors_t"].astype(np.int32)).to(dev)
    err = torch.empty(len(ar), dtype=torch.float64, device=dev)
    nat.check(nat.lib().ente_ragwitz_errors(nat.ptr(vals), v.shape[0], v.shape[1], 2, 2,
                                            nat.ptr(ar), nat.ptr(at), len(ar), 4, nat.ptr(err),
                                            nat.stream_handle()), "ragwitz")
    assert np.array_equal(err.cpu().numpy(), g[f"{name}_errs"])
    spec, table = optimize_embedding(EnsembleSeries("Y", v), [3, 1, 2, 2], [2, 1], k_pred=4,
                                     sample_budget=70, seed=5)
    keys = sorted(table)
    assert np.array_equal(np.array(keys), g[f"{name}_keys"])
    assert np.array_equal(np.array([table[k] for k in keys]), g[f"{name}_mse"])
    assert [spec.dim, spec.delay] == g[f"{name}_best"].tolist()


@pytest.mark.gpu
def test_gpu_matches_oracle_larger():
    import torch
    from paper_1401_4068_b200 import _native as nat
    rng = np.random.default_rng(3)
    v = np.round(np.cumsum(rng.standard_normal((40, 300)), axis=1), 0)  # many ties
    for d, tau, k in ((1, 1, 4), (3, 2, 4), (5, 1, 7)):
        span_lo = (d - 1) * tau
        ar = rng.integers(0, 40, 50).astype(np.int32)
        at = rng.integers(span_lo, 299, 50).astype(np.int32)
        dev = nat.device()
        err = torch.empty(50, dtype=torch.float64, device=dev)
        vals, ar_d, at_d = (torch.from_numpy(a).to(dev) for a in (v, ar, at))  # keep alive
        nat.check(nat.lib().ente_ragwitz_errors(nat.ptr(vals), 40, 300, d, tau, nat.ptr(ar_d),
                                                nat.ptr(at_d), 50, k, nat.ptr(err),
                                                nat.stream_handle()), "ragwitz")
        assert np.array_equal(err.cpu().numpy(), oracle.ragwitz_errors(v, d, tau, ar, at, k))
