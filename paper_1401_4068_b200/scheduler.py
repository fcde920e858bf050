"""Multi-GPU chunk scheduler: independent chunks sharded across ranks, one gather.

The reference has no distributed layer (batch_search is a
sequential Python loop, engine.py:210-216).  Here one process drives one GPU
(torchrun); every rank derives the same work list, permutations and jitter
states from the config (they are pure functions of the seeds,
inference.py:101-102,148,161-172), computes only its LPT share of the
(u, surrogate) chunks, and the per-chunk fp64 TE values are exchanged in a
single all_gather (KB-scale: latency-, not bandwidth-bound).  Per-chunk
results do not depend on placement, so any world size gives identical bits.
"""

from __future__ import annotations

import heapq

import numpy as np
import torch


def lpt_partition(costs, world: int):
    """Longest-processing-time-first assignment of items to `world` bins (deterministic)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    bins = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        bins[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(b) for b in bins]


def chunk_cost(n_points: int, dim: int) -> float:
    """Brute-force work of one chunk: 2 passes over ordered pairs x columns."""
    return 2.0 * dim * n_points * (n_points - 1)


def gather_te(values: torch.Tensor, dist, group=None) -> torch.Tensor:
    """all_gather of a variable-length fp64 vector; returns the rank-ordered concatenation."""
    world = dist.get_world_size(group)
    n = torch.tensor([values.numel()], dtype=torch.int64, device=values.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    padded = torch.zeros(cap, dtype=values.dtype, device=values.device)
    padded[:values.numel()] = values
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def sharded_run(run_fn, items, costs, dist, device=None, group=None) -> np.ndarray:
    """Run `run_fn(list_of_items) -> np.ndarray` on this rank's LPT share and gather.

    Returns the TE values of all items in input order on every rank.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bins = lpt_partition(costs, world)
    mine = bins[rank]
    local = run_fn([items[i] for i in mine]) if mine else np.empty(0)
    dev = device if device is not None else torch.device("cpu")
    vals = gather_te(torch.as_tensor(np.asarray(local, dtype=np.float64), device=dev), dist, group)
    ids = np.concatenate([np.asarray(b, dtype=np.int64) for b in bins])
    out = np.empty(len(items))
    out[ids] = vals.cpu().numpy()
    return out


def analyze_pair_distributed(source, target, spec_x, spec_y, config, dist, group=None):
    """analyze_pair with its (u, surrogate) chunks sharded over the process group.

    Same TEResult as inference.analyze_pair on every rank.  Supports the
    default "max" scan statistic (one exchange); "selected" falls back to the
    single-GPU call on every rank.
    """
    from .inference import PairPipeline, analyze_pair, cached_permutation, permutation_pvalue
    from .data import TEResult, validate_ensemble
    if config.scan_statistic != "max":
        return analyze_pair(source, target, spec_x, spec_y, config)
    validate_ensemble(source)
    validate_ensemble(target)
    grid = config.test_grid or config.u_candidates
    pipe = PairPipeline(source, target, spec_x, spec_y, config)
    s = config.n_surrogates
    pipe.set_perms([cached_permutation(config.seed, i, target.n_repetitions,
                                       config.strict_permutation) for i in range(s)])
    items = [(u, -1) for u in config.u_candidates] + [(u, i) for u in grid for i in range(s)]
    costs = [chunk_cost(pipe.m, pipe.dim)] * len(items)
    te = sharded_run(pipe.run, items, costs, dist, device=pipe.x.device, group=group)
    nu = len(config.u_candidates)
    curve = [(u, float(t)) for u, t in zip(config.u_candidates, te[:nu])]
    u_best, te_best = max(curve, key=lambda ut: (ut[1], -ut[0]))
    stat = max(t for u, t in curve if u in grid)
    surr = te[nu:].reshape(len(grid), s).max(axis=0)
    p = permutation_pvalue(stat, surr, config.conservative_pvalue)
    sig = p < config.alpha
    return TEResult(source=source.channel_name, target=target.channel_name, window=config.window,
                    u_selected=u_best, te_value=te_best, surrogate_values=surr, p_value=p,
                    significant=sig, significant_corrected=sig,
                    te_minus_median_surrogate=te_best - float(np.median(surr)), te_curve=curve)
