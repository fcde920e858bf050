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


def analyze_pairs_distributed(series_by_name: dict, pairs, specs_by_name: dict, config, dist,
                              group=None):
    """analyze_pairs with every (pair, u, surrogate) chunk sharded over the process group.

    The MEG-shaped workload of the paper (many channel pairs x delays x
    surrogates): all ranks build the same item list, run their
    LPT share pair by pair (one device batch per pair), exchange the TE values
    in one all_gather, and assemble the same TEResult list (plus the
    configured family-wise correction, inference.py:203-216) on every rank.
    "max" scan statistic only (one exchange); "selected" runs analyze_pairs.
    """
    from .inference import (PairPipeline, _assemble_result, analyze_pairs, cached_permutation,
                            correct_multiple)
    from .data import validate_ensemble
    if config.scan_statistic != "max":
        return analyze_pairs(series_by_name, pairs, specs_by_name, config)
    grid = tuple(config.test_grid or config.u_candidates)
    us = tuple(config.u_candidates)
    s = config.n_surrogates
    per_pair = [(u, -1) for u in us] + [(u, i) for u in grid for i in range(s)]
    items, costs, pipes = [], [], {}
    for pi, (a, b) in enumerate(pairs):
        validate_ensemble(series_by_name[a])
        validate_ensemble(series_by_name[b])
        m = series_by_name[b].n_repetitions * (config.window[1] - config.window[0] + 1)
        dim = 1 + specs_by_name[a].dim + specs_by_name[b].dim
        for u, i in per_pair:
            items.append((pi, u, i))
            costs.append(chunk_cost(m, dim))

    def run(mine):
        out = np.empty(len(mine))
        by_pair = {}
        for slot, (pi, u, i) in enumerate(mine):
            by_pair.setdefault(pi, []).append((slot, u, i))
        for pi, rows in by_pair.items():
            a, b = pairs[pi]
            pipe = pipes.get(pi)
            if pipe is None:
                src, tgt = series_by_name[a], series_by_name[b]
                pipe = PairPipeline(src, tgt, specs_by_name[a], specs_by_name[b], config)
                pipe.set_perms([cached_permutation(config.seed, i, tgt.n_repetitions,
                                                   config.strict_permutation) for i in range(s)])
                pipes[pi] = pipe
            te = pipe.run([(u, i) for _, u, i in rows])
            out[[slot for slot, _, _ in rows]] = te
        return out

    device = None
    if dist.get_backend(group) == "nccl":
        device = torch.device("cuda", torch.cuda.current_device())
    te = sharded_run(run, items, costs, dist, device=device, group=group)
    te = te.reshape(len(pairs), len(per_pair))
    results = []
    for pi, (a, b) in enumerate(pairs):
        row = te[pi]
        results.append(_assemble_result(series_by_name[a], series_by_name[b], config, list(us),
                                        grid, row[:len(us)], row[len(us):].reshape(len(grid), s)))
    decisions = correct_multiple([r.p_value for r in results], config.alpha, config.correction)
    for r, d in zip(results, decisions):
        r.significant_corrected = bool(d and r.significant)
    return results


def batch_search_split(items, k: int, dist, group=None):
    """batch_search with every chunk's references split over the ranks.

    For fewer chunks than GPUs (one 64k-point chunk on 8 GPUs): each rank
    uploads the same chunks, searches its part of every chunk's references
    (ente_search_split) into zeroed outputs, and one sum all_reduce of the
    fp64 distances and int32 counts (exact: every row is written by exactly
    one rank) gives every rank the full, bit-identical result.  Chunks must
    share (dim, marginals); returns NeighborCounts in input order.
    """
    from .engine import Chunk, NeighborCounts, _upload, column_mask, search_device
    pts = [np.ascontiguousarray(np.asarray(c.points, dtype=np.float64)) for c, _ in items]
    dim = pts[0].shape[1]
    margs = items[0][1]
    masks = [column_mask(cols, dim) for cols in margs]
    ns = np.array([p.shape[0] for p in pts], dtype=np.int64)
    rows0 = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)
    dev = _upload(pts)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    eps, counts, status = search_device(dev, rows0, ns, masks, k, split=(rank, world))
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(eps, group=group)
        dist.all_reduce(counts, group=group)
        eps_h, cnt_h = eps.cpu().numpy(), counts.cpu().numpy()
    else:  # gloo reduces host tensors
        e, c = eps.cpu(), counts.cpu()
        dist.all_reduce(e, group=group)
        dist.all_reduce(c, group=group)
        eps_h, cnt_h = e.numpy(), c.numpy()
    cnt_h = cnt_h.astype(np.int64)
    out = []
    for r0, n in zip(rows0.tolist(), ns.tolist()):
        out.append(NeighborCounts(eps_h[r0:r0 + n].copy(),
                                  tuple(cnt_h[m, r0:r0 + n].copy() for m in range(len(masks)))))
    return out
