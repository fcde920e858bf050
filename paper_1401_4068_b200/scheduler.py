"""Multi-GPU chunk scheduler: independent chunks sharded across ranks, one gather.

The reference has no distributed layer (batch_search is a
sequential Python loop, engine.py:210-216; analyze_pairs loops over pairs,
inference.py:203-216).  Here one process drives one GPU (torchrun); every
rank derives the same work list, permutations and jitter states from the
config (pure functions of the seeds, inference.py:101-102,148,161-172),
computes only its LPT share of the (pair, window, u, surrogate) chunks, and
the per-chunk fp64 TE values travel in ONE fixed-size all_gather together
with the per-chunk status codes (KB-scale: latency-, not bandwidth-bound).
Per-chunk results do not depend on placement, so any world size gives
identical bits, and errors are raised on every rank in the reference's
order (the lowest failing item of the reference's sequential loop).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np
import torch

# status of an item whose rank failed outside the per-chunk checks
# (e.g. a CUDA error); the owning rank re-raises its own exception
STATUS_RANK_FAILED = -1


def lpt_partition(costs, world: int):
    """Longest-processing-time-first assignment of items to `world` bins (deterministic).

    Equal costs (every chunk of an analysis has the same shape) give the
    same makespan as contiguous balanced blocks, which keep each rank's
    items of one pair together; that case is computed directly."""
    c = np.asarray(costs, dtype=np.float64)
    if c.size and np.all(c == c[0]):
        sizes = [c.size // world + (1 if r < c.size % world else 0) for r in range(world)]
        edges = np.concatenate([[0], np.cumsum(sizes)])
        return [list(range(int(edges[r]), int(edges[r + 1]))) for r in range(world)]
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


def exchange(values, status, bins, dist, group=None, device=None):
    """The single collective: every rank contributes a [cap, 2] fp64 block
    (TE value, status code) for its bin, cap = the largest bin (known to
    every rank, the bins being deterministic), in ONE all_gather_into_tensor.
    Returns (values, status) of all items in input order."""
    world = len(bins)
    cap = max(1, max(len(b) for b in bins))
    dev = device if device is not None else torch.device("cpu")
    mine = torch.zeros((cap, 2), dtype=torch.float64)
    n = len(values)
    if n:
        mine[:n, 0] = torch.from_numpy(np.asarray(values, dtype=np.float64))
        mine[:n, 1] = torch.from_numpy(np.asarray(status, dtype=np.float64))
    mine = mine.to(dev)
    out = torch.empty((world * cap, 2), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, mine, group=group)
    out = out.cpu().numpy()
    total = sum(len(b) for b in bins)
    vals = np.empty(total)
    st = np.zeros(total, dtype=np.int32)
    for r, b in enumerate(bins):
        if b:
            vals[b] = out[r * cap:r * cap + len(b), 0]
            st[b] = out[r * cap:r * cap + len(b), 1].astype(np.int32)
    return vals, st


def sharded_run(run_fn, items, costs, dist, device=None, group=None):
    """Run `run_fn(list_of_items) -> (values, status)` on this rank's LPT share
    and exchange; returns (values, status) of all items in input order on
    every rank.  A rank whose run_fn raises marks its items
    STATUS_RANK_FAILED instead of skipping the collective (no rank blocks),
    and re-raises after the exchange."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bins = lpt_partition(costs, world)
    mine = bins[rank]
    err = None
    if mine:
        try:
            share = items[np.asarray(mine)] if isinstance(items, np.ndarray) else \
                [items[i] for i in mine]
            vals, st = run_fn(share)
        except Exception as exc:  # noqa: BLE001 - re-raised below, after the collective
            err = exc
            vals = np.zeros(len(mine))
            st = np.full(len(mine), STATUS_RANK_FAILED, dtype=np.int32)
    else:
        vals, st = np.empty(0), np.zeros(0, dtype=np.int32)
    vals, st = exchange(vals, st, bins, dist, group, device)
    if err is not None:
        raise err
    if (st == STATUS_RANK_FAILED).any():
        owner = next(r for r, b in enumerate(bins) if b and st[b[0]] == STATUS_RANK_FAILED)
        raise RuntimeError(f"rank {owner} failed while computing its chunks")
    return vals, st


def raise_first(status) -> None:
    """Raise the reference exception of the lowest failing item, if any."""
    from .ksg import _raise_status
    bad = np.flatnonzero(np.asarray(status) != 0)
    if bad.size:
        _raise_status(int(status[bad[0]]))


# ---------------------------------------------------------------------------
# planning: every rank builds the same item list, in the reference's order
# ---------------------------------------------------------------------------
@dataclass
class _PairPlan:
    source: object
    target: object
    spec_x: object
    spec_y: object
    windows: list                  # [(t_lo, t_hi)] of config.window's width
    us: list                       # u values with a valid assembly (every window)
    items: list = field(default_factory=list)  # (u, perm_index, t_lo)
    terminal: Exception = None     # raised after the items before it succeed
    m: int = 0
    dim: int = 0


def _plan_pair(source, target, spec_x, spec_y, config, windows, with_surrogates, grid=None):
    """Items of one pair over `windows` in the order the reference's
    per-window analyze_pair calls would compute them (inference.py:143-175),
    truncated at the first error the reference raises before computing."""
    from .data import validate_ensemble
    from .embedding import check_assembly
    from .exceptions import EnteError, InvalidPermutation, KTooLarge
    plan = _PairPlan(source, target, spec_x, spec_y, list(windows), list(config.u_candidates))
    try:
        validate_ensemble(source)
        validate_ensemble(target)
    except EnteError as exc:
        plan.terminal, plan.windows, plan.us = exc, [], []
        return plan
    plan.m = target.n_repetitions * (config.window[1] - config.window[0] + 1)
    plan.dim = 1 + spec_y.dim + spec_x.dim
    s = config.n_surrogates
    grid = grid if grid is not None else (config.test_grid or config.u_candidates)
    for wi, win in enumerate(plan.windows):
        us = list(config.u_candidates)
        for i, u in enumerate(us):
            try:
                check_assembly(source, target, spec_x, spec_y, u, win)
            except EnteError as exc:
                plan.terminal = exc
                us = us[:i]
                break
        if plan.terminal is not None:
            # windows before wi run completely, window wi its originals up to the bad u
            for lo, _ in plan.windows[:wi]:
                plan.items += _window_items(config, lo, with_surrogates, grid)
            plan.items += [(u, -1, win[0]) for u in us]
            plan.windows = plan.windows[:wi]
            break
    # the first computed chunk raises KTooLarge when m <= k (ksg.py:77-78)
    computes = bool(plan.items) or (plan.terminal is None and plan.windows
                                    and len(config.u_candidates) > 0)
    if plan.m <= config.k and computes:
        plan.terminal = KTooLarge(f"need more than k={config.k} pooled points, got {plan.m}")
        plan.items, plan.windows = [], []
        return plan
    if plan.terminal is not None:
        return plan
    if with_surrogates and config.strict_permutation and target.n_repetitions < 2 and s > 0 \
            and plan.windows:
        plan.terminal = InvalidPermutation("strict permutation needs R >= 2")
        plan.items = [(u, -1, plan.windows[0][0]) for u in config.u_candidates]
        plan.windows = []
        return plan
    for lo, _ in plan.windows:
        plan.items += _window_items(config, lo, with_surrogates, grid)
    return plan


def _window_items(config, t_lo, with_surrogates, grid):
    items = [(u, -1, t_lo) for u in config.u_candidates]
    if with_surrogates:
        items += [(u, i, t_lo) for u in grid for i in range(config.n_surrogates)]
    return items


def pipeline_runner(pipes, make_pipe=None):
    """run_fn over an int array of items [n, 4] = (pair, u, perm_index, t_lo):
    each pair's items go through its PairPipeline in one device batch;
    returns (TE values, chunk status codes) in item order."""
    def run(mine):
        mine = np.asarray(mine, dtype=np.int64).reshape(-1, 4)
        vals = np.empty(len(mine))
        st = np.zeros(len(mine), dtype=np.int32)
        for pi in np.unique(mine[:, 0]).tolist():
            sel = np.flatnonzero(mine[:, 0] == pi)
            pipe = pipes.get(pi) if isinstance(pipes, dict) else pipes[pi]
            if pipe is None:
                pipe = make_pipe(pi, bool((mine[sel, 2] >= 0).any()))
                pipes[pi] = pipe
            te, code = pipe.run_status(np.ascontiguousarray(mine[sel, 1:4].astype(np.int32)))
            vals[sel] = te
            st[sel] = code
        return vals, st
    return run


def _run_plans(plans, config, dist, group):
    """Shard every planned item over the group, exchange once, and return the
    per-pair TE arrays; raises the reference's first error on every rank."""
    from .inference import PairPipeline, surrogate_perms
    sizes = [len(p.items) for p in plans]
    flat = np.zeros((sum(sizes), 4), dtype=np.int64)
    costs = np.empty(len(flat))
    pos = 0
    for pi, plan in enumerate(plans):
        if plan.items:
            flat[pos:pos + len(plan.items), 0] = pi
            flat[pos:pos + len(plan.items), 1:] = np.asarray(plan.items, dtype=np.int64)
            costs[pos:pos + len(plan.items)] = chunk_cost(plan.m, plan.dim)
        pos += len(plan.items)

    def make_pipe(pi, needs_perms):
        plan = plans[pi]
        pipe = PairPipeline(plan.source, plan.target, plan.spec_x, plan.spec_y, config)
        if needs_perms:
            pipe.set_perms(surrogate_perms(config.seed, config.n_surrogates,
                                           plan.target.n_repetitions, config.strict_permutation))
        return pipe

    run = pipeline_runner({}, make_pipe)
    device = None
    if len(flat) and dist.get_backend(group) == "nccl":
        device = torch.device("cuda", torch.cuda.current_device())
    vals, st = sharded_run(run, flat, costs, dist, device=device, group=group) if len(flat) else \
        (np.empty(0), np.zeros(0, dtype=np.int32))
    raise_first(st)
    for plan in plans:
        if plan.terminal is not None:
            raise plan.terminal
    out, pos = [], 0
    for n in sizes:
        out.append(vals[pos:pos + n])
        pos += n
    return out


def _plans_until_error(pair_inputs, config, with_surrogates, windows_of=None, grids=None):
    plans = []
    for pi, (src, tgt, sx, sy) in enumerate(pair_inputs):
        wins = windows_of(pi) if windows_of else [tuple(config.window)]
        plan = _plan_pair(src, tgt, sx, sy, config, wins, with_surrogates,
                          grids[pi] if grids else None)
        plans.append(plan)
        if plan.terminal is not None:
            break
    return plans


def _pairs_distributed(pair_inputs, config, dist, group=None):
    """TEResult per (source, target, spec_x, spec_y) pair, every chunk sharded."""
    from .inference import _assemble_result
    s = config.n_surrogates
    if config.scan_statistic != "selected":
        grid = tuple(config.test_grid or config.u_candidates)
        plans = _plans_until_error(pair_inputs, config, True)
        tes = _run_plans(plans, config, dist, group)
        nu = len(config.u_candidates)
        return [_assemble_result(p.source, p.target, config, list(config.u_candidates), grid,
                                 te[:nu], te[nu:].reshape(len(grid), s))
                for p, te in zip(plans, tes)]
    # "selected": the surrogate grid is each pair's own u* (inference.py:153-155),
    # known only after the originals -> two exchanges, errors kept in order
    plans = _plans_until_error(pair_inputs, config, False)
    err1 = None
    try:
        tes = _run_plans(plans, config, dist, group)
        n_ok = len(plans)
    except Exception as exc:  # noqa: BLE001 - pairs before the failing one still run phase 2
        err1 = exc
        tes, n_ok = None, 0
    if err1 is not None:
        # phase 1 failed somewhere: find the last pair whose originals all succeeded by
        # re-running phase 1 pair by pair is wasteful; instead rerun phase 1 without
        # raising to learn the failing pair, then finish the pairs before it
        n_ok = _first_failing_pair(plans, config, dist, group)
        if n_ok == 0:
            raise err1
        tes = _run_plans(plans[:n_ok], config, dist, group)
    us = list(config.u_candidates)
    grids = []
    for te in tes:
        curve = list(zip(us, te))
        grids.append((max(curve, key=lambda ut: (ut[1], -ut[0]))[0],))
    plans2 = []
    for pi in range(n_ok):
        p = plans[pi]
        plan = _PairPlan(p.source, p.target, p.spec_x, p.spec_y, p.windows, us, m=p.m, dim=p.dim)
        if config.strict_permutation and p.target.n_repetitions < 2 and s > 0:
            from .exceptions import InvalidPermutation
            plan.terminal = InvalidPermutation("strict permutation needs R >= 2")
            plans2.append(plan)
            break
        plan.items = [(grids[pi][0], i, config.window[0]) for i in range(s)]
        plans2.append(plan)
    tes2 = _run_plans(plans2, config, dist, group)
    if err1 is not None:
        raise err1
    return [_assemble_result(p.source, p.target, config, us, g, te, te2.reshape(1, s))
            for p, g, te, te2 in zip(plans, grids, tes, tes2)]


def _first_failing_pair(plans, config, dist, group) -> int:
    """Index of the first pair whose phase-1 items fail (all ranks agree)."""
    for pi in range(len(plans)):
        try:
            _run_plans(plans[pi:pi + 1], config, dist, group)
        except Exception:  # noqa: BLE001
            return pi
    return len(plans)


def analyze_pair_distributed(source, target, spec_x, spec_y, config, dist, group=None):
    """analyze_pair (inference.py:120-193) with its (u, surrogate) chunks sharded
    over the process group; the same TEResult on every rank.  "max" statistic:
    one exchange; "selected": one exchange for the originals and one for the
    surrogates of u* (the data-dependent grid)."""
    return _pairs_distributed([(source, target, spec_x, spec_y)], config, dist, group)[0]


def analyze_pairs_distributed(series_by_name: dict, pairs, specs_by_name: dict, config, dist,
                              group=None):
    """analyze_pairs (inference.py:203-216) with every (pair, u, surrogate) chunk
    sharded over the process group: the MEG-shaped workload of the paper (many
    channel pairs x delays x surrogates).  Every rank returns the
    same TEResult list, with the configured family-wise correction."""
    from .inference import correct_multiple
    inputs = [(series_by_name[a], series_by_name[b], specs_by_name[a], specs_by_name[b])
              for a, b in pairs]
    results = _pairs_distributed(inputs, config, dist, group)
    decisions = correct_multiple([r.p_value for r in results], config.alpha, config.correction)
    for r, d in zip(results, decisions):
        r.significant_corrected = bool(d and r.significant)
    return results


def analyze_windows_distributed(source, target, spec_x, spec_y, config, window_starts, dist,
                                group=None):
    """inference.analyze_windows (TE per time point) with every
    (window, u, surrogate) chunk sharded over the process group: one exchange,
    the same TEResult list on every rank, errors in the per-window order."""
    from .inference import _assemble_results, _width
    w = _width(config)
    windows = [(int(t), int(t) + w - 1) for t in window_starts]
    if config.scan_statistic == "selected":
        import dataclasses
        return [analyze_pair_distributed(source, target, spec_x, spec_y,
                                         dataclasses.replace(config, window=win), dist, group)
                for win in windows]
    if not windows:
        return []
    grid = tuple(config.test_grid or config.u_candidates)
    plan = _plan_pair(source, target, spec_x, spec_y, config, windows, True)
    (te,) = _run_plans([plan], config, dist, group)
    us = list(config.u_candidates)
    per_win = len(us) + len(grid) * config.n_surrogates
    te = te.reshape(len(windows), per_win)
    return _assemble_results(source, target, config, windows, us, grid, te[:, :len(us)],
                             te[:, len(us):].reshape(len(windows), len(grid),
                                                     config.n_surrogates))


def batch_search_split(items, k: int, dist, group=None):
    """batch_search with every chunk's references split over the ranks.

    For fewer chunks than GPUs (one 64k-point chunk on 8 GPUs): each rank
    uploads the same chunks, searches its part of every chunk's references
    (ente_search_split) into zeroed outputs, and one sum all_reduce of the
    fp64 distances and int32 counts (exact: every row is written by exactly
    one rank) gives every rank the full, bit-identical result.  Returns
    batch_search's list: NeighborCounts or the slot's exception
    (ShapeMismatch for a bad marginal or mismatched layouts, KTooLarge for k
    outside [1, n-1], engine.py:173-174,196-197), in input order.
    """
    from .engine import NeighborCounts, _upload, column_mask, search_device
    from .exceptions import EnteError, KTooLarge, ShapeMismatch
    from .ksg import _raise_status
    out = [None] * len(items)
    live = []
    first = None
    for i, (chunk, margs) in enumerate(items):
        pts = np.ascontiguousarray(np.asarray(chunk.points, dtype=np.float64))
        n, dim = pts.shape
        try:
            if not 1 <= k <= n - 1:
                raise KTooLarge(f"k={k} must be in [1, n-1] for n={n}")
            masks = tuple(column_mask(cols, dim) for cols in margs)
            if first is None:
                first = (dim, masks)
            elif (dim, masks) != first:
                raise ShapeMismatch("batch_search_split: chunks must share dim and marginals")
            live.append((i, pts))
        except EnteError as exc:
            out[i] = exc
    if live:
        dim, masks = first
        ns = np.array([p.shape[0] for _, p in live], dtype=np.int64)
        rows0 = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)
        dev = _upload([p for _, p in live])
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        eps, counts, status = search_device(dev, rows0, ns, list(masks), k, split=(rank, world))
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(eps, group=group)
            dist.all_reduce(counts, group=group)
            eps_h, cnt_h = eps.cpu().numpy(), counts.cpu().numpy()
        else:  # gloo reduces host tensors
            e, c = eps.cpu(), counts.cpu()
            dist.all_reduce(e, group=group)
            dist.all_reduce(c, group=group)
            eps_h, cnt_h = e.numpy(), c.numpy()
        st = status.cpu().numpy()
        cnt_h = cnt_h.astype(np.int64)
        for (i, _), r0, n, code in zip(live, rows0.tolist(), ns.tolist(), st.tolist()):
            if code != 0:
                try:
                    _raise_status(int(code))
                except EnteError as exc:
                    out[i] = exc
                continue
            out[i] = NeighborCounts(eps_h[r0:r0 + n].copy(),
                                    tuple(cnt_h[m, r0:r0 + n].copy() for m in range(len(masks))))
    return out
