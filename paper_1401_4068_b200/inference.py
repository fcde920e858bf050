"""Surrogate testing and delay scanning; every TE of a pair in one device batch.

Drop-in for /root/reference/pkg/src/ente/inference.py: SurrogateSpec 27-38,
draw_permutation 41-49, shuffle_target 52-59, permutation_pvalue 62-74,
correct_multiple 77-98, _surrogate_seed 101-102, _permuted_bundle 105-117,
analyze_pair 120-193, scan_delays 196-200, analyze_pairs 203-216.

analyze_pair differs from the reference only in HOW it computes: instead of
one estimate_te_batch call per u (inference.py:147,173) it packs every
(u, surrogate) chunk on the device from the two ensembles (ente_pack_te),
jitters, searches and reduces them in one pipeline, then runs the same host
statistics.  Permutations and jitter states are derived exactly as the
reference derives them (numpy SeedSequence / Generator) and cached per
(seed, index), so repeated windows and pairs reuse them.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import seeds
from .data import AnalysisConfig, EnsembleSeries, TEResult, validate_ensemble
from .embedding import EmbeddingSpec, PointSetBundle, check_assembly
from .engine import SharedY
from .exceptions import EnteError, InvalidPermutation, KTooLarge, UnknownMethod
from .ksg import _raise_status, te_chunks_device

# rows per device wave (fp64 joint + fp32 copies + counts + events + tie copy ~ 300 B/row: ~40 GB)
MAX_ROWS_PER_WAVE = 1 << 27
# a wave runs as up to SUB_BATCHES sub-batches on two streams (>= MIN_SUB_BATCH chunks each)
SUB_BATCHES = int(os.environ.get("ENTE_SUB_BATCHES", "1"))
MIN_SUB_BATCH = 64
# batches of one window count the y marginals once per target point
# (ente_search_te_shared); ENTE_SHARED_Y=0 sweeps every chunk (A/B, tests)
SHARED_Y = os.environ.get("ENTE_SHARED_Y", "1") != "0"


@dataclass(frozen=True)
class SurrogateSpec:
    """A repetition permutation phi (0-based) and the seed it came from."""

    permutation: np.ndarray
    seed: object = None

    def __post_init__(self):
        perm = np.asarray(self.permutation, dtype=np.int64)
        object.__setattr__(self, "permutation", perm)
        if perm.ndim != 1 or not np.array_equal(np.sort(perm), np.arange(perm.size)):
            raise InvalidPermutation("not a bijection on {0..R-1}")


def draw_permutation(n_repetitions: int, seed, strict: bool = True) -> SurrogateSpec:
    """numpy permutation of range(R); with strict, redrawn until phi(r) != r for all r."""
    if strict and n_repetitions < 2:
        raise InvalidPermutation("strict permutation needs R >= 2")
    gen = np.random.default_rng(seed)
    ident = np.arange(n_repetitions)
    perm = gen.permutation(n_repetitions)
    while strict and (perm == ident).any():
        perm = gen.permutation(n_repetitions)
    return SurrogateSpec(perm, seed)


def shuffle_target(target: EnsembleSeries, spec: SurrogateSpec) -> EnsembleSeries:
    """Target with repetition r replaced by repetition phi(r) (input untouched)."""
    if spec.permutation.size != target.n_repetitions:
        raise InvalidPermutation(
            f"permutation length {spec.permutation.size} != R={target.n_repetitions}")
    return EnsembleSeries(target.channel_name, target.values[spec.permutation],
                          target.sample_rate)


def permutation_pvalue(te_original: float, te_surrogates, conservative: bool = False) -> float:
    surr = np.asarray(te_surrogates, dtype=np.float64)
    if surr.size < 1:
        raise ValueError("need at least one surrogate value")
    hits = int(np.count_nonzero(surr >= te_original))
    return (hits + 1) / (surr.size + 1) if conservative else hits / surr.size


def correct_multiple(pvalues, alpha: float, method: str = "bonferroni"):
    """Family-wise decisions: none (p < a), bonferroni (p < a/m), fdr (BH step-up)."""
    p = np.asarray(pvalues, dtype=np.float64)
    m = p.size
    if method == "none":
        return (p < alpha).tolist()
    if method == "bonferroni":
        return (p < alpha / m).tolist()
    if method == "fdr":
        ranked = np.sort(p, kind="stable")
        ok = np.flatnonzero(ranked <= alpha * np.arange(1, m + 1) / m)
        if ok.size == 0:
            return [False] * m
        return (p <= ranked[ok[-1]]).tolist()
    raise UnknownMethod(f"unknown correction method {method!r}")


def _surrogate_seed(master_seed, index: int):
    return np.random.SeedSequence((master_seed, index))


def _permuted_bundle(bundle: PointSetBundle, permutation: np.ndarray,
                     window_width: int) -> PointSetBundle:
    """Host form of the surrogate joint: y columns take block rows perm[r]*w + t."""
    src_rows = (np.asarray(permutation)[:, None] * window_width
                + np.arange(window_width)[None, :]).reshape(-1)
    joint = bundle.joint.copy()
    ny = 1 + bundle.d_y
    joint[:, :ny] = bundle.joint[src_rows, :ny]
    return PointSetBundle(joint, bundle.d_y, bundle.d_x, bundle.row_origin)


# ---------------------------------------------------------------------------
# random streams: native batch derivation (csrc/seeds.cu), bit-equal to numpy
# ---------------------------------------------------------------------------
def surrogate_perms(master_seed, count: int, reps: int, strict: bool) -> np.ndarray:
    """The S = count surrogate permutations of analyze_pair, [count, reps] int32:
    draw_permutation(reps, SeedSequence((master_seed, i)), strict) for i < count
    (inference.py:101-102, 161-164), drawn natively in one call."""
    if strict and reps < 2 and count > 0:
        raise InvalidPermutation("strict permutation needs R >= 2")
    return seeds.surrogate_permutations(master_seed, count, reps, strict)


def cached_permutation(master_seed, idx: int, reps: int, strict: bool) -> np.ndarray:
    """Surrogate permutation idx alone (int64, as draw_permutation returns it)."""
    if strict and reps < 2:
        raise InvalidPermutation("strict permutation needs R >= 2")
    return seeds.surrogate_permutations_at(master_seed, [idx], reps, strict)[0].astype(np.int64)


def jitter_state(seed_tuple) -> tuple:
    """PCG64 (state, inc) of default_rng(SeedSequence(seed_tuple)) as 4 uint64."""
    return tuple(int(v) for v in seeds.pcg_states([np.random.SeedSequence(seed_tuple)])[0])


class PairPipeline:
    """Device pipeline for the chunks of one (source, target) pair.

    run(items) takes (u, perm_index) items (perm_index -1 = original data),
    or (u, perm_index, t_lo) items whose window starts at sample t_lo (all
    windows config.window's width), and returns their TE values in order;
    errors are raised for the first failing item, as the reference's per-u
    estimate_te_batch calls would.
    """

    def __init__(self, source, target, spec_x, spec_y, config: AnalysisConfig,
                 x_device=None, y_device=None):
        self.cfg = config
        self._pinned_keep = []  # pinned jitter-state buffers of the wave in flight
        self.sx, self.sy = spec_x, spec_y
        self.reps, self.n_samples = target.values.shape
        self.t_lo, self.t_hi = config.window
        self.w = self.t_hi - self.t_lo + 1
        self.m = self.reps * self.w
        self.dim = 1 + spec_y.dim + spec_x.dim
        dev = nat.device()
        # x_device / y_device: the ensembles already in HBM (io_formats.load_ensemble_device)
        self.x = x_device if x_device is not None else \
            torch.from_numpy(np.array(source.values, dtype=np.float64)).to(dev)
        self.y = y_device if y_device is not None else \
            torch.from_numpy(np.array(target.values, dtype=np.float64)).to(dev)
        self.perm_dev = None
        self.inv_perm_dev = None
        self.perm_count = 0
        self.target_values = np.asarray(target.values, dtype=np.float64)
        self.source_values = np.asarray(source.values, dtype=np.float64)
        self._shared = {}

    def set_perms(self, perms):
        arr = np.ascontiguousarray(np.asarray(perms, dtype=np.int32).reshape(-1, self.reps))
        self.perm_dev = torch.from_numpy(arr).to(nat.device())
        inv = np.empty_like(arr)
        np.put_along_axis(inv, arr.astype(np.int64), np.arange(self.reps, dtype=np.int32)[None, :], 1)
        self.inv_perm_dev = torch.from_numpy(np.ascontiguousarray(inv)).to(nat.device())
        self.perm_count = len(perms)

    def shared_pays(self, t_lo: int, u: int) -> bool:
        """Whether the shared-y search is the faster one for this window: its m3
        / joint sweeps walk the principal-axis order, which only embedded
        low-dimensional dynamics get (the test the device applies per chunk:
        variance off the two leading principal axes < 5 % of the first,
        >= 4096 points; here on every 4th repetition of the window's first
        chunk).  Noise-driven data keeps the fused sweep."""
        key = ("pays", t_lo)
        hit = self._shared.get(key)
        if hit is None:
            hit = False
            if self.m >= 4096:
                yv, xv = self.target_values[::4], self.source_values[::4]
                times = np.arange(t_lo, t_lo + self.w)
                cols = [yv[:, times - 1]] + [yv[:, times - 2 - j * self.sy.delay]
                                             for j in range(self.sy.dim)]
                cols += [xv[:, times - 1 - u - j * self.sx.delay] for j in range(self.sx.dim)]
                joint = np.stack([c.reshape(-1) for c in cols[:8]], axis=1)
                lam = np.sort(np.linalg.eigvalsh(np.cov(joint, rowvar=False)))[::-1]
                hit = bool(lam[0] > 0 and lam[2:].sum() < 0.05 * lam[0])
            self._shared[key] = hit
        return hit

    def shared_y(self, t_lo: int, perm_index):
        """SharedY of the window starting at t_lo (every chunk of the window
        pools the same target rows): the unjittered y columns
        (embedding.py:109-113), gathered on the device from the resident
        target, and the jitter margin 2 hw + rounding, hw = amplitude x the
        columns' std (ksg.py:52-59)."""
        hit = self._shared.get(t_lo)
        if hit is None:
            yv = self.target_values
            times = np.arange(t_lo, t_lo + self.w)
            idx = [times - 1] + [times - 2 - j * self.sy.delay for j in range(self.sy.dim)]
            hw = self.cfg.jitter_amplitude * max(float(yv[:, ix].std()) for ix in idx) * (1.0 + 1e-9)
            vmax = max(float(np.abs(yv[:, ix]).max()) for ix in idx)
            margin = 2.0 * hw * (1.0 + 1e-12) + 2.0 ** -48 * (vmax + hw)
            cols = torch.from_numpy(np.stack(idx, axis=1).reshape(-1)).to(self.y.device)
            y0 = self.y[:, cols].reshape(self.reps, self.w, len(idx)).reshape(self.m, len(idx))
            hit = (y0.contiguous(), margin)
            self._shared[t_lo] = hit
        y0, margin = hit
        if self.perm_dev is None:
            perms = inv = torch.zeros((1, self.reps), dtype=torch.int32, device=nat.device())
        else:
            perms, inv = self.perm_dev, self.inv_perm_dev
        return SharedY(y0, self.reps, self.w, np.asarray(perm_index, dtype=np.int32), perms, inv,
                       margin)

    def seed_tuple(self, u, perm_index):
        return (self.cfg.seed, u, 0 if perm_index < 0 else perm_index + 1)

    def _items(self, items) -> np.ndarray:
        if isinstance(items, np.ndarray) and items.dtype == np.int32 and items.ndim == 2 \
                and items.shape[1] == 3 and items.flags.c_contiguous:
            return items
        it = np.asarray(items, dtype=np.int64)
        if it.ndim != 2 or it.shape[1] not in (2, 3):
            raise ValueError("items must be (u, perm_index) or (u, perm_index, t_lo) tuples")
        if it.shape[1] == 2:
            it = np.concatenate([it, np.full((len(it), 1), self.t_lo, dtype=np.int64)], axis=1)
        return np.ascontiguousarray(it.astype(np.int32))

    def run(self, items) -> np.ndarray:
        te, st = self.run_status(items)
        if (st != 0).any():
            _raise_status(int(st[np.flatnonzero(st)[0]]))
        return te

    def run_status(self, items):
        """TE values and per-item chunk status codes (0 = ok, else the
        ente_chunk_status the reference would raise for that item); raises
        only for errors common to every item (KTooLarge: m <= k)."""
        if len(items) == 0:
            return np.empty(0), np.zeros(0, dtype=np.int32)
        if self.m <= self.cfg.k:
            raise KTooLarge(f"need more than k={self.cfg.k} pooled points, got {self.m}")
        it = self._items(items)
        per_wave = max(1, MAX_ROWS_PER_WAVE // self.m)
        tes, sts = [], []
        for s in range(0, len(it), per_wave):
            te, st = self._wave(it[s:s + per_wave])
            tes.append(te)
            sts.append(st)
        return np.concatenate(tes), np.concatenate(sts).astype(np.int32)

    def _states(self, it: np.ndarray) -> np.ndarray:
        """Jitter PCG64 states per item: SeedSequence((seed, u, 0 | idx + 1)), independent
        of the window (inference.py:148, 171-172).  Written to pinned memory, so
        ente_jitter's copy of them does not hold the host; the buffer is kept
        until the wave has been read back (_wave clears the list)."""
        buf = torch.empty((len(it), 4), dtype=torch.int64, pin_memory=True)
        out = buf.numpy().view(np.uint64)
        seeds.jitter_states(self.cfg.seed, it[:, 0], it[:, 1].astype(np.int64) + 1, out=out)
        self._pinned_keep.append(buf)
        return out

    def _wave(self, it: np.ndarray):
        """One device batch, split into sub-batches alternating over two CUDA
        streams so that one sub-batch's latency-bound kernels (pack, jitter,
        sorts, gathers, reduction) overlap another's compute-bound sweeps.
        Returns (te, status), read once at the end."""
        n = len(it)
        self._pinned_keep = []  # the previous wave was read back: its staging is free
        nsub = 1 if n < 2 * MIN_SUB_BATCH else min(SUB_BATCHES, n // MIN_SUB_BATCH)
        bounds = np.linspace(0, n, nsub + 1).astype(int)
        main = torch.cuda.current_stream()
        streams = _streams(min(2, nsub))
        outs = []
        for b in range(nsub):
            lo, hi = int(bounds[b]), int(bounds[b + 1])
            stream = streams[b % len(streams)]
            stream.wait_stream(main)
            with torch.cuda.stream(stream):
                outs.append(self._sub(it[lo:hi], f".s{b % len(streams)}"))
        for stream in streams:
            main.wait_stream(stream)
        te = torch.cat([t for t, _ in outs]).cpu().numpy()
        st = torch.cat([s for _, s in outs]).cpu().numpy()
        return te, st

    def _sub(self, it: np.ndarray, tag: str):
        L = nat.lib()
        n = len(it)
        pts = nat.scratch("pipe.joint" + tag, (n * self.m, self.dim), torch.float64)
        perms_ptr = nat.ptr(self.perm_dev) if self.perm_dev is not None else None
        nat.check(L.ente_pack_te_items(nat.ptr(self.x), nat.ptr(self.y), self.reps,
                                       self.n_samples, self.sx.dim, self.sx.delay, self.sy.dim,
                                       self.sy.delay, self.w,
                                       it.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int32)),
                                       n, perms_ptr, nat.ptr(pts), nat.stream_handle()),
                  "ente_pack_te_items")
        states = self._states(it)  # host work while the device packs
        rows0 = np.arange(n, dtype=np.int64) * self.m
        ns = np.full(n, self.m, dtype=np.int64)
        shared = None
        if SHARED_Y and (it[:, 2] == it[0, 2]).all() and self.shared_pays(int(it[0, 2]), int(it[0, 0])):
            shared = self.shared_y(int(it[0, 2]), it[:, 1])  # one window: one target point set
        return te_chunks_device(pts, rows0, ns, self.sy.dim, self.sx.dim, self.cfg.k,
                                self.cfg.jitter_amplitude, np.ascontiguousarray(states),
                                sync=False, tag=tag, shared=shared)


_STREAMS: dict = {}


def _streams(count: int):
    """Per-device side streams for sub-batch overlap (created once)."""
    key = (torch.cuda.current_device(), count)
    s = _STREAMS.get(key)
    if s is None:
        s = [torch.cuda.Stream() for _ in range(count)]
        _STREAMS[key] = s
    return s


def analyze_pair(source: EnsembleSeries, target: EnsembleSeries,
                 spec_x: EmbeddingSpec, spec_y: EmbeddingSpec,
                 config: AnalysisConfig, x_device=None, y_device=None) -> TEResult:
    """Delay scan + surrogate test for one directed pair in one window (TE in nats).

    x_device / y_device optionally pass the two ensembles already resident in
    HBM (same values as source / target), skipping their upload.  Errors are
    raised in the reference's order (inference.py:143-193): the originals of
    the u values before a failing assembly are estimated first.
    """
    validate_ensemble(source)
    validate_ensemble(target)
    selected = config.scan_statistic == "selected"
    grid = None if selected else (config.test_grid or config.u_candidates)
    us = list(config.u_candidates)
    assembly_error = None
    for i, u in enumerate(us):
        try:
            check_assembly(source, target, spec_x, spec_y, u, config.window)
        except EnteError as exc:
            assembly_error = exc
            us = us[:i]
            break
    pipe = PairPipeline(source, target, spec_x, spec_y, config, x_device, y_device)
    reps = target.n_repetitions
    s = config.n_surrogates
    can_draw = reps >= 2 or not config.strict_permutation
    originals = [(u, -1) for u in us]

    if not selected and assembly_error is None and can_draw:
        pipe.set_perms(surrogate_perms(config.seed, s, reps, config.strict_permutation))
        surr_items = [(u, i) for u in grid for i in range(s)]
        te_all = pipe.run(originals + surr_items)
        te_orig = te_all[:len(us)]
        te_surr = te_all[len(us):].reshape(len(grid), s)
    else:
        te_orig = pipe.run(originals)
        if assembly_error is not None:
            raise assembly_error
        if grid is None:
            curve = list(zip(us, te_orig))
            grid = (max(curve, key=lambda ut: (ut[1], -ut[0]))[0],)
        pipe.set_perms(surrogate_perms(config.seed, s, reps, config.strict_permutation))
        te_surr = pipe.run([(u, i) for u in grid for i in range(s)]).reshape(len(grid), s)
    return _assemble_result(source, target, config, us, grid, te_orig, te_surr)


def analyze_windows(source: EnsembleSeries, target: EnsembleSeries, spec_x: EmbeddingSpec,
                    spec_y: EmbeddingSpec, config: AnalysisConfig, window_starts) -> list:
    """analyze_pair for many windows of config.window's width in ONE device batch.

    Equivalent to [analyze_pair(..., replace(config, window=(t, t + w - 1)))
    for t in window_starts] (inference.py:120-193 per window; the seeds do not
    depend on the window, so each window reuses the same permutations and
    jitter streams, exactly as the per-window calls would).  This is the
    non-stationary, TE-per-time-point analysis of the paper: every (window,
    u, surrogate) chunk goes through one pack / jitter / search / reduce
    sequence.  Errors surface in the per-window calls' order: the windows
    before the first failing assembly run first (their own errors win), then
    the failing window's analyze_pair raises.
    """
    validate_ensemble(source)
    validate_ensemble(target)
    w = _width(config)
    windows = [(int(t), int(t) + w - 1) for t in window_starts]
    if config.scan_statistic == "selected":
        return [analyze_pair(source, target, spec_x, spec_y, _at_window(config, win))
                for win in windows]
    for wi, win in enumerate(windows):
        try:
            for u in config.u_candidates:
                check_assembly(source, target, spec_x, spec_y, u, win)
        except EnteError:
            analyze_windows(source, target, spec_x, spec_y, config, window_starts[:wi])
            analyze_pair(source, target, spec_x, spec_y, _at_window(config, win))
            raise  # pragma: no cover (analyze_pair raised above)
    reps, s = target.n_repetitions, config.n_surrogates
    if not windows:
        return []
    if config.strict_permutation and reps < 2:
        # originals of the first window, then InvalidPermutation (inference.py:147,161)
        analyze_pair(source, target, spec_x, spec_y, _at_window(config, windows[0]))
    grid = config.test_grid or config.u_candidates
    us = list(config.u_candidates)
    pipe = PairPipeline(source, target, spec_x, spec_y, config)
    pipe.set_perms(surrogate_perms(config.seed, s, reps, config.strict_permutation))
    per_win = np.array([(u, -1) for u in us] + [(u, i) for u in grid for i in range(s)],
                       dtype=np.int32).reshape(-1, 2)
    starts = np.array([lo for lo, _ in windows], dtype=np.int32)
    items = np.empty((len(starts) * len(per_win), 3), dtype=np.int32)  # window-major
    items[:, :2] = np.tile(per_win, (len(starts), 1))
    items[:, 2] = np.repeat(starts, len(per_win))
    te_all = pipe.run(items).reshape(len(windows), len(per_win))
    return _assemble_results(source, target, config, windows, us, grid,
                             te_all[:, :len(us)], te_all[:, len(us):].reshape(len(windows), len(grid), s))


def _at_window(config, win):
    import dataclasses
    return dataclasses.replace(config, window=tuple(win))


def _assemble_results(source, target, config, windows, us, grid, te_orig, te_surr) -> list:
    """The host statistics of analyze_pair (inference.py:153-193) for many
    windows: te_orig [windows, len(us)], te_surr [windows, len(grid), S]."""
    s = config.n_surrogates
    te_orig = np.asarray(te_orig, dtype=np.float64)
    # surrogate statistic: running np.maximum over the grid rows from -inf
    surrogates = np.full((len(windows), s), -np.inf)
    for g in range(len(grid)):
        np.maximum(surrogates, te_surr[:, g, :], out=surrogates)
    medians = np.median(surrogates, axis=1)
    results = []
    for wi, win in enumerate(windows):
        curve = [(u, float(t)) for u, t in zip(us, te_orig[wi])]
        u_best, te_best = max(curve, key=lambda ut: (ut[1], -ut[0]))
        stat_orig = max(t for u, t in curve if u in grid)
        p = permutation_pvalue(stat_orig, surrogates[wi], config.conservative_pvalue)
        sig = p < config.alpha
        results.append(TEResult(source=source.channel_name, target=target.channel_name,
                                window=win, u_selected=u_best, te_value=te_best,
                                surrogate_values=surrogates[wi].copy(), p_value=p, significant=sig,
                                significant_corrected=sig,
                                te_minus_median_surrogate=te_best - float(medians[wi]),
                                te_curve=curve))
    return results


def _width(config) -> int:
    return config.window[1] - config.window[0] + 1


def _assemble_result(source, target, config, us, grid, te_orig, te_surr) -> TEResult:
    """Host statistics of analyze_pair (inference.py:153-193) for one window."""
    te_surr = np.asarray(te_surr, dtype=np.float64).reshape(1, len(grid), config.n_surrogates)
    return _assemble_results(source, target, config, [config.window], us, grid,
                             np.asarray(te_orig, dtype=np.float64)[None], te_surr)[0]


def scan_delays(source, target, spec_x, spec_y, config) -> TEResult:
    """Alias of analyze_pair (which always scans)."""
    return analyze_pair(source, target, spec_x, spec_y, config)


def analyze_pairs(series_by_name: dict, pairs, specs_by_name: dict, config: AnalysisConfig):
    """analyze_pair per directed pair + the configured family-wise correction."""
    results = [analyze_pair(series_by_name[a], series_by_name[b], specs_by_name[a],
                            specs_by_name[b], config) for a, b in pairs]
    decisions = correct_multiple([r.p_value for r in results], config.alpha, config.correction)
    for r, d in zip(results, decisions):
        r.significant_corrected = bool(d and r.significant)
    return results
