"""Batched exact max-norm kNN distances and strict radius counts on the GPU.

Drop-in for the reference neighbour engine
(/root/reference/pkg/src/ente/engine.py): same names, argument meaning,
outputs (float64 kth_distance, int64 counts, input order) and per-chunk
error slots.  All arithmetic runs in the sm_100a kernels of
libente_b200.so (ente_search / ente_radius_counts); results are
bit-identical to the reference's fp64 sweep.

  Chunk              engine.py:46-59     NeighborCounts   engine.py:62-67
  knn_kth_distances  engine.py:170-176   radius_counts    engine.py:179-188
  batch_search       engine.py:203-216   set_workers / max_workers 31-43
"""

from __future__ import annotations

import ctypes
import gc
import os
import threading
import warnings
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as nat
from .exceptions import KTooLarge, ShapeMismatch

MAX_DIM = 32   # column bitmasks are uint32 in the C ABI
MAX_K = 64     # exact warp top-k merge keeps <= 64 slots per lane
MAX_MARG = 8
MAX_WAVE_ROWS = 1 << 27  # points per device wave of batch_search

_workers = [os.cpu_count() or 1]


def max_workers() -> int:
    """Host threads available for host-side preparation (seeding, permutations)."""
    return os.cpu_count() or 1


def set_workers(n: int) -> int:
    """Set the host worker count (never changes results); returns the count in effect."""
    _workers[0] = max(1, min(int(n), max_workers()))
    return _workers[0]


@dataclass(frozen=True)
class Chunk:
    """One search problem: an [n >= 2, dim >= 1] finite point matrix (fp64 copy)."""

    points: np.ndarray
    chunk_id: int = 0

    def __post_init__(self):
        pts = np.ascontiguousarray(np.asarray(self.points, dtype=np.float64))
        if pts.ndim != 2 or pts.shape[0] < 2 or pts.shape[1] < 1:
            raise ShapeMismatch(f"chunk needs an [n>=2 x dim>=1] matrix, got {pts.shape}")
        if not np.isfinite(pts).all():
            raise ShapeMismatch("chunk contains non-finite values")
        object.__setattr__(self, "points", pts)


@dataclass(frozen=True)
class NeighborCounts:
    """kth_distance (float64 [n]) and one int64 [n] count array per marginal."""

    kth_distance: np.ndarray
    radius_counts: tuple


def column_mask(cols, dim: int) -> int:
    cols = np.asarray(cols, dtype=np.intp).ravel()
    if cols.size < 1 or cols.min() < 0 or cols.max() >= dim:
        raise ShapeMismatch(f"marginal columns {cols} out of range")
    mask = 0
    for c in cols.tolist():
        mask |= 1 << c
    return mask


class SlowPathWarning(RuntimeWarning):
    """A search layout runs the fp64 O(n^2) scan instead of the pruned fp32 sweeps."""


_PATHS: dict = {}


def search_path(dim: int, masks, k: int) -> int:
    """ente_search_path: 1 TE-layout sweeps, 2 kNN sweep + generic marginal
    counts, 0 the fp64 scan (warned once per layout: it is O(n^2) unpruned)."""
    key = (dim, tuple(masks), k)
    path = _PATHS.get(key)
    if path is None:
        path = int(nat.lib().ente_search_path(int(dim), nat.masks_array(masks), len(masks),
                                              int(k)))
        _PATHS[key] = path
        if path == 0:
            warnings.warn(f"dim={dim}, marginal masks {[hex(m) for m in masks]}, k={k}: no compiled "
                          "sweep layout; this search runs the fp64 O(n^2) scan", SlowPathWarning,
                          stacklevel=3)
    return path


# ---------------------------------------------------------------------------
# device-level entry points (tensors in, tensors out; used by ksg / bench)
# ---------------------------------------------------------------------------
def search_device(pts64: torch.Tensor, rows0, ns, masks, k: int, reuse: bool = False,
                  tag: str = "", split=None, split_fill=(0.0, 0), table=None):
    """ente_search on a device-resident [rows, dim] fp64 matrix.

    Returns (eps [rows] f64, counts [n_marg, rows] int32, status [n_chunks] int32),
    all on the device, stream-ordered on the current stream.  With reuse the
    outputs live in the named scratch pool (valid until the next reuse call).
    """
    if pts64.dtype != torch.float64 or not pts64.is_cuda or not pts64.is_contiguous():
        raise TypeError("pts64 must be a contiguous CUDA float64 tensor")
    rows, dim = pts64.shape
    L = nat.lib()
    if table is None:  # (callers running several stages on one batch pass theirs)
        table = nat.chunk_table(rows0, ns)
    marr = nat.masks_array(masks)
    if reuse:
        eps = nat.scratch("search.eps" + tag, (rows,), torch.float64)
        counts = nat.scratch("search.counts" + tag, (max(1, len(masks)), rows), torch.int32)
        status = nat.scratch("search.status" + tag, (max(1, len(ns)),), torch.int32)
    else:
        eps = torch.empty(rows, dtype=torch.float64, device=pts64.device)
        counts = torch.empty((max(1, len(masks)), rows), dtype=torch.int32, device=pts64.device)
        status = torch.empty(max(1, len(ns)), dtype=torch.int32, device=pts64.device)
    need = L.ente_search_workspace_size(table, len(ns), dim, len(masks), int(k))
    ws = nat.workspace(need, tag)
    if split is None:
        nat.check(L.ente_search(nat.ptr(pts64), rows, dim, table, len(ns), marr, len(masks),
                                int(k), nat.ptr(eps), nat.ptr(counts), nat.ptr(status),
                                nat.ptr(ws), ws.numel(), nat.stream_handle()), "ente_search")
    else:  # (index, count): this part's references only, other rows = split_fill
        eps.fill_(split_fill[0])
        counts.fill_(split_fill[1])
        nat.check(L.ente_search_split(nat.ptr(pts64), rows, dim, table, len(ns), marr, len(masks),
                                      int(k), int(split[0]), int(split[1]), nat.ptr(eps),
                                      nat.ptr(counts), nat.ptr(status), nat.ptr(ws), ws.numel(),
                                      nat.stream_handle()), "ente_search_split")
    return eps, counts[:len(masks)], status[:len(ns)]


@dataclass(frozen=True)
class SharedY:
    """The common target point set of a TE batch (ente_search_te_shared):
    y0 [reps * w, 1 + d_y] unjittered y columns on the device, every chunk's
    surrogate index (-1 = original), the permutation tables (and inverses)
    on the device, and the jitter margin."""

    y0: torch.Tensor
    reps: int
    w: int
    chunk_perm: np.ndarray
    perms: torch.Tensor
    inv_perms: torch.Tensor
    margin: float


def search_te_shared_device(pts64: torch.Tensor, rows0, ns, d_y: int, k: int, shared: SharedY,
                            tag: str = "", table=None):
    """ente_search_te_shared on device-resident TE chunks: (eps, counts [3, rows], status)."""
    rows, dim = pts64.shape
    L = nat.lib()
    if table is None:
        table = nat.chunk_table(rows0, ns)
    eps = nat.scratch("search.eps" + tag, (rows,), torch.float64)
    counts = nat.scratch("search.counts" + tag, (3, rows), torch.int32)
    status = nat.scratch("search.status" + tag, (max(1, len(ns)),), torch.int32)
    need = L.ente_search_te_shared_workspace_size(table, len(ns), dim, int(d_y), int(k))
    ws = nat.workspace(need, tag)
    cp = np.ascontiguousarray(shared.chunk_perm, dtype=np.int32)
    nat.check(L.ente_search_te_shared(
        nat.ptr(pts64), rows, dim, table, len(ns), int(d_y), int(k), nat.ptr(shared.y0),
        int(shared.reps), int(shared.w), cp.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        nat.ptr(shared.perms), nat.ptr(shared.inv_perms), float(shared.margin), nat.ptr(eps),
        nat.ptr(counts), nat.ptr(status), nat.ptr(ws), ws.numel(), nat.stream_handle()),
        "ente_search_te_shared")
    return eps, counts, status[:len(ns)]


class _Pinned(threading.local):
    bufs = None


_pinned = _Pinned()


def _pinned_buffer(nbytes: int, slot: int = 0) -> torch.Tensor:
    """Grow-only pinned host staging buffer (page-locking per call costs more than the copy)."""
    if _pinned.bufs is None:
        _pinned.bufs = {}
    buf = _pinned.bufs.get(slot)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8).pin_memory()
        _pinned.bufs[slot] = buf
    return buf


try:  # chunk pointers through the buffer protocol in C (csrc/pyhost.cpp)
    from . import _pyhost
except ImportError:  # not built: the same values one Python attribute at a time
    _pyhost = None


def _scan(points_list):
    """(addresses, byte sizes, rows) of C-contiguous arrays as int64 numpy arrays."""
    if _pyhost is not None:
        a, b, r = _pyhost.scan(points_list)
        return (np.frombuffer(a, dtype=np.int64), np.frombuffer(b, dtype=np.int64),
                np.frombuffer(r, dtype=np.int64))
    n = len(points_list)
    return (np.fromiter((p.ctypes.data for p in points_list), dtype=np.int64, count=n),
            np.fromiter((p.nbytes for p in points_list), dtype=np.int64, count=n),
            np.fromiter((p.shape[0] for p in points_list), dtype=np.int64, count=n))


def _upload(points_list, slot: int = 0, tag: str = "", scan=None):
    """Concatenate the chunks straight into pinned memory (multi-threaded,
    ente_host_gather) and copy them to the device in one transfer on the
    current stream.  Staging slot `slot` must be free (its previous copy done).
    scan: _scan(points_list), when the caller has it."""
    addrs, sizes, ns = scan if scan is not None else _scan(points_list)
    rows = int(ns.sum())
    dim = points_list[0].shape[1]
    stage = _pinned_buffer(rows * dim * 8, slot)[:rows * dim * 8].view(torch.float64).view(rows, dim)
    addrs = np.ascontiguousarray(addrs)
    sizes = np.ascontiguousarray(sizes)
    nat.check(nat.lib().ente_host_gather(addrs.ctypes.data_as(ctypes.POINTER(ctypes.c_void_p)),
                                         sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                         len(addrs), stage.data_ptr()), "ente_host_gather")
    dev = nat.scratch("engine.points" + tag, (rows, dim), torch.float64)
    dev.copy_(stage, non_blocking=True)
    return dev


PIPE_BYTES = int(os.environ.get("ENTE_PIPE_MB", "96")) << 20  # host-input bytes per pipelined part of a batch_search wave
_PIPE_STREAMS: dict = {}


def _pipe_streams():
    key = torch.cuda.current_device()
    s = _PIPE_STREAMS.get(key)
    if s is None:
        s = _PIPE_STREAMS[key] = (torch.cuda.Stream(), torch.cuda.Stream())
    return s


def _parts(ns, dim):
    """Contiguous chunk ranges of about PIPE_BYTES of input each."""
    limit = max(1, PIPE_BYTES // (8 * dim))
    bounds, acc = [0], 0
    for i, n in enumerate(ns.tolist()):
        if acc and acc + n > limit:
            bounds.append(i)
            acc = 0
        acc += n
    bounds.append(len(ns))
    return list(zip(bounds[:-1], bounds[1:]))


def _new_counts(eps, cnts):
    o = object.__new__(NeighborCounts)  # frozen dataclass: fill the instance dict directly
    d = o.__dict__
    d["kth_distance"] = eps
    d["radius_counts"] = cnts
    return o


def _run_group(points_list, dim, masks, k, scan=None):
    """One wave: upload, search and read back, pipelined in parts of about
    PIPE_BYTES on two streams so the host gather and the PCIe copies of one
    part overlap the searches of the others."""
    search_path(dim, masks, k)
    n_chunks = len(points_list)
    addrs, sizes, ns = scan if scan is not None else _scan(points_list)
    rows0 = np.zeros(n_chunks, dtype=np.int64)
    np.cumsum(ns[:-1], out=rows0[1:])
    total = int(ns.sum())
    nm = len(masks)
    # results land in fresh pinned host tensors (torch's caching host allocator:
    # no page-locking or first-touch per call), counts widened to int64 on the
    # device, so the host does no conversion pass
    eps_p = torch.empty(total, dtype=torch.float64, pin_memory=True)
    # one 1-D tensor per marginal: each part's slice is contiguous, so its
    # copy stays a single async DMA (a strided pinned slice would be copied
    # through a pageable temporary, synchronously)
    cnt_p = [torch.empty(total, dtype=torch.int64, pin_memory=True) for _ in range(nm)]
    st_p = torch.empty(n_chunks, dtype=torch.int32, pin_memory=True)
    parts = _parts(ns, dim)
    main = torch.cuda.current_stream()
    streams = _pipe_streams() if len(parts) > 1 else (main,)
    staged = [None] * len(streams)  # event: the slot's previous H2D is done
    for j, (a, b) in enumerate(parts):
        slot = j % len(streams)
        st = streams[slot]
        if st is not main:
            st.wait_stream(main)
        if staged[slot] is not None:
            staged[slot].synchronize()
        r0, r1 = int(rows0[a]), int(rows0[b - 1] + ns[b - 1])
        tag = f".p{slot}" if len(parts) > 1 else ""
        with torch.cuda.stream(st):
            dev = _upload(points_list[a:b], slot, tag, (addrs[a:b], sizes[a:b], ns[a:b]))
            ev = torch.cuda.Event()
            ev.record(st)
            staged[slot] = ev
            eps, counts, status = search_device(dev, rows0[a:b] - r0, ns[a:b], masks, k, reuse=True,
                                                tag=tag)
            eps_p[r0:r1].copy_(eps, non_blocking=True)
            if nm:
                c64 = counts.to(torch.int64)
                for m in range(nm):
                    cnt_p[m][r0:r1].copy_(c64[m], non_blocking=True)
            st_p[a:b].copy_(status, non_blocking=True)
    for st in streams:
        st.synchronize()
    st_h, eps_h, cnt_h = st_p.numpy(), eps_p.numpy(), [c.numpy() for c in cnt_p]
    return _assemble(st_h, eps_h, cnt_h, rows0, ns, k)


def _assemble(st_h, eps_h, cnt_h, rows0, ns, k):
    """Per-chunk NeighborCounts views into one call's result arrays."""
    n_chunks, nm = len(ns), len(cnt_h)
    gc_on = gc.isenabled()
    gc.disable()  # tens of thousands of small containers: no collector passes meanwhile
    try:
        if n_chunks > 1 and (ns == ns[0]).all():  # uniform chunks: row views made in C
            n = int(ns[0])
            es = list(eps_h.reshape(n_chunks, n))
            cs = zip(*[list(c.reshape(n_chunks, n)) for c in cnt_h]) if nm else [()] * n_chunks
            out = [_new_counts(e, c) for e, c in zip(es, cs)]
        else:
            out = []
            for r0, n in zip(rows0.tolist(), ns.tolist()):
                end = r0 + n
                out.append(_new_counts(eps_h[r0:end], tuple([c[r0:end] for c in cnt_h])))
        bad = np.flatnonzero(st_h)
        for i in bad.tolist():
            code = st_h[i]
            if code == nat.CHUNK_NONFINITE:
                out[i] = ShapeMismatch("chunk contains non-finite values")
            elif code == nat.CHUNK_K_TOO_LARGE:
                out[i] = KTooLarge(f"k={k} not in [1, n-1] for n={int(ns[i])}")
    finally:
        if gc_on:
            gc.enable()
    return out


def batch_search(items: Sequence, k: int):
    """kNN + marginal radius counts for many chunks; one slot per chunk, in order.

    Each slot is a NeighborCounts or the exception raised for that chunk
    (KTooLarge before ShapeMismatch, as engine.py:191-200 checks them).
    Chunks sharing (dim, marginal layout) go to the GPU in one launch sequence.
    """
    results = [None] * len(items)
    fast = _uniform_batch(items, k)
    if fast is not None:  # one validated layout for every chunk: no per-item checks
        dim, masks, pts_list, scan = fast
        _run_waves(list(enumerate(pts_list)), dim, masks, k, results, scan)
        return results
    groups = {}
    mask_cache = {}  # (id(marginals), dim) -> (marginals, masks): items usually share one list
    for slot, (chunk, marginals) in enumerate(items):
        pts = chunk.points
        if not (isinstance(pts, np.ndarray) and pts.dtype == np.float64 and pts.flags.c_contiguous):
            pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64))
        n, dim = pts.shape
        if k < 1 or k > n - 1:
            results[slot] = KTooLarge(f"k={k} not in [1, n-1] for n={n}")
            continue
        hit = mask_cache.get((id(marginals), dim))
        if hit is not None and hit[0] is marginals:
            masks = hit[1]
        else:
            try:
                masks = tuple(column_mask(cols, dim) for cols in marginals)
            except ShapeMismatch as exc:
                results[slot] = exc
                continue
            mask_cache[(id(marginals), dim)] = (marginals, masks)
        if dim > MAX_DIM or k > MAX_K or len(masks) > MAX_MARG:
            results[slot] = NotImplementedError(
                f"dim={dim} (<= {MAX_DIM}), k={k} (<= {MAX_K}), marginals={len(masks)} "
                f"(<= {MAX_MARG}) exceed the compiled engine limits")
            continue
        groups.setdefault((dim, masks), []).append((slot, pts))
    for (dim, masks), members in groups.items():
        _run_waves(members, dim, masks, k, results)
    return results


def _uniform_batch(items, k):
    """(dim, masks, points) when every item is a Chunk of one width sharing one
    marginal list object with k in range -- the batch_search calls of the
    estimator and the bench -- so the per-item checks can be skipped."""
    if not items:
        return None
    first = items[0][1]
    if any(m is not first for _, m in items) or not all(type(c) is Chunk for c, _ in items):
        return None
    pts_list = [c.points for c, _ in items]  # Chunk validated these (fp64, 2-D, contiguous, finite)
    scan = _scan(pts_list)
    dim = int(pts_list[0].shape[1])
    if (scan[1] != scan[2] * (8 * dim)).any() or k < 1 or k > int(scan[2].min()) - 1:
        return None  # mixed widths, or k out of range for some chunk
    try:
        masks = tuple(column_mask(cols, dim) for cols in first)
    except ShapeMismatch:
        return None
    if dim > MAX_DIM or k > MAX_K or len(masks) > MAX_MARG:
        return None
    return dim, masks, pts_list, scan


def _run_waves(members, dim, masks, k, results, scan=None):
    """Device waves of at most MAX_WAVE_ROWS points (the search workspace is a
    few hundred bytes per point); members are (slot, points) pairs, scan their
    _scan() when the caller has it."""
    pts = [p for _, p in members]
    if scan is None:
        scan = _scan(pts)
    ns = scan[2]
    start = 0
    while start < len(members):
        stop, rows = start, 0
        while stop < len(members) and (stop == start or rows + int(ns[stop]) <= MAX_WAVE_ROWS):
            rows += int(ns[stop])
            stop += 1
        outs = _run_group(pts[start:stop], dim, list(masks), k,
                          tuple(a[start:stop] for a in scan))
        for (slot, _), res in zip(members[start:stop], outs):
            results[slot] = res
        start = stop


def knn_kth_distances(chunk: Chunk, k: int) -> np.ndarray:
    """Distance from each point to its k-th nearest neighbour (self excluded)."""
    n = chunk.points.shape[0]
    if k < 1 or k > n - 1:
        raise KTooLarge(f"k={k} not in [1, n-1] for n={n}")
    (res,) = batch_search([(chunk, [])], k)
    if isinstance(res, Exception):
        raise res
    return res.kth_distance


def knn_indices_device(pts64: torch.Tensor, rows0, ns, k: int):
    """(eps [rows] f64, idx [rows, k] int32, status) on the device: the k nearest
    neighbours of every point, ascending (fp64 distance, chunk-local index)."""
    rows, dim = pts64.shape
    eps, _, status = search_device(pts64, rows0, ns, [], k)
    L = nat.lib()
    table = nat.chunk_table(rows0, ns)
    idx = torch.empty((rows, k), dtype=torch.int32, device=pts64.device)
    ws = nat.workspace(L.ente_search_workspace_size(table, len(ns), dim, 0, int(k)))
    st2 = torch.empty_like(status)
    nat.check(L.ente_knn_indices(nat.ptr(pts64), rows, dim, table, len(ns), int(k), nat.ptr(eps),
                                 nat.ptr(idx), nat.ptr(st2), nat.ptr(ws), ws.numel(),
                                 nat.stream_handle()), "ente_knn_indices")
    return eps, idx, status


def knn_indices(chunk: Chunk, k: int) -> np.ndarray:
    """[n, k] int64 indices of each point's k nearest neighbours (self excluded).

    Order: ascending max-norm distance, ties by ascending index -- the
    canonical order the reference implies but never materialises (its
    engine keeps only the k-th distance, engine.py:70-123).  Row i's k-th
    entry is a neighbour at exactly knn_kth_distances(chunk, k)[i].
    """
    pts = chunk.points
    n, dim = pts.shape
    if k < 1 or k > n - 1:
        raise KTooLarge(f"k={k} not in [1, n-1] for n={n}")
    if dim > MAX_DIM or k > MAX_K:
        raise NotImplementedError(f"dim={dim} (<= {MAX_DIM}) / k={k} (<= {MAX_K}) above the engine limits")
    dev = _upload([pts])
    _, idx, status = knn_indices_device(dev, [0], [n], k)
    if int(status.cpu()[0]) == nat.CHUNK_NONFINITE:
        raise ShapeMismatch("chunk contains non-finite values")
    return idx.cpu().numpy().astype(np.int64)


def radius_counts(chunk: Chunk, radii) -> np.ndarray:
    """#{j != i : maxnorm(p_i, p_j) < radii[i]} over all columns of the chunk."""
    radii = np.ascontiguousarray(np.asarray(radii, dtype=np.float64))
    pts = chunk.points
    n, dim = pts.shape
    if radii.shape != (n,):
        raise ShapeMismatch(f"radii shape {radii.shape} does not match n={n}")
    if (radii < 0).any():
        raise ShapeMismatch("radii must be nonnegative")
    if dim > MAX_DIM:
        raise NotImplementedError(f"dim={dim} exceeds {MAX_DIM}")
    if dim > 17:
        warnings.warn(f"radius_counts over {dim} columns: no compiled sweep layout; this runs the "
                      "fp64 O(n^2) scan", SlowPathWarning, stacklevel=2)
    L = nat.lib()
    dev = _upload([pts])
    r = torch.from_numpy(radii).to(dev.device)
    counts = torch.empty((1, n), dtype=torch.int32, device=dev.device)
    status = torch.empty(1, dtype=torch.int32, device=dev.device)
    table = nat.chunk_table([0], [n])
    marr = nat.masks_array([(1 << dim) - 1])
    ws = nat.workspace(L.ente_radius_counts_workspace_size(table, 1, dim))
    nat.check(L.ente_radius_counts(nat.ptr(dev), n, dim, table, 1, marr, 1, nat.ptr(r),
                                   nat.ptr(counts), nat.ptr(status), nat.ptr(ws), ws.numel(),
                                   nat.stream_handle()), "ente_radius_counts")
    return counts[0].cpu().numpy().astype(np.int64)
