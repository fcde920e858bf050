"""KSG transfer entropy from pooled point sets, computed on the GPU.

Drop-in for /root/reference/pkg/src/ente/ksg.py: digamma 20-26,
TermCounts 29-36, te_from_counts 39-49, estimate_te_batch 66-90,
estimate_te 93-96.  estimate_te_batch runs jitter (ente_jitter), the fused
kNN + marginal-count search (ente_search) and the digamma reduction
(ente_te_reduce) on the device; the values equal the reference's bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
from scipy import special

from . import _native as nat
from .engine import MAX_K, search_device, search_te_shared_device
from .exceptions import DegenerateData, DomainError, KTooLarge, ShapeMismatch

EULER_GAMMA = 0.5772156649015329


def digamma(x):
    """psi(x) for x > 0, scalar or array (host helper of the API, as in the reference)."""
    x = np.asarray(x, dtype=np.float64)
    if (x <= 0).any():
        raise DomainError("digamma requires x > 0")
    out = special.digamma(x)
    return float(out) if out.ndim == 0 else out


@dataclass(frozen=True)
class TermCounts:
    """Per-point neighbour counts in the three marginal spaces."""

    k: int
    n_ypast: np.ndarray
    n_y_ypast: np.ndarray
    n_ypast_xpast: np.ndarray


class _PsiTable:
    """Device table psi(m + 1), m = 0..size-1 (scipy values), grown on demand."""

    def __init__(self):
        self.table = None

    def get(self, size: int) -> torch.Tensor:
        dev = nat.device()
        if self.table is None or self.table.numel() < size or self.table.device != dev:
            n = 1 << max(10, int(size - 1).bit_length())
            host = special.digamma(np.arange(1, n + 1, dtype=np.float64))
            self.table = torch.from_numpy(host).to(dev)
        return self.table


_PSI = _PsiTable()


def te_reduce_device(counts: torch.Tensor, rows0, ns, k: int, tag: str = "", table=None) -> torch.Tensor:
    """ente_te_reduce over a [3, rows] int32 device count matrix; returns [n_chunks] f64.
    table: nat.chunk_table(rows0, ns) when the caller has it."""
    L = nat.lib()
    rows = counts.shape[1]
    psi = _PSI.get(int(np.max(ns)) + 2)
    out = torch.empty(len(ns), dtype=torch.float64, device=counts.device)
    if table is None:
        table = nat.chunk_table(rows0, ns)
    ws = nat.workspace(L.ente_te_reduce_workspace_size(table, len(ns)), tag)
    nat.check(L.ente_te_reduce(nat.ptr(counts), rows, table, len(ns), nat.ptr(psi), psi.numel(),
                               float(special.digamma(k)), nat.ptr(out), nat.ptr(ws), ws.numel(),
                               nat.stream_handle()), "ente_te_reduce")
    return out


def te_from_counts(counts: TermCounts) -> float:
    """psi(k) + mean of the sorted per-point terms (device reduction)."""
    a = np.asarray(counts.n_ypast, dtype=np.int64)
    b = np.asarray(counts.n_y_ypast, dtype=np.int64)
    c = np.asarray(counts.n_ypast_xpast, dtype=np.int64)
    if a.size == 0:
        return float("nan")
    if min(a.min(), b.min(), c.min()) < 0:
        raise DomainError("digamma requires x > 0 (negative count)")
    mat = torch.from_numpy(np.stack([a, b, c]).astype(np.int32)).to(nat.device())
    return float(te_reduce_device(mat, [0], [a.size], counts.k).cpu()[0])


def jitter_device(pts64: torch.Tensor, rows0, ns, amplitude: float, seeds,
                  tag: str = "", table=None) -> torch.Tensor:
    """ente_jitter in place on a device [rows, dim] matrix; returns the status tensor."""
    L = nat.lib()
    dim = pts64.shape[1]
    if table is None:
        table = nat.chunk_table(rows0, ns)
    states = None
    if amplitude > 0:
        if isinstance(seeds, np.ndarray) and seeds.dtype == np.uint64:
            st = np.ascontiguousarray(seeds.reshape(len(ns), 4))  # precomputed (state, inc)
        else:
            st = nat.pcg_states(seeds, [n * dim for n in ns])
        states = st.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_uint64))
    status = torch.zeros(len(ns), dtype=torch.int32, device=pts64.device)
    ws = nat.workspace(L.ente_jitter_workspace_size(len(ns), dim), tag)
    nat.check(L.ente_jitter(nat.ptr(pts64), dim, table, len(ns), states, float(amplitude),
                            nat.ptr(status), nat.ptr(ws), ws.numel(), nat.stream_handle()),
              "ente_jitter")
    return status


def te_masks(d_y: int, d_x: int):
    """Column masks of (y-past, y + y-past, y-past + x-past) -- embedding.py:50-60."""
    yp = sum(1 << c for c in range(1, 1 + d_y))
    yyp = sum(1 << c for c in range(0, 1 + d_y))
    ypxp = sum(1 << c for c in range(1, 1 + d_y + d_x))
    return [yp, yyp, ypxp]


def te_chunks_device(pts64: torch.Tensor, rows0, ns, d_y: int, d_x: int, k: int,
                     amplitude: float, seeds, sync: bool = True, tag: str = "", shared=None):
    """jitter -> checks -> search -> reduce for TE-layout chunks already on the device.

    sync=True: returns (te [n_chunks] f64 device tensor or None, status numpy
    array); the status read-back after the jitter checks is the only host
    synchronisation, and chunks are not searched when any check failed.
    sync=False: everything is queued on the current stream and (te, status)
    come back as device tensors; the caller reads status before using te
    (a failed chunk's TE is meaningless).  `tag` selects per-stream scratch.
    """
    table = nat.chunk_table(rows0, ns)  # one host chunk table for every stage
    status = jitter_device(pts64, rows0, ns, amplitude, seeds, tag, table)
    if sync:
        st = status.cpu().numpy()
        if (st != 0).any():
            return None, st
    if shared is not None:  # every chunk pools the same target rows: y marginals once per point
        _, counts, _ = search_te_shared_device(pts64, rows0, ns, d_y, k, shared, tag=tag, table=table)
    else:
        _, counts, _ = search_device(pts64, rows0, ns, te_masks(d_y, d_x), k, reuse=True, tag=tag,
                                     table=table)
    te = te_reduce_device(counts, rows0, ns, k, tag, table)
    return (te, st) if sync else (te, status)


def _raise_status(code: int):
    if code == nat.CHUNK_DEGENERATE:
        raise DegenerateData("all pooled points are identical")
    if code == nat.CHUNK_NONFINITE:
        raise ShapeMismatch("chunk contains non-finite values")
    raise RuntimeError(f"unexpected chunk status {code}")


def estimate_te_batch(bundles, k: int, jitter_amplitude: float = 1e-8, seeds=None):
    """TE (nats) of many bundles through one device pipeline, in input order.

    Errors follow the reference order: the first bundle that fails raises,
    KTooLarge (n_rows <= k) or DegenerateData / ShapeMismatch after jitter.
    """
    bundles = list(bundles)
    if seeds is None:
        seeds = range(len(bundles))
    pairs = list(zip(bundles, seeds, strict=True))
    first_small = next((i for i, (b, _) in enumerate(pairs) if b.n_rows <= k), None)
    todo = pairs if first_small is None else pairs[:first_small]
    if k > MAX_K:
        raise NotImplementedError(f"k={k} exceeds {MAX_K}")
    values = [None] * len(todo)
    groups = {}
    for i, (b, s) in enumerate(todo):
        groups.setdefault((int(b.d_y), int(b.d_x)), []).append(i)
    first_bad = None
    for (d_y, d_x), idxs in groups.items():
        joints = [np.ascontiguousarray(todo[i][0].joint, dtype=np.float64) for i in idxs]
        ns = [j.shape[0] for j in joints]
        rows0 = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)
        host = torch.from_numpy(np.concatenate(joints, axis=0))
        dev = host.pin_memory().to(nat.device(), non_blocking=True)
        te, st = te_chunks_device(dev, rows0, ns, d_y, d_x, k, jitter_amplitude,
                                  [todo[i][1] for i in idxs])
        if te is None:
            for i, code in zip(idxs, st):
                if code != 0 and (first_bad is None or i < first_bad[0]):
                    first_bad = (i, int(code))
            continue
        for i, v in zip(idxs, te.cpu().numpy()):
            values[i] = float(v)
    if first_bad is not None:
        _raise_status(first_bad[1])
    if first_small is not None:
        n = pairs[first_small][0].n_rows
        raise KTooLarge(f"need more than k={k} pooled points, got {n}")
    return values


def estimate_te(bundle, k: int, jitter_amplitude: float = 1e-8, seed=0) -> float:
    """TE estimate in nats for one pooled point-set bundle."""
    return estimate_te_batch([bundle], k, jitter_amplitude, [seed])[0]
