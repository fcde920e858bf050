"""Native (C++) derivation of the reference's random streams.

The reference seeds every jitter stream with
``default_rng(SeedSequence((seed, u, 0 | idx + 1)))`` (inference.py:148,
171-172; ksg.py:55) and every surrogate with
``default_rng(SeedSequence((seed, idx))).permutation(R)``, redrawn until no
repetition maps to itself (inference.py:41-49, 101-102, 161-164).  numpy
pays tens of microseconds of Python per stream; ``ente_seed_states`` and
``ente_draw_permutations`` (csrc/seeds.cu) restate SeedSequence, PCG64 and
Generator.permutation in C++ and produce the same bits for a whole batch
in microseconds (pinned against numpy by tests/test_seeds.py).

Seeds that are not plain SeedSequence entropy (a Generator, a BitGenerator,
a SeedSequence with a non-default pool) keep numpy's own construction:
that is the reference API's host-side seed handling, not a compute path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat

_MASK32 = (1 << 32) - 1
_POOL = 4


def _int_words(n) -> list:
    n = int(n)
    if n < 0:
        raise ValueError("expected non-negative integer")
    if n == 0:
        return [0]
    out = []
    while n > 0:
        out.append(n & _MASK32)
        n >>= 32
    return out


def _coerce(x) -> list | None:
    """numpy's _coerce_to_uint32_array for ints and (nested) int sequences."""
    if isinstance(x, (bool, np.bool_)):
        return _int_words(int(x))
    if isinstance(x, (int, np.integer)):
        return _int_words(x)
    if isinstance(x, np.ndarray) and x.dtype == np.uint32:
        return [int(v) for v in x.ravel()]
    if isinstance(x, (tuple, list, np.ndarray)):
        out = []
        for v in x:
            w = _coerce(v)
            if w is None:
                return None
            out.extend(w)
        return out
    return None


def entropy_words(seed) -> np.ndarray | None:
    """SeedSequence entropy words of a seed default_rng would accept, or None
    when the seed is not plain SeedSequence entropy (Generator, BitGenerator,
    custom pool size)."""
    if seed is None:
        return None
    if isinstance(seed, np.random.SeedSequence):
        if seed.pool_size != _POOL or seed.entropy is None:
            return None
        run = _coerce(seed.entropy)
        spawn = _coerce(seed.spawn_key) if len(seed.spawn_key) else []
        if run is None or spawn is None:
            return None
        if spawn and len(run) < _POOL:
            run = run + [0] * (_POOL - len(run))
        return np.asarray(run + spawn, dtype=np.uint32)
    if isinstance(seed, (np.random.Generator, np.random.BitGenerator, str, float)):
        return None
    w = _coerce(seed)
    return None if w is None else np.asarray(w, dtype=np.uint32)


def _flat(word_lists):
    sizes = np.fromiter((len(w) for w in word_lists), dtype=np.int64, count=len(word_lists))
    offsets = np.zeros(len(word_lists) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    words = np.ascontiguousarray(np.concatenate(word_lists).astype(np.uint32)) if len(word_lists) \
        else np.zeros(1, dtype=np.uint32)
    return words, offsets


def _tuple_words(master_seed, *columns):
    """Entropy words of SeedSequence((master_seed, c0[i], c1[i], ...)) for every i,
    vectorised when every column value fits one 32-bit word."""
    prefix = _coerce(master_seed)
    if prefix is None:
        raise TypeError(f"seed must be an int or a sequence of ints, got {master_seed!r}")
    cols = [np.asarray(c, dtype=np.int64).reshape(-1) for c in columns]
    n = len(cols[0]) if cols else 0
    if any((c < 0).any() for c in cols):
        raise ValueError("expected non-negative integer")
    if all(int(c.max(initial=0)) <= _MASK32 for c in cols):
        k = len(prefix) + len(cols)
        words = np.empty((n, k), dtype=np.uint32)
        words[:, :len(prefix)] = np.asarray(prefix, dtype=np.uint32)
        for j, c in enumerate(cols):
            words[:, len(prefix) + j] = c.astype(np.uint32)
        return np.ascontiguousarray(words.reshape(-1)), np.arange(n + 1, dtype=np.int64) * k
    lists = [np.asarray(prefix + sum((_int_words(c[i]) for c in cols), []), dtype=np.uint32)
             for i in range(n)]
    return _flat(lists)


def _states_from_words(words, offsets) -> np.ndarray:
    n = len(offsets) - 1
    out = np.empty((n, 4), dtype=np.uint64)
    if n == 0:
        return out
    nat.check(nat.lib().ente_seed_states(
        words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
        offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n,
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))), "ente_seed_states")
    return out


def jitter_states(master_seed, us, stream_ids, out=None) -> np.ndarray:
    """PCG64 (state_hi, state_lo, inc_hi, inc_lo) of
    default_rng(SeedSequence((master_seed, u, stream_id))) per item, [n, 4] uint64
    (stream_id = 0 for the original data, idx + 1 for surrogate idx).
    out: a C-contiguous [n, 4] uint64 array to fill (e.g. pinned memory)."""
    prefix = _coerce(master_seed)
    if prefix is None:
        raise TypeError(f"seed must be an int or a sequence of ints, got {master_seed!r}")
    cols = np.stack([np.asarray(us, dtype=np.int64).reshape(-1),
                     np.asarray(stream_ids, dtype=np.int64).reshape(-1)])
    n = cols.shape[1]
    if out is None:
        out = np.empty((n, 4), dtype=np.uint64)
    elif out.shape != (n, 4) or out.dtype != np.uint64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous [n, 4] uint64 array")
    if n == 0:
        return out
    if (cols < 0).any():
        raise ValueError("expected non-negative integer")
    if int(cols.max()) > _MASK32 or len(prefix) + 2 > 16:  # multi-word values: per-item word lists
        out[...] = _states_from_words(*_tuple_words(master_seed, us, stream_ids))
        return out
    pre = np.asarray(prefix, dtype=np.uint32)
    nat.check(nat.lib().ente_seed_states_cols(
        pre.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), len(pre),
        cols.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 2, n,
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))), "ente_seed_states_cols")
    return out


def pcg_states(seeds) -> np.ndarray:
    """PCG64 states of default_rng(seed) for SeedSequence-entropy seeds, [n, 4] uint64."""
    lists = []
    for s in seeds:
        w = entropy_words(s)
        if w is None:
            raise TypeError(f"not plain SeedSequence entropy: {s!r}")
        lists.append(w)
    return _states_from_words(*_flat(lists))


def surrogate_permutations(master_seed, count: int, reps: int, strict: bool) -> np.ndarray:
    """draw_permutation(reps, SeedSequence((master_seed, i)), strict) for i < count,
    as an int32 [count, reps] array (inference.py:41-49, 101-102, 161-164)."""
    return surrogate_permutations_at(master_seed, np.arange(count), reps, strict)


def surrogate_permutations_at(master_seed, indices, reps: int, strict: bool) -> np.ndarray:
    """The same for the surrogate indices given, [len(indices), reps] int32."""
    indices = np.asarray(indices, dtype=np.int64).reshape(-1)
    count = len(indices)
    out = np.empty((count, reps), dtype=np.int32)
    if count == 0:
        return out
    words, offsets = _tuple_words(master_seed, indices)
    nat.check(nat.lib().ente_draw_permutations(
        words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
        offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), count, int(reps), int(bool(strict)),
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "ente_draw_permutations")
    return out
