"""ctypes binding of libente_b200.so (declared in include/ente_b200.h).

There is no CPU fallback: importing the compute functions on a machine
without the built library or without a CUDA device raises.  PyTorch is only
the device-memory / stream plumbing: tensors are allocated with torch and
their raw pointers handed to the C ABI together with the current stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# ENTE_LIB overrides the library path (development A/B builds only)
LIB_PATH = os.environ.get("ENTE_LIB") or os.path.join(PKG_DIR, "libente_b200.so")

CHUNK_OK, CHUNK_K_TOO_LARGE, CHUNK_NONFINITE, CHUNK_DEGENERATE = 0, 1, 2, 3


class NativeError(RuntimeError):
    """A C-ABI call returned an error code."""


class ChunkDesc(ctypes.Structure):
    _fields_ = [("row0", ctypes.c_int64), ("n", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_lib = None
_lock = threading.Lock()


def _declare(L):
    vp, sz, i32, i64, dbl = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    cp = ctypes.POINTER(ChunkDesc)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    i32p = ctypes.POINTER(ctypes.c_int32)
    sig = {
        "ente_version": ([], ctypes.c_char_p),
        "ente_last_error": ([], ctypes.c_char_p),
        "ente_search_workspace_size": ([cp, i32, i32, i32, i32], sz),
        "ente_search": ([vp, i64, i32, cp, i32, u32p, i32, i32, vp, vp, vp, vp, sz, vp], i32),
        "ente_ragwitz_errors": ([vp, i32, i32, i32, i32, vp, vp, i32, i32, vp, vp], i32),
        "ente_knn_indices": ([vp, i64, i32, cp, i32, i32, vp, vp, vp, vp, sz, vp], i32),
        "ente_search_split": ([vp, i64, i32, cp, i32, u32p, i32, i32, i32, i32, vp, vp, vp, vp, sz,
                               vp], i32),
        "ente_radius_counts_workspace_size": ([cp, i32, i32], sz),
        "ente_search_path": ([i32, u32p, i32, i32], i32),
        "ente_search_te_shared_workspace_size": ([cp, i32, i32, i32, i32], sz),
        "ente_search_te_shared": ([vp, i64, i32, cp, i32, i32, i32, vp, i32, i32, i32p, vp, vp, dbl,
                                   vp, vp, vp, vp, sz, vp], i32),
        "ente_radius_counts": ([vp, i64, i32, cp, i32, u32p, i32, vp, vp, vp, vp, sz, vp], i32),
        "ente_jitter_workspace_size": ([i32, i32], sz),
        "ente_jitter": ([vp, i32, cp, i32, u64p, dbl, vp, vp, sz, vp], i32),
        "ente_pack_te": ([vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32p, i32, vp, vp, vp], i32),
        "ente_pack_te_items": ([vp, vp, i32, i32, i32, i32, i32, i32, i32, i32p, i32, vp, vp, vp],
                               i32),
        "ente_te_reduce_workspace_size": ([cp, i32], sz),
        "ente_te_reduce": ([vp, i64, cp, i32, vp, i64, dbl, vp, vp, sz, vp], i32),
        "ente_launch_count": ([], i64),
        "ente_profile_enable": ([i32], None),
        "ente_profile_reset": ([], None),
        "ente_profile_read": ([ctypes.c_char_p, sz, ctypes.POINTER(i64), ctypes.POINTER(dbl), i32],
                              i32),
        "ente_microbench_pce": ([i32, i32, ctypes.POINTER(dbl), vp], i32),
        "ente_search_work": ([ctypes.POINTER(ctypes.c_ulonglong)] * 2, None),
        "ente_seed_states": ([u32p, ctypes.POINTER(i64), i64, u64p], i32),
        "ente_seed_states_cols": ([u32p, i32, ctypes.POINTER(i64), i32, i64, u64p], i32),
        "ente_host_gather": ([ctypes.POINTER(vp), ctypes.POINTER(i64), i64, vp], i32),
        "ente_draw_permutations": ([u32p, ctypes.POINTER(i64), i64, i32, i32, i32p], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """The loaded library (loaded once; raises if it was never built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with `python -m paper_1401_4068_b200.build` "
                        "(there is no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1401_4068_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed ({rc}): {lib().ente_last_error().decode()}")


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


_CHUNK_DTYPE = np.dtype([("row0", "<i8"), ("n", "<i4"), ("reserved", "<i4")])


def chunk_table(rows0, ns):
    """ente_chunk[] for the C ABI (vectorised; the pointer keeps the array alive)."""
    arr = np.zeros(len(ns), dtype=_CHUNK_DTYPE)
    arr["row0"] = np.asarray(rows0, dtype=np.int64)
    arr["n"] = np.asarray(ns, dtype=np.int32)
    return arr.ctypes.data_as(ctypes.POINTER(ChunkDesc))


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class _Workspace(threading.local):
    bufs = None


_ws = _Workspace()


def workspace(nbytes: int, tag: str = "") -> torch.Tensor:
    """A per-thread (and per-tag: one per concurrent stream) device scratch buffer of
    at least nbytes, grown on demand."""
    if _ws.bufs is None:
        _ws.bufs = {}
    buf = _ws.bufs.get(tag)
    if buf is None or buf.numel() < nbytes or buf.device != device():
        _ws.bufs[tag] = None
        del buf
        buf = torch.empty(max(int(nbytes), 1 << 20), dtype=torch.uint8, device=device())
        _ws.bufs[tag] = buf
    return buf


class _Scratch(threading.local):
    bufs = None


_scratch = _Scratch()


def scratch(name: str, shape, dtype: torch.dtype) -> torch.Tensor:
    """A named, grow-only, per-thread device buffer viewed as `shape` of `dtype`.

    The pipeline's big per-wave arrays (packed joints, eps, counts) live here
    so that repeated waves reuse the same resident HBM instead of going
    through the caching allocator (whose splits of multi-GB blocks ended in
    fresh cudaMalloc + first-touch costs of hundreds of ms per call).  The
    contents are overwritten by the next call that uses the same name, so
    callers copy results out before returning them.
    """
    if _scratch.bufs is None:
        _scratch.bufs = {}
    numel = 1
    for s in shape:
        numel *= int(s)
    nbytes = max(1, numel * torch.empty((), dtype=dtype).element_size())
    dev = device()
    buf = _scratch.bufs.get(name)
    if buf is None or buf.numel() < nbytes or buf.device != dev:
        _scratch.bufs[name] = None
        del buf
        buf = torch.empty(nbytes + (nbytes >> 4), dtype=torch.uint8, device=dev)
        _scratch.bufs[name] = buf
    return buf[:nbytes].view(dtype).view(tuple(int(s) for s in shape))


def masks_array(masks):
    arr = (ctypes.c_uint32 * max(1, len(masks)))()
    for i, m in enumerate(masks):
        arr[i] = int(m)
    return arr


def pcg_states(seeds, draws_per_seed):
    """numpy PCG64 (state, inc) per seed as the uint64 quadruples of ente_jitter.

    Mirrors np.random.default_rng(seed) as used by the reference jitter
    (ksg.py:55): a Generator passed as seed is used as is and advanced by the
    number of draws the reference would consume.
    """
    out = np.empty((len(seeds), 4), dtype=np.uint64)
    mask = (1 << 64) - 1
    for i, (seed, draws) in enumerate(zip(seeds, draws_per_seed)):
        gen = np.random.default_rng(seed)
        st = gen.bit_generator.state
        if st.get("bit_generator") != "PCG64":
            raise TypeError(f"jitter seeds must produce PCG64 generators, got {st.get('bit_generator')}")
        s, inc = st["state"]["state"], st["state"]["inc"]
        out[i] = (s >> 64, s & mask, inc >> 64, inc & mask)
        if isinstance(seed, np.random.Generator):
            gen.bit_generator.advance(int(draws))
    return out


def launch_count() -> int:
    return int(lib().ente_launch_count())


class KernelProfile:
    """Per-kernel on-stream timing of the library's launches (CUDA events)."""

    def __enter__(self):
        lib().ente_profile_reset()
        lib().ente_profile_enable(1)
        return self

    def __exit__(self, *exc):
        lib().ente_profile_enable(0)
        return False

    @staticmethod
    def read() -> dict:
        L = lib()
        cap = 64
        names = ctypes.create_string_buffer(4096)
        launches = (ctypes.c_int64 * cap)()
        ms = (ctypes.c_double * cap)()
        n = L.ente_profile_read(names, len(names), launches, ms, cap)
        keys = [k.decode() for k in names.raw.split(b"\0")[:n]]
        return {k: {"launches": int(launches[i]), "ms": float(ms[i])} for i, k in enumerate(keys)}


def microbench_pce(iters: int = 200) -> float:
    out = ctypes.c_double()
    check(lib().ente_microbench_pce(int(iters), 0, ctypes.byref(out), stream_handle()),
          "ente_microbench_pce")
    return out.value


def search_work() -> tuple[int, int]:
    """(knn, count) reference-candidate pairs evaluated since the last call."""
    a, b = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    lib().ente_search_work(ctypes.byref(a), ctypes.byref(b))
    return int(a.value), int(b.value)
