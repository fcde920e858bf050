"""The C-ABI library loads and exports every entry point include/ente_b200.h declares.

No compute calls: only host-side functions (sizes, argument validation,
version) are exercised, so this runs without a GPU.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1401_4068_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ente_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ente_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared_functions()
    for required in ("ente_search", "ente_radius_counts", "ente_jitter", "ente_pack_te",
                     "ente_te_reduce", "ente_last_error", "ente_version"):
        assert required in names


def test_library_exports_every_declared_symbol():
    L = nat.lib()
    for name in declared_functions():
        assert hasattr(L, name), f"{name} declared in ente_b200.h but not exported"


def test_version_and_sm100a():
    assert b"sm_100a" in nat.lib().ente_version()


def test_argument_validation_without_gpu():
    L = nat.lib()
    table = nat.chunk_table([0], [10])
    masks = nat.masks_array([1])
    # dim out of range -> ENTE_ERR_ARG before any CUDA call
    rc = L.ente_search(None, 10, 40, table, 1, masks, 1, 4, None, None, None, None, 0, None)
    assert rc == -1 and b"dim=40" in L.ente_last_error()
    rc = L.ente_search(None, 10, 3, table, 1, masks, 1, 0, None, None, None, None, 0, None)
    assert rc == -1 and b"k=0" in L.ente_last_error()
    bad_mask = nat.masks_array([1 << 5])
    rc = L.ente_search(None, 10, 3, table, 1, bad_mask, 1, 4, None, None, None, None, 0, None)
    assert rc == -1 and b"mask" in L.ente_last_error()


def test_workspace_sizes_are_host_only():
    L = nat.lib()
    table = nat.chunk_table([0, 30000], [30000, 30000])
    n = L.ente_search_workspace_size(table, 2, 7, 3, 4)
    # fp32 copy (8 floats / padded row) + events (16 x u32 / row) dominate
    assert n > 60000 * (8 * 4 + 16 * 4)
    assert L.ente_te_reduce_workspace_size(table, 2) >= 2 * 60000 * 8
    assert L.ente_jitter_workspace_size(2, 7) > 0
    table = nat.chunk_table([0, 10], [10, 20])
    assert L.ente_radius_counts_workspace_size(table, 2, 7) > 0
    assert L.ente_search_path(7, nat.masks_array([0b1110, 0b1111, 0b1111110]), 3, 4) == 1
    assert L.ente_search_path(7, nat.masks_array([0b101]), 1, 4) == 2
    assert L.ente_search_path(20, nat.masks_array([1]), 1, 4) == 0


def test_chunk_struct_layout():
    assert ctypes.sizeof(nat.ChunkDesc) == 16


def test_pyhost_scan_matches_numpy_attributes():
    """The C buffer-protocol scan (csrc/pyhost.cpp) built beside the library
    reports each chunk's data pointer, byte size and row count."""
    from paper_1401_4068_b200 import engine

    assert engine._pyhost is not None, "_pyhost was not built (python -m paper_1401_4068_b200.build)"
    rng = np.random.default_rng(0)
    arrs = [np.ascontiguousarray(rng.standard_normal((int(n), 5))) for n in rng.integers(1, 50, 30)]
    a, s, r = engine._scan(arrs)
    assert a.tolist() == [x.ctypes.data for x in arrs]
    assert s.tolist() == [x.nbytes for x in arrs]
    assert r.tolist() == [x.shape[0] for x in arrs]
    with pytest.raises((BufferError, ValueError)):  # numpy: ValueError, not C-contiguous
        engine._scan([np.zeros((4, 4))[:, ::2]])
