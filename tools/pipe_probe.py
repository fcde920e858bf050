"""Host-side phase timing of one pipelined batch_search wave (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1401_4068_b200 import engine, workloads  # noqa: E402
from paper_1401_4068_b200.engine import Chunk, batch_search  # noqa: E402

orig_upload, orig_search, orig_asm = engine._upload, engine.search_device, engine._assemble
T = []


def up(*a, **k):
    t = time.perf_counter()
    r = orig_upload(*a, **k)
    T.append(("upload", time.perf_counter() - t))
    return r


def se(*a, **k):
    t = time.perf_counter()
    r = orig_search(*a, **k)
    T.append(("search", time.perf_counter() - t))
    return r


def asm(*a, **k):
    t = time.perf_counter()
    r = orig_asm(*a, **k)
    T.append(("assemble", time.perf_counter() - t))
    return r


engine._upload, engine.search_device, engine._assemble = up, se, asm
for cell in sys.argv[1:]:
  n, dim, chunks = (int(v) for v in cell.split(","))
  margs = workloads.c3_marginals(dim, "te")
  base = [workloads.c3_chunk(n, dim, c, False) for c in range(16)]
  items = [(Chunk(base[c % 16].copy(), chunk_id=c), margs) for c in range(chunks)]
  for it in range(5):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = batch_search(items, 4)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    up_ms = sum(b for a, b in T if a == "upload") * 1e3
    asm_ms = sum(b for a, b in T if a == "assemble") * 1e3
    print(f"{cell} call {it}: {tot * 1e3:.1f} ms; upload {up_ms:.1f} assemble {asm_ms:.1f} parts "
          f"{sum(1 for a, _ in T if a == 'search')}", flush=True)
