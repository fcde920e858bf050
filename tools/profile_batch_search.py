"""Host-side phase timing of batch_search on a C3 cell (e2e vs device).

    python tools/profile_batch_search.py n dim chunks layout
"""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.engine import Chunk, batch_search

n, dim, chunks, layout = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
margs = workloads.c3_marginals(dim, layout)
host = [workloads.c3_chunk(n, dim, c) for c in range(chunks)]
items = [(Chunk(p, chunk_id=i), margs) for i, p in enumerate(host)]
for _ in range(3):
    res = batch_search(items, 4)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    res = batch_search(items, 4)
torch.cuda.synchronize()
print(f"batch_search {(time.perf_counter() - t) / 3 * 1e3:.1f} ms per call")
pr = cProfile.Profile()
pr.enable()
res = batch_search(items, 4)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
print(s.getvalue())
