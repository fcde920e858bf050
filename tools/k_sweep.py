"""Time batch_search on one C2-sized chunk for several k (fast path k <= 15, exact path above)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_1401_4068_b200.engine import search_device
rng = np.random.default_rng(0)
n, dim = 30000, 7
pts = torch.from_numpy(rng.standard_normal((n * 8, dim))).cuda()
rows0 = np.arange(8) * n
ns = np.full(8, n)
masks = [0b1110, 0b1111, 0b1111110]
for k in (4, 10, 15, 16, 20, 32):
    search_device(pts, rows0, ns, masks, k, reuse=True); torch.cuda.synchronize()
    t = time.perf_counter()
    search_device(pts, rows0, ns, masks, k, reuse=True); torch.cuda.synchronize()
    print(f"k={k:3d}: {(time.perf_counter() - t) * 1e3:8.1f} ms for 8 chunks of {n}", flush=True)
