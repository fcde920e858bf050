"""Host enqueue time per stage of one TE step (development probe; no syncs
inside the step), against the device step time.

    python tools/c4_host.py [C4]
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1401_4068_b200 import engine, inference, ksg, scheduler  # noqa: E402
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C4"
wl, s, x, y = bench.workload(cfg_name, None)
spec = EmbeddingSpec(*wl.spec)
cfg = AnalysisConfig(u_candidates=wl.u_candidates, window=wl.window, k=wl.k, n_surrogates=s, seed=wl.seed)
series = bench._series_of(wl, x, y)
pipes, flat, costs = bench._job(wl, s, series, cfg)
run = scheduler.pipeline_runner(pipes)
T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        T[name] = T.get(name, 0.0) + (time.perf_counter() - t) * 1e3
        return r
    setattr(mod, name, g)


for mod, name in [(ksg, "jitter_device"), (ksg, "search_device"), (ksg, "search_te_shared_device"),
                  (ksg, "te_reduce_device"), (inference.PairPipeline, "_states"),
                  (inference.PairPipeline, "shared_y"), (inference.PairPipeline, "_sub")]:
    if hasattr(mod, name):
        wrap(mod, name)
for _ in range(3):
    run(flat)
torch.cuda.synchronize()
for rep in range(3):
    T.clear()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    vals, st = run(flat)
    b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"{cfg_name} step: device {a.elapsed_time(b):.1f} ms, wall {wall:.1f} ms; host ms:",
          {k: round(v, 1) for k, v in T.items()}, flush=True)
