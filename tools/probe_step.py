"""Development probe: C2 step time under the bench's instrumentation variants."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import bench
from paper_1401_4068_b200 import _native as nat, workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.inference import PairPipeline, cached_permutation, analyze_pair

wl = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
x, y = wl.ensembles()
spec = EmbeddingSpec(*wl.spec)
s = wl.n_surrogates
cfg = AnalysisConfig(u_candidates=wl.u_candidates, window=wl.window, k=wl.k, n_surrogates=s, seed=0)
X, Y = EnsembleSeries("X", x), EnsembleSeries("Y", y)
pipe = PairPipeline(X, Y, spec, spec, cfg)
pipe.set_perms([cached_permutation(0, i, x.shape[0], True) for i in range(s)])
items = wl.items(s)


def timed(tag, fn, n=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    print(f"{tag:30s} event {a.elapsed_time(b)/n:8.1f} ms  wall {(time.perf_counter()-t0)/n*1e3:8.1f} ms", flush=True)


timed("pipe.run plain", lambda: pipe.run(items))
timed("analyze_pair", lambda: analyze_pair(X, Y, spec, spec, cfg))
with nat.KernelProfile():
    timed("pipe.run profiled", lambda: pipe.run(items))
    prof = nat.KernelProfile.read()
print({k: round(v["ms"], 1) for k, v in prof.items()})
clk = bench.ClockSampler(0).__enter__()
timed("pipe.run + clocks", lambda: pipe.run(items))
clk.__exit__(None, None, None)
timed("pipe.run plain again", lambda: pipe.run(items))

# stage timing of one wave (host-synchronised between stages)
from paper_1401_4068_b200 import ksg, engine
L = nat.lib()
it = pipe._items(items)
for rep in range(4):
    T = {}
    def mark(tag, t0=[0]):
        torch.cuda.synchronize(); t = time.perf_counter(); T[tag] = (t - t0[0]) * 1e3; t0[0] = t
    mark("start")
    n = len(it)
    pts = torch.empty((n * pipe.m, pipe.dim), dtype=torch.float64, device="cuda")
    mark("alloc")
    nat.check(L.ente_pack_te_items(nat.ptr(pipe.x), nat.ptr(pipe.y), pipe.reps, pipe.n_samples,
                                   pipe.sx.dim, pipe.sx.delay, pipe.sy.dim, pipe.sy.delay, pipe.w,
                                   it.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int32)), n,
                                   nat.ptr(pipe.perm_dev), nat.ptr(pts), nat.stream_handle()), "pack")
    mark("pack")
    rows0 = np.arange(n, dtype=np.int64) * pipe.m
    ns = np.full(n, pipe.m, dtype=np.int64)
    states = pipe._states(it)
    mark("states")
    status = ksg.jitter_device(pts, rows0, ns, 1e-8, states)
    mark("jitter")
    _, counts, _ = engine.search_device(pts, rows0, ns, ksg.te_masks(3, 3), 4)
    mark("search")
    te = ksg.te_reduce_device(counts, rows0, ns, 4)
    mark("reduce")
    te.cpu()
    mark("d2h")
    del T["start"]
    print({k: round(v, 1) for k, v in T.items()}, flush=True)
