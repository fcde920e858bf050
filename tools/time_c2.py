"""Quick timing of the C2 pipeline stages (development tool)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.inference import PairPipeline, cached_permutation, analyze_pair
from paper_1401_4068_b200 import ksg, engine
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nsurr = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = workloads.CONFIGS[name]
xv, yv = wl.ensembles()
spec = EmbeddingSpec(*wl.spec)
cfg = AnalysisConfig(u_candidates=wl.u_candidates, window=wl.window, k=4, n_surrogates=nsurr, seed=0)
X, Y = EnsembleSeries("X", xv), EnsembleSeries("Y", yv)
pipe = PairPipeline(X, Y, spec, spec, cfg)
pipe.set_perms([cached_permutation(0, i, xv.shape[0], True) for i in range(nsurr)])
items = [(u, -1) for u in wl.u_candidates] + [(u, i) for u in wl.u_candidates for i in range(nsurr)]
pipe.run(items[:4]); torch.cuda.synchronize()
# stage timing
L = __import__('paper_1401_4068_b200._native', fromlist=['x'])
m = pipe.m; n = len(items)
t0 = time.perf_counter()
te = pipe.run(items); torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"{name}: {n} chunks of {m} points: {t1-t0:.3f} s -> {n/(t1-t0):.1f} TE/s")
# search-only timing on packed data
rows0 = np.arange(n, dtype=np.int64) * m
pts = torch.empty((n*m, pipe.dim), dtype=torch.float64, device='cuda')
import ctypes
it = np.ascontiguousarray(np.array(items, dtype=np.int32))
from paper_1401_4068_b200 import _native as nat
nat.check(nat.lib().ente_pack_te(nat.ptr(pipe.x), nat.ptr(pipe.y), pipe.reps, pipe.n_samples, spec.dim, spec.delay, spec.dim, spec.delay, pipe.t_lo, pipe.t_hi, it.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n, nat.ptr(pipe.perm_dev), nat.ptr(pts), nat.stream_handle()), "pack")
masks = ksg.te_masks(spec.dim, spec.dim)
for rep in range(3):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); eps, counts, st = engine.search_device(pts, rows0, [m]*n, masks, 4); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    D = pipe.dim
    W = 2 * D * m * (m - 1) * n
    print(f"search: {ms:.2f} ms  PCE/s {W/ms/1e-3:.3e}  frac(74.4T/2) {W/ms/1e-3/3.72e13:.3f}")
