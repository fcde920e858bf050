"""Feasibility of shared y-point-set counting on C2 (statistics only).

Every chunk of an analyze_pair batch has the same y columns (y_t, y-past)
point multiset: surrogates permute target repetitions, u moves only x-past.
For each original point p: R_p = max over all chunks of eps at the row whose
y-part is p; list sizes = #{q : D_ypast(p, q) <= R_p} (3-D) and the 4-D
(y_t + y-past) one.  Prints their distribution.
"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_1401_4068_b200 import _native as nat, workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.inference import PairPipeline, surrogate_perms
from paper_1401_4068_b200.ksg import jitter_device
from paper_1401_4068_b200.engine import search_device, radius_counts, Chunk

wl = workloads.CONFIGS["C2"]
x, y = wl.ensembles()
spec = EmbeddingSpec(*wl.spec)
s = wl.n_surrogates
cfg = AnalysisConfig(u_candidates=wl.u_candidates, window=wl.window, k=4, n_surrogates=s, seed=0)
pipe = PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec, spec, cfg)
perms = surrogate_perms(0, s, x.shape[0], True)
pipe.set_perms(perms)
items = pipe._items(wl.items(s))
n_items = len(items)
m, w, reps = pipe.m, pipe.w, pipe.reps
L = nat.lib()
Rp = np.zeros(m)
eps_all_typ = []
for s0 in range(0, n_items, 400):
    it = items[s0:s0 + 400]
    n = len(it)
    pts = torch.empty((n * m, pipe.dim), dtype=torch.float64, device="cuda")
    nat.check(L.ente_pack_te_items(nat.ptr(pipe.x), nat.ptr(pipe.y), reps, pipe.n_samples,
                                   spec.dim, spec.delay, spec.dim, spec.delay, w,
                                   it.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int32)), n,
                                   nat.ptr(pipe.perm_dev), nat.ptr(pts), nat.stream_handle()), "pack")
    rows0 = np.arange(n, dtype=np.int64) * m
    ns = np.full(n, m, dtype=np.int64)
    st = jitter_device(pts, rows0, ns, 1e-8, pipe._states(it))
    eps, _, _ = search_device(pts, rows0, ns, [], 4)
    e = eps.cpu().numpy().reshape(n, m)
    for c in range(n):
        idx = int(it[c, 1])
        phi = np.arange(reps) if idx < 0 else perms[idx]
        p = (phi[:, None] * w + np.arange(w)[None, :]).reshape(-1)  # row (r, t) -> y source p
        np.maximum.at(Rp, p, e[c])
    eps_all_typ.append(np.median(e))
print("eps median", np.median(eps_all_typ), "R_p: median", np.median(Rp), "p99", np.percentile(Rp, 99), "max", Rp.max())
# original y columns of the pair (u=1 original chunk, unjittered)
it = items[:1]
pts = torch.empty((m, pipe.dim), dtype=torch.float64, device="cuda")
nat.check(L.ente_pack_te_items(nat.ptr(pipe.x), nat.ptr(pipe.y), reps, pipe.n_samples,
                               spec.dim, spec.delay, spec.dim, spec.delay, w,
                               it.ctypes.data_as(nat.ctypes.POINTER(nat.ctypes.c_int32)), 1,
                               nat.ptr(pipe.perm_dev), nat.ptr(pts), nat.stream_handle()), "pack")
Y = pts.cpu().numpy()
R = Rp * (1 + 1e-6) + 1e-6
for name, cols in (("ypast 3D", [1, 2, 3]), ("y_ypast 4D", [0, 1, 2, 3])):
    cnt = radius_counts(Chunk(np.ascontiguousarray(Y[:, cols])), R)
    print(name, "list sizes: mean %.0f median %.0f p99 %.0f max %d total %.3e" %
          (cnt.mean(), np.median(cnt), np.percentile(cnt, 99), cnt.max(), cnt.sum()))
