"""Host/device timeline of consecutive pipeline steps (development tool).

Wraps the library's entry points with host timestamps and CUDA events so
host-side gaps between launches show up."""
import sys, os, time, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_1401_4068_b200 import _native as nat, workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.inference import PairPipeline, cached_permutation

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
wl = workloads.CONFIGS[name]
x, y = wl.ensembles()
spec = EmbeddingSpec(*wl.spec)
s = int(sys.argv[2]) if len(sys.argv) > 2 else wl.n_surrogates
cfg = AnalysisConfig(u_candidates=wl.u_candidates, window=wl.window, k=wl.k, n_surrogates=s, seed=0)
pipe = PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec, spec, cfg)
pipe.set_perms([cached_permutation(0, i, x.shape[0], True) for i in range(s)])
items = wl.items(s)
L = nat.lib()
log = []


class Wrap:
    def __init__(self, fn, tag):
        self.fn, self.tag = fn, tag
        self.argtypes, self.restype = fn.argtypes, fn.restype

    def __call__(self, *a):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter(); e0.record()
        r = self.fn(*a)
        e1.record(); h1 = time.perf_counter()
        log.append((self.tag, h0, h1, e0, e1))
        return r


for nm in ("ente_pack_te_items", "ente_jitter", "ente_search", "ente_te_reduce"):
    setattr(L, nm, Wrap(getattr(L, nm), nm))
from paper_1401_4068_b200 import ksg, engine
hlog = []


def htime(mod, nm):
    fn = getattr(mod, nm)

    def w(*a, **k):
        h0 = time.perf_counter()
        r = fn(*a, **k)
        hlog.append((nm, h0, time.perf_counter()))
        return r
    setattr(mod, nm, w)


for mod, nm in ((ksg, "jitter_device"), (ksg, "search_device"), (ksg, "te_reduce_device"),
                (nat, "workspace"), (nat, "scratch"), (nat, "chunk_table")):
    htime(mod, nm)
import gc
gc.callbacks.append(lambda phase, info: hlog.append(("gc-" + phase, time.perf_counter(), time.perf_counter())))
for it in range(8):
    hlog.clear()
    log.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); g0 = torch.cuda.Event(enable_timing=True); g0.record()
    pipe.run(items)
    g1 = torch.cuda.Event(enable_timing=True); g1.record(); torch.cuda.synchronize()
    t1 = time.perf_counter()
    rows = []
    for tag, h0, h1, e0, e1 in log:
        rows.append(f"{tag[5:]}: host@{(h0-t0)*1e3:.1f}+{(h1-h0)*1e3:.1f} dev@{g0.elapsed_time(e0):.1f}+{e0.elapsed_time(e1):.1f}")
    print("   host:", " ".join(f"{nm}@{(h0-t0)*1e3:.1f}+{(h1-h0)*1e3:.1f}" for nm, h0, h1 in hlog))
    print(f"step {it}: wall {(t1-t0)*1e3:.1f} dev {g0.elapsed_time(g1):.1f} | " + " | ".join(rows), flush=True)
