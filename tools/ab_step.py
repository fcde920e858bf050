"""A/B timing of one config's pipeline step for the library named by ENTE_LIB."""
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
ref = pipe.run(items)
for _ in range(2):
    pipe.run(items)
torch.cuda.synchronize()
nat.search_work()
with nat.KernelProfile():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        te = pipe.run(items)
    b.record(); torch.cuda.synchronize()
    prof = nat.KernelProfile.read()
assert np.array_equal(te, ref)
ks = nat.search_work()
print(json.dumps({"lib": os.environ.get("ENTE_LIB", "default"), "config": name,
                  "ms_per_step": a.elapsed_time(b) / 3, "te_sum": float(te.sum()),
                  "kernels": {k: round(v["ms"] / 3, 2) for k, v in prof.items()},
                  "subtiles_per_step": [v / 3 for v in ks]}), flush=True)
