"""One pipeline pass over a slice of config C2 (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1401_4068_b200 import workloads
from paper_1401_4068_b200.data import AnalysisConfig, EmbeddingSpec, EnsembleSeries
from paper_1401_4068_b200.inference import PairPipeline, cached_permutation
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = workloads.CONFIGS[name]
x, y = wl.ensembles()
spec = EmbeddingSpec(*wl.spec)
cfg = AnalysisConfig(u_candidates=wl.u_candidates, window=wl.window, k=4, n_surrogates=ns, seed=0)
pipe = PairPipeline(EnsembleSeries("X", x), EnsembleSeries("Y", y), spec, spec, cfg)
pipe.set_perms([cached_permutation(0, i, x.shape[0], True) for i in range(ns)])
items = [(u, -1) for u in wl.u_candidates] + [(u, i) for u in wl.u_candidates for i in range(ns)]
te = pipe.run(items)
torch.cuda.synchronize()
print(name, len(items), "chunks", te[:3])
