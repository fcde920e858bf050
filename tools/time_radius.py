"""radius_counts on the paper geometry (30094 x 17, caller radii) vs the TE count pass.

    python tools/time_radius.py [chunks]

Prints one JSON line: per-kernel ms of (a) a TE-layout search (d_y = d_x = 8,
the three marginals fused) and (b) ente_radius_counts over all 17 columns
with the kNN radii (the generic path), both device-resident.
"""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
from paper_1401_4068_b200 import _native as nat, workloads
from paper_1401_4068_b200.engine import search_device

chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n, dim = 30094, 17
host = np.concatenate([workloads.c3_chunk(n, dim, c) for c in range(chunks)])
dev = torch.from_numpy(host).cuda()
rows0 = np.arange(chunks, dtype=np.int64) * n
ns = np.full(chunks, n, dtype=np.int64)
te_masks = [sum(1 << c for c in m) for m in workloads.c3_marginals(dim, "te")]
L = nat.lib()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    with nat.KernelProfile():
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t) / reps * 1e3
        prof = nat.KernelProfile.read()
    return wall, {k: round(v["ms"] / reps, 3) for k, v in prof.items()}


eps, _, _ = search_device(dev, rows0, ns, [], 4)
radii = eps.clone()
table = nat.chunk_table(rows0, ns)
out = torch.empty((1, chunks * n), dtype=torch.int32, device="cuda")
status = torch.empty(chunks, dtype=torch.int32, device="cuda")
full = nat.masks_array([(1 << dim) - 1])
ws = nat.workspace(L.ente_radius_counts_workspace_size(table, chunks, dim))


def radius():
    nat.check(L.ente_radius_counts(nat.ptr(dev), chunks * n, dim, table, chunks, full, 1,
                                   nat.ptr(radii), nat.ptr(out), nat.ptr(status), nat.ptr(ws),
                                   ws.numel(), nat.stream_handle()), "ente_radius_counts")


te_wall, te_prof = timed(lambda: search_device(dev, rows0, ns, te_masks, 4, reuse=True))
r_wall, r_prof = timed(radius)
print(json.dumps({"chunks": chunks, "n": n, "dim": dim,
                  "te_search_ms": te_wall, "te_kernels": te_prof,
                  "radius_counts_ms": r_wall, "radius_kernels": r_prof,
                  "radius_vs_te_count_pass": r_prof.get("count_pass", 0) / te_prof["count_pass"]}))
