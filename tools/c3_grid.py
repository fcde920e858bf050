"""C3 sweep: kNN + range searches/s per chunk shape, with a CPU baseline per shape.

    python tools/c3_grid.py [--out profiles/r02_c3.jsonl] [--budget-s 1.5] [--quick]

SURVEY.md 8(d) C3: n in {1k..64k} U {30094} points per chunk x chunks in
{1, 10, 100, 1000, 10000} x joint dims 3..17 (odd), two layouts (te: the
three KSG marginals with d_y = d_x = (D-1)/2; bench: one marginal, the first
(D-1)/2 columns, bench.py:56), plus the tied variant of a few shapes and the
64-chunk paper-geometry cell of acceptance criterion 8 (30094 x 17, bench).

One JSON line per cell, in one process (a bench.py run per cell would pay the
CUDA/numba start-up 640 times):
  value        device-resident searches/s (CUDA events, 2 warm-up + 3 steps;
               inputs larger than L2 or L2 flushed between steps)
  roofline     dominant sweep: algorithmic work / time / nominal FP32 peak,
               and the lane-level evaluated work (bench.roofline_of)
  cpu_baseline the unmodified reference (ente.engine.batch_search, numba, all
               host threads; oracle/_ref) on 1-2 chunks of the shape, or the C
               port when the reference is not staged (bench.c3_cpu_sample)
  e2e          batch_search from host numpy (cells up to 1 GB of input)
Chunks of a cell are 16 distinct generated chunks tiled (the reference's
run_bench duplicates one chunk, bench.py:64).  Cells whose predicted step
exceeds --budget-s, or that exceed one device wave (2^27 rows), are skipped.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1401_4068_b200 import _native as nat, workloads  # noqa: E402
from paper_1401_4068_b200.engine import Chunk, batch_search, column_mask, search_device  # noqa: E402

K = 4
NS = [1024, 2048, 4096, 8192, 16384, 30094, 32768, 65536]
DIMS = [3, 5, 7, 9, 11, 13, 15, 17]
CHUNKS = [1, 10, 100, 1000, 10000]
MAX_ROWS = 1 << 27


_FLUSH = {}


def flush_ms(flush):
    if "ms" not in _FLUSH:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        a.record()
        for _ in range(20):
            flush.zero_()
        b.record()
        torch.cuda.synchronize()
        _FLUSH["ms"] = a.elapsed_time(b) / 20
    return _FLUSH["ms"]


def run_cell(n, dim, chunks, layout, tied, base_host, flush, warmup=2, steps=3):
    margs = workloads.c3_marginals(dim, layout)
    masks = [column_mask(c, dim) for c in margs]
    reps = (chunks + len(base_host) - 1) // len(base_host)
    host = np.concatenate([np.concatenate(base_host)] * reps)[:chunks * n]
    pts = torch.from_numpy(host).cuda()
    rows0 = np.arange(chunks, dtype=np.int64) * n
    ns = np.full(chunks, n, dtype=np.int64)
    small = chunks * n * dim * 8 < 2 * 126e6

    def step():
        if small:
            flush.zero_()
        search_device(pts, rows0, ns, masks, K, reuse=True)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    nat.search_work()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with nat.KernelProfile():
        start.record()
        for _ in range(steps):
            step()
        stop.record()
        torch.cuda.synchronize()
        prof = nat.KernelProfile.read()
    knn_sub, cnt_sub = nat.search_work()
    ms = start.elapsed_time(stop) / steps
    if small:  # the L2 flush between steps is not search work
        ms = max(ms - flush_ms(flush), 1e-6)
    union = len(set(c for cols in margs for c in cols))
    pairs = chunks * n * (n - 1)
    roof = bench.roofline_of(prof, steps, {"knn_pass": pairs * dim, "count_pass": pairs * union},
                             knn_sub, cnt_sub, dim, 0, f"C3:{n},{dim},{chunks},{layout}", union)
    e2e = None
    if chunks * n * dim * 8 <= 1 << 30:
        items = [(Chunk(host[c * n:(c + 1) * n], chunk_id=c), margs) for c in range(chunks)]
        res = None
        for _ in range(3):  # warm-up shaped like the timed loop (two live result sets)
            res = batch_search(items, K)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            res = batch_search(items, K)
        torch.cuda.synchronize()
        e_s = (time.perf_counter() - t0) / steps
        assert not any(isinstance(r, Exception) for r in res)
        e2e = {"value": chunks * n / e_s, "unit": "searches/s", "ms": e_s * 1e3,
               "h2d_bytes_per_step": chunks * n * dim * 8,
               "d2h_bytes_per_step": chunks * n * (8 + 8 * len(masks)) + 4 * chunks,
               "api": "paper_1401_4068_b200.batch_search"}
    del pts
    return ms, roof, e2e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_c3.jsonl"))
    ap.add_argument("--budget-s", type=float, default=1.5)
    ap.add_argument("--cpu-budget-s", type=float, default=3.0)
    ap.add_argument("--quick", action="store_true", help="a few shapes only (smoke)")
    ap.add_argument("--layouts", default="te,bench")
    ap.add_argument("--dims", default=",".join(map(str, DIMS)))
    ap.add_argument("--tied", action="store_true", help="include the tied shapes")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dims = [int(d) for d in args.dims.split(",")]
    shapes = [(n, d, lay, False) for lay in args.layouts.split(",") for d in dims for n in NS]
    if args.tied:
        shapes += [(30094, 7, "te", True), (30094, 17, "bench", True), (8192, 5, "te", True),
                   (65536, 3, "te", True)]
    if args.quick:
        shapes = [(1024, 3, "te", False), (30094, 17, "bench", False)]
    ref = bench.reference_module()
    clk = bench.ClockSampler(0).__enter__()
    t_start = time.time()
    with open(args.out, "a") as out:
        for n, dim, layout, tied in shapes:
            base = [workloads.c3_chunk(n, dim, c, tied) for c in range(16)]
            cpu = bench.c3_cpu_sample(n, dim, layout, tied, K, budget_s=args.cpu_budget_s,
                                      max_chunks=2)
            chunk_list = list(CHUNKS)
            if (n, dim, layout, tied) == (30094, 17, "bench", False):
                chunk_list = sorted(set(chunk_list + [64]))  # acceptance criterion 8 geometry
            per_chunk_ms = None
            for chunks in chunk_list:
                if chunks * n > MAX_ROWS:
                    continue
                if per_chunk_ms is not None and per_chunk_ms * chunks > args.budget_s * 1e3:
                    continue
                ms, roof, e2e = run_cell(n, dim, chunks, layout, tied, base, flush)
                per_chunk_ms = ms / chunks
                line = {"metric": "kNN+range searches/sec", "value": chunks * n / (ms * 1e-3),
                        "unit": "searches/s", "n_gpus": 1, "ms_per_step": ms, "steps": 3,
                        "warmup": 2, "higher_is_better": True, "dtype": "f32+f64",
                        "config": bench.c3_config(n, dim, chunks, layout, tied, K, 1),
                        "roofline": {k: roof[k] for k in ("kernel", "achieved", "peak", "frac",
                                                          "evaluated_fraction", "evaluated_frac",
                                                          "evaluated_frac_of_measured_loop",
                                                          "kernels_ms_per_step")},
                        "cpu_baseline": cpu, "e2e": e2e,
                        "reference_staged": ref is not None}
                out.write(json.dumps(line) + "\n")
                out.flush()
                print(f"{n:6d} x {dim:2d} {layout:5s}{' tied' if tied else '     '} x {chunks:5d}: "
                      f"{line['value']:.3e} searches/s  ({ms:8.2f} ms)  cpu {cpu['value']:.3e}"
                      f"  e2e {e2e['value'] if e2e else float('nan'):.3e}", flush=True)
    clk.__exit__(None, None, None)
    print(json.dumps({"grid_clocks": clk.summary(), "wall_s": time.time() - t_start}))


if __name__ == "__main__":
    main()
