"""Benchmark harness: one batched device search versus a chunk-at-a-time loop.

Drop-in for /root/reference/pkg/src/ente/bench.py (BenchReport 24-39,
_counts_equal 42-45, run_bench 48-96).  Same inputs, same row keys, same
correctness gate: one random chunk (default_rng(seed).standard_normal,
bench.py:54-55) duplicated n_chunks times, marginal = the first
marginal_dim columns (bench.py:56); every timing row is accepted only after
the batched and the sequential results compare bit-identical
(ResultMismatch otherwise, bench.py:84-86).

What "parallel" and "sequential" mean here: the batched arm is ONE
batch_search call, i.e. one device launch sequence over all chunks (the
paper's many-chunks-per-launch design); the sequential arm
is one batch_search call per chunk (one launch sequence each), the GPU
analogue of the reference's single-worker loop.  Timings include the host
upload and read-back of every call, as the reference's include its Python
loop.  Rows add searches/s (reference points per second) of the batched arm.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import Chunk, batch_search, max_workers, set_workers
from .exceptions import ResultMismatch


@dataclass
class BenchReport:
    chunk_points: int
    joint_dim: int
    marginal_dim: int
    k: int
    repeats: int
    hardware: str
    rows: list = field(default_factory=list)  # n_chunks / timings / speedup / searches

    def to_csv(self) -> str:
        lines = ["n_chunks,seconds_parallel,seconds_sequential,speedup"]
        for row in self.rows:
            lines.append(f"{row['n_chunks']},{row['seconds_parallel']!r},"
                         f"{row['seconds_sequential']!r},{row['speedup']!r}")
        return "\n".join(lines) + "\n"


def _counts_equal(a, b) -> bool:
    if not np.array_equal(a.kth_distance, b.kth_distance):
        return False
    return all(np.array_equal(x, y) for x, y in zip(a.radius_counts, b.radius_counts))


def _hardware() -> str:
    if torch.cuda.is_available():
        p = torch.cuda.get_device_properties(torch.cuda.current_device())
        return f"{p.name} ({p.multi_processor_count} SMs) sm_{p.major}{p.minor}"
    return "no CUDA device"


def run_bench(chunk_points: int, joint_dim: int, marginal_dim: int, k: int,
              n_chunks_list, repeats: int = 3, seed: int = 0,
              workers: int | None = None, sequential: bool = True) -> BenchReport:
    """Time batched vs sequential search for each chunk count in n_chunks_list.

    sequential=False skips the chunk-at-a-time arm (its timing and speedup
    are then None) and gates the batched result against a single-chunk
    search of the first chunk instead: every chunk is the same data, so every
    slot must equal it.
    """
    if sorted(n_chunks_list) != list(n_chunks_list):
        raise ValueError("n_chunks_list must be ascending")
    rng = np.random.default_rng(seed)
    points = rng.standard_normal((chunk_points, joint_dim))
    marginal_cols = [list(range(marginal_dim))]
    workers = workers or max_workers()
    report = BenchReport(chunk_points, joint_dim, marginal_dim, k, repeats, _hardware())

    for n_chunks in n_chunks_list:
        items = [(Chunk(points, chunk_id=i), marginal_cols) for i in range(n_chunks)]
        set_workers(workers)
        batch_search(items[:1], k)  # warm-up (library load, workspace growth)
        par_times, par_result = [], None
        for _ in range(repeats):
            t0 = time.perf_counter()
            par_result = batch_search(items, k)
            par_times.append(time.perf_counter() - t0)

        seq_times, seq_result = [], None
        if sequential:
            for _ in range(repeats):
                t0 = time.perf_counter()
                seq_result = [batch_search([item], k)[0] for item in items]
                seq_times.append(time.perf_counter() - t0)
        else:
            seq_result = batch_search(items[:1], k) * n_chunks
        set_workers(workers)

        for a, b in zip(par_result, seq_result):
            if isinstance(a, Exception) or isinstance(b, Exception) or not _counts_equal(a, b):
                raise ResultMismatch(f"parallel/sequential mismatch at n_chunks={n_chunks}")

        sec_par = float(np.median(par_times))
        sec_seq = float(np.median(seq_times)) if seq_times else None
        report.rows.append({
            "n_chunks": n_chunks,
            "seconds_parallel": sec_par,
            "seconds_sequential": sec_seq,
            "speedup": (sec_seq / sec_par) if sec_seq is not None else None,
            "searches_per_s": n_chunks * chunk_points / sec_par,
        })
    return report
