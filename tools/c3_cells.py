"""Selected C3 cells (device value and batch_search e2e), one JSON line each.

    python tools/c3_cells.py 1024,7,10000,te 1024,5,10000,te ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import c3_grid  # noqa: E402
from paper_1401_4068_b200 import workloads  # noqa: E402


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cell in sys.argv[1:]:
        n, dim, chunks, layout = cell.split(",")
        n, dim, chunks = int(n), int(dim), int(chunks)
        base = [workloads.c3_chunk(n, dim, c, False) for c in range(16)]
        ms, roof, e2e = c3_grid.run_cell(n, dim, chunks, layout, False, base, flush)
        print(json.dumps({"cell": cell, "value": chunks * n / (ms * 1e-3), "ms": ms,
                          "e2e": e2e, "ratio": (chunks * n / (ms * 1e-3)) / e2e["value"]}),
              flush=True)


if __name__ == "__main__":
    main()
