"""Condense tools/ab.sh output: lib, ms/step and the sweep kernels' ms per step."""
import json, sys
for line in sys.stdin:
    try:
        d = json.loads(line)
    except ValueError:
        continue
    k = d["kernels"]
    print(f'{d["lib"]:28s} {d["ms_per_step"]:8.2f} ms  knn {k.get("knn_pass", 0):6.2f}  count {k.get("count_pass", 0):6.2f}'
          f'  te_sum {d["te_sum"]!r}')
