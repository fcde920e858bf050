#!/bin/bash
# C3 sweep: searches/s per chunk shape (one bench.py line per cell).
#   tools/sweep_c3.sh <out.jsonl> [cells...]   cell = n,dim,chunks,layout[,tied]
set -u
out=${1:-gpurun_out/c3_sweep.jsonl}; shift || true
cells=("$@")
if [ ${#cells[@]} -eq 0 ]; then
  cells=(1024,3,10000,te 1024,7,10000,te 1024,17,1000,te
         4096,3,1000,te 4096,7,1000,te 4096,17,100,te
         16384,7,100,te 16384,17,10,te
         30094,17,10,bench 30094,17,10,te 30094,7,100,te 30094,7,100,te,tied
         65536,3,10,te 65536,7,10,te 65536,17,1,te)
fi
mkdir -p "$(dirname "$out")"
: > "$out"
for c in "${cells[@]}"; do
  timeout 300 python bench.py --config C3 --shape "$c" --steps 3 --warmup 3 --no-cpu >> "$out" 2>> "${out%.jsonl}.err"
  echo "cell $c rc=$?"
done
