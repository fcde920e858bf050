#!/bin/bash
# One GPU session: bench line, ncu launch list, ncu --set full of the two sweeps.
#   tools/gpu_profile.sh <tag>      (outputs under gpurun_out/<tag>_*)
set -u
tag=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; tail -c 4000 gpurun_out/${tag}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/${tag}_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'knn_pass|count_pass' -c 2 \
    -o gpurun_out/${tag}_prof -f python tools/profile_run.py C2 8 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_ncu.log
