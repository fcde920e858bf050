#!/bin/bash
# One GPU session: bench line, ncu launch list, ncu --set full of the two sweeps
# on the bench's own launches (C2, 2010 chunks), summaries under gpurun_out/.
#   tools/gpu_profile.sh <tag> [config]
set -u
tag=${1:-r01}
cfg=${2:-C2}
mkdir -p gpurun_out
timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/${tag}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/${tag}_launches.log 2>&1
echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'knn_pass|knn_compact|count_pass' -c 2 \
    -o gpurun_out/${tag}_prof -f python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_ncu.log
python tools/ncu_summary.py gpurun_out/${tag}_prof.ncu-rep > gpurun_out/${tag}_ncu_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_prof.ncu-rep --traffic --merge profiles/ncu_traffic.json --config $cfg > gpurun_out/${tag}_ncu_traffic.json 2>&1
cp profiles/ncu_traffic.json gpurun_out/${tag}_ncu_traffic_all.json
cat gpurun_out/${tag}_ncu_traffic.json
# instruction mix / hot lines of the two sweeps (text), then drop the report
# unless KEEP_REP=1 (gpurun copies back at most 64 MiB)
python tools/ncu_hot.py gpurun_out/${tag}_prof.ncu-rep count_pass > gpurun_out/${tag}_count_mix.txt 2>&1
python tools/ncu_hot.py gpurun_out/${tag}_prof.ncu-rep knn > gpurun_out/${tag}_knn_mix.txt 2>&1
if [ "${KEEP_REP:-0}" != "1" ]; then rm -f gpurun_out/${tag}_prof.ncu-rep; fi
