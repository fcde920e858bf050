#!/bin/bash
# A/B of two library builds on the bench configs (kernel ms from live events).
#   tools/ab.sh <baseline.so> <tag> [configs...]
cd $GRAFT_REPO_ROOT
base=$1; tag=$2; shift 2
cfgs=${@:-C2 C1 C4}
for c in $cfgs; do
  for v in base new; do
    if [ $v = base ]; then export ENTE_LIB=$base; else unset ENTE_LIB; fi
    python bench.py --config $c --steps 5 --no-cpu --no-weak --no-e2e > gpurun_out/ab_${tag}_${v}_$c.json 2> gpurun_out/ab_${tag}_${v}_$c.err
  done
done
unset ENTE_LIB
python - "$tag" $cfgs <<'P'
import json, sys
tag = sys.argv[1]
for c in sys.argv[2:]:
    for v in ["base", "new"]:
        try:
            d = json.loads(open(f"gpurun_out/ab_{tag}_{v}_{c}.json").read().strip().splitlines()[-1])
            k = d["roofline"]["kernels_ms_per_step"]
            top = sorted(k.items(), key=lambda x: -x[1])[:5]
            print(c, v, round(d["value"]), round(d["ms_per_step"], 2), " ".join(f"{a}:{b:.2f}" for a, b in top))
        except Exception as e:
            print(c, v, "ERR", e)
P
