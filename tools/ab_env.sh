#!/bin/bash
# A/B the pipeline step over environment settings: tools/ab_env.sh <config> "VAR=a" "VAR=b" ...
cfg=$1; shift; surr=${SURR:-}
for e in "$@"; do
  env $e timeout 300 python tools/ab_step.py $cfg $surr | sed "s/^/[$e] /"
done
