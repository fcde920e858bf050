#!/bin/bash
# A/B the pipeline step over library variants: tools/ab.sh <config> lib1.so lib2.so ...
cfg=$1; shift; surr=${SURR:-}
for l in "$@"; do
  if [ "$l" = default ]; then timeout 300 python tools/ab_step.py $cfg $surr; else ENTE_LIB=$l timeout 300 python tools/ab_step.py $cfg $surr; fi
done
