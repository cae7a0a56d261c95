#!/bin/bash
# A/B prefill-kernel variants (same sources, different -D flags), interleaved to average out clock drift.
# usage: bash tools/ab_prefill.sh "name1:DEF=1,DEF2=3" "name2:..."   -> gpurun_out/ab_prefill.log
set -u
specs=("$@")
for sp in "${specs[@]}"; do
  name=${sp%%:*}; defs=${sp#*:}
  python -c "from paper_2502_12574_b200 import build as b; b.build_variant('$name', [d for d in '$defs'.split(',') if d])" || exit 1
done
for rep in 1 2 3; do
  for sp in "${specs[@]}"; do
    name=${sp%%:*}
    HI_LIB_VARIANT=$name timeout 120 python tools/quick_perf.py 131072 4 2>&1 | grep "prefill chunk" | tail -2 | sed "s/^/$name rep$rep /" >> gpurun_out/ab_prefill.log
  done
done
