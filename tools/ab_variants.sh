#!/bin/bash
# A/B of library variants (build/variants/libheadinfer_<name>.so) on the prefill probe:
#   tools/ab_variants.sh "<ctx> <layers> <chunk>" reps name1 name2 ...
cd "$(dirname "$0")/.."
cfg=$1; reps=$2; shift 2
for r in $(seq 1 $reps); do
  for v in "$@"; do
    HI_LIB_VARIANT=$v timeout 300 python tools/quick_perf.py $cfg > /tmp/ab_$v.txt 2>&1
    echo "$v rep$r $(grep 'prefill chunk' /tmp/ab_$v.txt | tail -1)"
  done
done
