#!/bin/bash
# NEXT-2 head-group sweep (Tab. 5-7 style): prefill/decode time vs kv heads per unit, at short and long contexts.
cd "$(dirname "$0")/.."
for cfg in "16384 4 2048" "32768 4 4096" "131072 4 18944"; do
  set -- $cfg
  for G in 1 2 4 8; do
    echo "== ctx=$1 L=$2 chunk=$3 G=$G"
    HI_QP_GROUP=$G timeout 300 python tools/quick_perf.py $1 $2 $3 2>&1 > /tmp/qp.txt; grep "prefill chunk" /tmp/qp.txt | tail -1; grep "decode s=" /tmp/qp.txt | tail -1
  done
done
