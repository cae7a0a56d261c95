#!/bin/bash
# round-2 GPU job AF: with the K/V release change, re-test the P release point (96 keys), 1/8 FMA-pipe exponentials,
# and both
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/af_build.log 2>&1 || { tail -30 gpurun_out/af_build.log; exit 1; }
python - > gpurun_out/af_variants.log 2>&1 <<'PY' || { tail gpurun_out/af_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('ks96', ['HI_P_SPLIT_KEYS=96']), ('m01', ['HI_POLY_MASK8=0x01']), ('ks96m01', ['HI_P_SPLIT_KEYS=96', 'HI_POLY_MASK8=0x01'])]
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
for rep in 1 2 3; do
  for v in base ks96 m01 ks96m01; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/af_ab.jsonl 2>> gpurun_out/af_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/af_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
