#!/bin/bash
# round-2 GPU job BD: FMA-pipe exponential shares (1/8, 1/4) re-tested on the final kernel, same box, interleaved
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bd_build.log 2>&1 || { tail -30 gpurun_out/bd_build.log; exit 1; }
python - > gpurun_out/bd_variants.log 2>&1 <<'PY' || { tail gpurun_out/bd_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('m01', ['HI_POLY_MASK8=0x01']), ('m11', ['HI_POLY_MASK8=0x11'])]
with ThreadPoolExecutor(3) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
for rep in 1 2 3; do
  for v in base m01 m11; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/bd_ab.jsonl 2>> gpurun_out/bd_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/bd_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r.get('dist', ''), r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
