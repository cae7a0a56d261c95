#!/bin/bash
# round-2 GPU job AZ: same-box A/B of the final-O commit order (last vs before the stage release)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/az_build.log 2>&1 || { tail -30 gpurun_out/az_build.log; exit 1; }
python - > gpurun_out/az_variants.log 2>&1 <<'PY' || { tail gpurun_out/az_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('ofirst', ['HI_O_COMMIT_FIRST=1'])]
with ThreadPoolExecutor(2) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
for rep in 1 2 3; do
  for v in base ofirst; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/az_ab.jsonl 2>> gpurun_out/az_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/az_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r.get('dist', ''), r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
