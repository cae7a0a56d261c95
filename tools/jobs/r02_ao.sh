#!/bin/bash
# round-2 GPU job AO: MMA descriptors passed as low words only (HI_DESC_LO, ~13 instead of ~19 issue-warp
# instructions per tcgen05.mma): parity, then the sustained probe vs HI_DESC_LO=0
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ao_build.log 2>&1 || { tail -30 gpurun_out/ao_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py tests/test_gpu_fullsize.py -x -q > gpurun_out/ao_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ao_tests.log
python - > gpurun_out/ao_variants.log 2>&1 <<'PY' || { tail gpurun_out/ao_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('lo0', ['HI_DESC_LO=0'])]
with ThreadPoolExecutor(2) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
for rep in 1 2 3; do
  for v in base lo0; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/ao_ab.jsonl 2>> gpurun_out/ao_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/ao_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r.get('dist', ''), r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
