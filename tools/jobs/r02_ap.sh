#!/bin/bash
# round-2 GPU job AP: one MMA issuer warp per Q tile (HI_TWO_ISSUERS=1): parity through the variant library, then the
# sustained 1M probe against the product
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ap_build.log 2>&1 || { tail -30 gpurun_out/ap_build.log; exit 1; }
python - > gpurun_out/ap_variants.log 2>&1 <<'PY' || { tail gpurun_out/ap_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('two', ['HI_TWO_ISSUERS=1'])]
with ThreadPoolExecutor(2) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
HI_LIB_VARIANT=two timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py tests/test_gpu_fullsize.py -x -q > gpurun_out/ap_tests.log 2>&1; echo "two tests rc=$?"; tail -2 gpurun_out/ap_tests.log
for rep in 1 2 3; do
  for v in base two; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/ap_ab.jsonl 2>> gpurun_out/ap_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/ap_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r.get('dist', ''), r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
