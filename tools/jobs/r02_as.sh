#!/bin/bash
# round-2 GPU job AS: tile-to-warp mixing (HI_TILE_MIX=1: each tile's softmax warps get the higher issue priority on
# two of the four SMSPs): parity through the variant library, then the sustained probe vs the product
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/as_build.log 2>&1 || { tail -30 gpurun_out/as_build.log; exit 1; }
python - > gpurun_out/as_variants.log 2>&1 <<'PY' || { tail gpurun_out/as_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('mix', ['HI_TILE_MIX=1'])]
with ThreadPoolExecutor(2) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
HI_LIB_VARIANT=mix timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py -x -q > gpurun_out/as_tests.log 2>&1; echo "mix tests rc=$?"; tail -2 gpurun_out/as_tests.log
for rep in 1 2 3; do
  for v in base mix; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/as_ab.jsonl 2>> gpurun_out/as_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/as_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r.get('dist', ''), r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
