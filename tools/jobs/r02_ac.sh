#!/bin/bash
# round-2 GPU job AC: separate K / V stage release (K(i+2) prefetched 2.5 tile steps ahead): parity, then the sustained
# 1M probe against the joint release (HI_KV_JOINT=1), with and without the softmax math
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ac_build.log 2>&1 || { tail -30 gpurun_out/ac_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py tests/test_gpu_hazards.py tests/test_gpu_fullsize.py -x -q > gpurun_out/ac_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ac_tests.log
python - > gpurun_out/ac_variants.log 2>&1 <<'PY' || { tail gpurun_out/ac_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('joint', ['HI_KV_JOINT=1']), ('fake', ['HI_FAKE_SOFTMAX']), ('fakejoint', ['HI_FAKE_SOFTMAX', 'HI_KV_JOINT=1'])]
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
for rep in 1 2 3; do
  for v in base joint fake fakejoint; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/ac_ab.jsonl 2>> gpurun_out/ac_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/ac_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
