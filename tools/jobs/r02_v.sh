#!/bin/bash
# round-2 GPU job V: warp-converged MMA issue (elect.sync inside tcgen05.mma / commit) vs lane-0 issue
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v_build.log 2>&1 || { tail -30 gpurun_out/v_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('wissue', ['HI_WARP_ISSUE=1'])" > gpurun_out/v_variants.log 2>&1 || { tail gpurun_out/v_variants.log; exit 1; }
HI_LIB_VARIANT=wissue timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py -x -q > gpurun_out/v_parity.log 2>&1; echo "wissue parity rc=$?"; tail -2 gpurun_out/v_parity.log
for rep in 1 2 3; do
  for v in base wissue; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/v_ab.jsonl 2>> gpurun_out/v_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/v_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
