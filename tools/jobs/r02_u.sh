#!/bin/bash
# round-2 GPU job U: two softmax warps per row (SPLIT = 2) with rolled MMA-issue loops vs the product kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1 || { tail -30 gpurun_out/u_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('roll', ['HI_ROLL_ISSUE=1']); b.build_variant('s2', ['HI_ROLL_ISSUE=1', 'HI_SOFTMAX_SPLIT=2']); b.build_variant('s2spec', ['HI_ROLL_ISSUE=1', 'HI_SOFTMAX_SPLIT=2', 'HI_SPEC_SPLIT=1'])" > gpurun_out/u_variants.log 2>&1 || { tail gpurun_out/u_variants.log; exit 1; }
HI_LIB_VARIANT=s2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or group_size or chunk_size" > gpurun_out/u_parity.log 2>&1; echo "s2 parity rc=$?"; tail -2 gpurun_out/u_parity.log
for rep in 1 2; do
  for v in base roll s2 s2spec; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/u_ab.jsonl 2>> gpurun_out/u_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/u_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
