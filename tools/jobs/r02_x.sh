#!/bin/bash
# round-2 GPU job X: with warp-converged issue, re-test softmax-side options (rolled issue, 2 warps per row,
# speculative first half) on the sustained 1M probe
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1 || { tail -30 gpurun_out/x_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('roll', ['HI_ROLL_ISSUE=1']); b.build_variant('s2roll', ['HI_ROLL_ISSUE=1', 'HI_SOFTMAX_SPLIT=2']); b.build_variant('spec', ['HI_SPEC_SPLIT=1'])" > gpurun_out/x_variants.log 2>&1 || { tail gpurun_out/x_variants.log; exit 1; }
for rep in 1 2; do
  for v in base roll s2roll spec; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/x_ab.jsonl 2>> gpurun_out/x_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/x_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
