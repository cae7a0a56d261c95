#!/bin/bash
# round-2 GPU job AE: the one-tile / three-S-buffer kernel (tc1) with the warp-converged issue vs the product kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ae_build.log 2>&1 || { tail -30 gpurun_out/ae_build.log; exit 1; }
python -c "from paper_2502_12574_b200 import build as b; b.build_variant('cmp', [])" > gpurun_out/ae_variants.log 2>&1 || { tail gpurun_out/ae_variants.log; exit 1; }
for rep in 1 2; do
  HI_LIB_VARIANT=cmp timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/ae_ab.jsonl 2>> gpurun_out/ae_ab.err
  HI_LIB_VARIANT=cmp timeout 300 python tools/prefill_probe.py --seconds 8 --flags 0x40 >> gpurun_out/ae_ab.jsonl 2>> gpurun_out/ae_ab.err
done
python -c "
import json
for l in open('gpurun_out/ae_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
