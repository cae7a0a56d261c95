#!/bin/bash
# round-2 GPU job AB: the CTA-pair (cta_group::2) kernel with the warp-converged issue: parity, then the sustained
# 1M probe against the product kernel (interleaved)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1 || { tail -30 gpurun_out/ab_build.log; exit 1; }
python -c "from paper_2502_12574_b200 import build as b; b.build_variant('cmp', [])" > gpurun_out/ab_variants.log 2>&1 || { tail gpurun_out/ab_variants.log; exit 1; }
HI_LIB_VARIANT=cmp timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -k "pair" > gpurun_out/ab_tests.log 2>&1; echo "pair tests rc=$?"; tail -3 gpurun_out/ab_tests.log
for rep in 1 2 3; do
  HI_LIB_VARIANT=cmp timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/ab_ab.jsonl 2>> gpurun_out/ab_ab.err
  HI_LIB_VARIANT=cmp timeout 300 python tools/prefill_probe.py --seconds 8 --flags 0x20 >> gpurun_out/ab_ab.jsonl 2>> gpurun_out/ab_ab.err
done
python -c "
import json
for l in open('gpurun_out/ab_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
