#!/bin/bash
# round-2 GPU job T: A/B of the LPT order (same box), 3 interleaved repetitions; sanitizer passes
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1 || { tail -30 gpurun_out/t_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('nolpt', ['HI_NO_LPT=1'])" > gpurun_out/t_variants.log 2>&1 || { tail gpurun_out/t_variants.log; exit 1; }
for rep in 1 2 3; do
  for v in base nolpt; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/t_ab.jsonl 2>> gpurun_out/t_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/t_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
bash tools/sanitize.sh; cat gpurun_out/sanitize_summary.txt
