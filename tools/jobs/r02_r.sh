#!/bin/bash
# round-2 GPU job R: ceilings without the exponentials (HI_FAKE_SOFTMAX) for the product kernel and the P-in-smem one
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1 || { tail -30 gpurun_out/r_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('basefake', ['HI_FAKE_SOFTMAX=1']); b.build_variant('psmfake', ['HI_PSMEM_DEFAULT=1', 'HI_FAKE_SOFTMAX=1'])" > gpurun_out/r_variants.log 2>&1 || { tail gpurun_out/r_variants.log; exit 1; }
for v in basefake psmfake; do
  HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 6 >> gpurun_out/r_ab.jsonl 2>> gpurun_out/r_ab.err
done
cat gpurun_out/r_ab.jsonl
