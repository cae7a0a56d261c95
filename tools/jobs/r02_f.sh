#!/bin/bash
# round-2 GPU job F: MUFU ping-pong variant -- parity on the variant library, then A/B on the sustained 1M probe
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1 || { tail -30 gpurun_out/f_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('pp', ['HI_PINGPONG=1'])" > gpurun_out/f_variants.log 2>&1 || { tail gpurun_out/f_variants.log; exit 1; }
HI_LIB_VARIANT=pp timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py -x -q > gpurun_out/f_pp_tests.log 2>&1; tail -4 gpurun_out/f_pp_tests.log
for rep in 1 2; do
  for v in base pp; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/f_ab.jsonl 2>> gpurun_out/f_ab.err
  done
done
cat gpurun_out/f_ab.jsonl
