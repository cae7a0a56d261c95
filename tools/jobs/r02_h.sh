#!/bin/bash
# round-2 GPU job H: resident-decode wave sizing A/B (32 layers at 1M, all resident), then the full -m gpu suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1 || { tail -30 gpurun_out/h_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
for w in (1, 2, 3, 4): b.build_variant(f'dw{w}', [f'HI_DECODE_WAVES={w}'])" > gpurun_out/h_variants.log 2>&1 || { tail gpurun_out/h_variants.log; exit 1; }
for rep in 1 2; do
  for w in 1 2 3 4; do
    echo "dw$w rep$rep $(HI_LIB_VARIANT=dw$w timeout 600 python tools/decode_probe.py 1048576 32 -1 2>&1 | tail -1)" >> gpurun_out/h_decode_ab.txt
  done
done
cat gpurun_out/h_decode_ab.txt
timeout 3000 python -m pytest tests -x -q -m gpu > gpurun_out/h_gpu_tests.log 2>&1; tail -15 gpurun_out/h_gpu_tests.log
