#!/bin/bash
# round-2 GPU job AL: with the MMA side fixed (warp issue + K/V release), re-test the S(j+1)_lo-early schedule
# (HI_SPLIT_S=1: P in the upper 64 S columns, QK^T of the next tile's first 64 keys issued as soon as S(j) is in
# registers) and the unsplit P release (HI_SPLIT_S=0) against the product schedule; plus the new GEMM test
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/al_build.log 2>&1 || { tail -30 gpurun_out/al_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/al_tests_gemm.log 2>&1; echo "gemm tests rc=$?"; tail -2 gpurun_out/al_tests_gemm.log
python - > gpurun_out/al_variants.log 2>&1 <<'PY' || { tail gpurun_out/al_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('base', []), ('s1', ['HI_SPLIT_S=1']), ('s0', ['HI_SPLIT_S=0'])]
with ThreadPoolExecutor(3) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
for rep in 1 2 3; do
  for v in base s1 s0; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/al_ab.jsonl 2>> gpurun_out/al_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/al_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r.get('dist', ''), r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
