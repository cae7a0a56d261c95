#!/bin/bash
# round-2 GPU job Z: timeline trace of the current (warp-issue, split-P) prefill kernel, and the FMA-pipe exp2
# share re-tested now that the MMA issuer no longer throttles the tensor pipe (sustained 1M probe, interleaved)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1 || { tail -30 gpurun_out/z_build.log; exit 1; }
python - > gpurun_out/z_variants.log 2>&1 <<'PY' || { tail gpurun_out/z_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('trace', ['HI_TRACE']), ('base', []), ('m01', ['HI_POLY_MASK8=0x01']), ('m11', ['HI_POLY_MASK8=0x11']),
        ('m52', ['HI_POLY_MASK8=0x52']), ('ks96', ['HI_P_SPLIT_KEYS=96'])]
with ThreadPoolExecutor(5) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
timeout 300 python tools/trace_prefill.py > gpurun_out/z_trace.txt 2>&1; tail -16 gpurun_out/z_trace.txt
for rep in 1 2 3; do
  for v in base m01 m11 m52 ks96; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/z_ab.jsonl 2>> gpurun_out/z_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/z_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
