#!/bin/bash
# round-2 GPU job AA: (1) parity of the mask-path change (row token re-read from shared memory); (2) trace with the
# TMEM-load completion stamp; (3) pipeline ceiling without the softmax math (fake) and the speculative first half,
# with the warp-converged issue; (4) launch list of the bench's own command (our kernels only)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aa_build.log 2>&1 || { tail -30 gpurun_out/aa_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py tests/test_gpu_hazards.py -x -q > gpurun_out/aa_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/aa_tests.log
python - > gpurun_out/aa_variants.log 2>&1 <<'PY' || { tail gpurun_out/aa_variants.log; exit 1; }
from concurrent.futures import ThreadPoolExecutor
from paper_2502_12574_b200 import build as b
jobs = [('trace', ['HI_TRACE']), ('base', []), ('fake', ['HI_FAKE_SOFTMAX']), ('spec', ['HI_SPEC_SPLIT=1'])]
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda j: b.build_variant(*j), jobs))
PY
timeout 300 python tools/trace_prefill.py > gpurun_out/aa_trace.txt 2>&1; tail -16 gpurun_out/aa_trace.txt
for rep in 1 2; do
  for v in base fake spec; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/aa_ab.jsonl 2>> gpurun_out/aa_ab.err
  done
done
python -c "
import json
for l in open('gpurun_out/aa_ab.jsonl'):
    r = json.loads(l); print(r['variant'], r['kernel_tflops'], r['clocks']['sm_mhz'], round(r['kernel_tflops'] / r['clocks']['sm_mhz'] * 1000, 1))"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill_tc|pack_kv|decode_|hl_|gemm" -c 2200 --csv \
  --log-file gpurun_out/launches_r02_bench.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/aa_ncu_launches.log 2>&1; tail -2 gpurun_out/aa_ncu_launches.log
python tools/launch_summary.py gpurun_out/launches_r02_bench.csv gpurun_out/launches_r02_bench.txt; cat gpurun_out/launches_r02_bench.txt
