#!/bin/bash
# round-2 GPU job Q: P-in-shared-memory kernel (3-slot K/V ring, event-driven MMA issue): trap-checked smoke, parity, A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1 || { tail -30 gpurun_out/q_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('psm', ['HI_PSMEM_DEFAULT=1']); b.build_variant('psmdbg', ['HI_PSMEM_DEFAULT=1', 'HI_DEBUG_WAIT=1'])" > gpurun_out/q_variants.log 2>&1 || { tail gpurun_out/q_variants.log; exit 1; }
HI_LIB_VARIANT=psmdbg timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny_config_end_to_end" > gpurun_out/q_dbg.log 2>&1; echo "dbg rc=$?"; tail -3 gpurun_out/q_dbg.log
HI_LIB_VARIANT=psm timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py -x -q > gpurun_out/q_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/q_parity.log
for rep in 1 2; do
  for v in base psm; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/q_ab.jsonl 2>> gpurun_out/q_ab.err
  done
done
cat gpurun_out/q_ab.jsonl
timeout 600 ncu --set full --clock-control none -k regex:prefill_tcp_kernel -s 12 -c 1 -o gpurun_out/prof_psm_r02 env HI_LIB_VARIANT=psm python tools/prefill_probe.py --seconds 1 > gpurun_out/q_ncu.log 2>&1; tail -2 gpurun_out/q_ncu.log
