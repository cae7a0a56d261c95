#!/bin/bash
# round-2 GPU job P: P-in-shared-memory prefill kernel (k_prefill_tcp.cu): deadlock-checked smoke, parity, A/B
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1 || { tail -30 gpurun_out/p_build.log; exit 1; }
python -c "
from paper_2502_12574_b200 import build as b
b.build_variant('base', []); b.build_variant('psm', ['HI_PSMEM_DEFAULT=1']); b.build_variant('psmdbg', ['HI_PSMEM_DEFAULT=1', 'HI_DEBUG_WAIT=1'])" > gpurun_out/p_variants.log 2>&1 || { tail gpurun_out/p_variants.log; exit 1; }
HI_LIB_VARIANT=psmdbg timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny_config_end_to_end" > gpurun_out/p_dbg.log 2>&1; echo "dbg rc=$?"; tail -15 gpurun_out/p_dbg.log
HI_LIB_VARIANT=psm timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py -x -q > gpurun_out/p_parity.log 2>&1; echo "parity rc=$?"; tail -5 gpurun_out/p_parity.log
for rep in 1 2; do
  for v in base psm; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/p_ab.jsonl 2>> gpurun_out/p_ab.err
  done
done
cat gpurun_out/p_ab.jsonl
