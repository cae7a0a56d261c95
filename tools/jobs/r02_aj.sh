#!/bin/bash
# round-2 GPU job AJ: the CTA-pair (cta_group::2, 256 x 256 tiles) NEXT-4 GEMM: GEMM + layer parity, then ours vs
# cuBLAS on the 8B projections (pair kernel = product build, single-CTA kernel = variant HI_GEMM_2CTA=0); and a
# quick prefill probe of HEAD (per-clock check after reverting the shared-memory re-reads)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aj_build.log 2>&1 || { tail -30 gpurun_out/aj_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/aj_tests_gemm.log 2>&1; echo "gemm tests rc=$?"; tail -2 gpurun_out/aj_tests_gemm.log
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_layer_tp.py -x -q > gpurun_out/aj_tests_layer.log 2>&1; echo "layer tests rc=$?"; tail -2 gpurun_out/aj_tests_layer.log
python -c "from paper_2502_12574_b200 import build as b; b.build_variant('g1', ['HI_GEMM_2CTA=0'])" > gpurun_out/aj_variants.log 2>&1 || { tail gpurun_out/aj_variants.log; exit 1; }
for rep in 1 2; do
  timeout 300 python tools/gemm_bench.py > gpurun_out/aj_gemm_pair_$rep.json 2> gpurun_out/aj_gemm_pair_$rep.err; tail -c 300 gpurun_out/aj_gemm_pair_$rep.json
  HI_LIB_VARIANT=g1 timeout 300 python tools/gemm_bench.py > gpurun_out/aj_gemm_one_$rep.json 2> gpurun_out/aj_gemm_one_$rep.err; tail -c 300 gpurun_out/aj_gemm_one_$rep.json
done
timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/aj_probe.jsonl 2>> gpurun_out/aj_probe.err; tail -1 gpurun_out/aj_probe.jsonl
