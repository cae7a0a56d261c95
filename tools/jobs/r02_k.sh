#!/bin/bash
# round-2 GPU job K: GEMM + bench contract tests after fixes; whole 1M prefill (linearity check of the headline)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1 || { tail -30 gpurun_out/k_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py -x -q > gpurun_out/k_gemm_tests.log 2>&1; tail -6 gpurun_out/k_gemm_tests.log
timeout 900 python -m pytest tests/test_bench.py -x -q -m gpu > gpurun_out/k_bench_tests.log 2>&1; tail -6 gpurun_out/k_bench_tests.log
timeout 1200 python tools/full_prefill.py > gpurun_out/k_full_prefill.json 2> gpurun_out/k_full_prefill.err; tail -3 gpurun_out/k_full_prefill.err; tail -c 1500 gpurun_out/k_full_prefill.json
