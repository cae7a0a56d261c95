#!/bin/bash
# round-2 GPU job AX: CTA-pair GEMM with the producer tail (each CTA waits for the last multicast commits before
# exiting): GEMM / layer / TP parity and the GEMM bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ax_build.log 2>&1 || { tail -30 gpurun_out/ax_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_layer_tp.py -x -q > gpurun_out/ax_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ax_tests.log
timeout 300 python tools/gemm_bench.py > gpurun_out/ax_gemm.json 2> gpurun_out/ax_gemm.err; tail -c 200 gpurun_out/ax_gemm.json
