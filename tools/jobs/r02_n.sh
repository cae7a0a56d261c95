#!/bin/bash
# round-2 GPU job N: NEXT-4 tensor parallelism (emulated ranks vs the oracle; bench --model over 2 ranks sharing the
# GPU), GEMM/layer regressions, 1M --model bench with the phase split at W = 1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1 || { tail -30 gpurun_out/n_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_layer_tp.py tests/test_gpu_layer.py tests/test_gpu_gemm.py -x -q > gpurun_out/n_tests.log 2>&1; tail -8 gpurun_out/n_tests.log
timeout 900 python bench.py --workload 8B-128K --model --steps 2 --warmup 3 --gpus 2 --ranks-share-gpu --no-cpu-baseline > gpurun_out/n_tp2.json 2> gpurun_out/n_tp2.err; tail -3 gpurun_out/n_tp2.err; head -c 600 gpurun_out/n_tp2.json
