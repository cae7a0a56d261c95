#!/bin/bash
# round-2 GPU job B: softmax microbenchmark, bench contract tests (N=1 tiny, 2 ranks sharing the GPU), 8B-128K bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1 || { tail -30 gpurun_out/b_build.log; exit 1; }
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -maxrregcount=208 softmax_row.cu -o softmax_row && ./softmax_row) > gpurun_out/ubench_softmax_row.txt 2>&1; cat gpurun_out/ubench_softmax_row.txt
timeout 1500 python -m pytest tests/test_bench.py -x -q -m gpu > gpurun_out/b_tests.log 2>&1; tail -15 gpurun_out/b_tests.log
timeout 600 python bench.py --workload 8B-128K --steps 3 --warmup 3 > gpurun_out/b_bench128k.json 2> gpurun_out/b_bench128k.err; tail -3 gpurun_out/b_bench128k.err; head -c 3000 gpurun_out/b_bench128k.json
