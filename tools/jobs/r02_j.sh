#!/bin/bash
# round-2 GPU job J: NEXT-4 tcgen05 GEMM (tests, vs cuBLAS), layer tests, bench contract tests, 8B-1M bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j_build.log 2>&1 || { tail -30 gpurun_out/j_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/j_gemm_tests.log 2>&1; tail -12 gpurun_out/j_gemm_tests.log
timeout 600 python tools/gemm_bench.py > gpurun_out/j_gemm_bench.json 2> gpurun_out/j_gemm_bench.err; cat gpurun_out/j_gemm_bench.err | tail -5
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_bench.py -x -q -m gpu > gpurun_out/j_layer_bench_tests.log 2>&1; tail -12 gpurun_out/j_layer_bench_tests.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err; tail -2 gpurun_out/j_bench.err
python - <<'PY'
import json
r = json.loads(open("gpurun_out/j_bench.json").read().strip().splitlines()[-1])
print(r["value"], r["config"]["timed_chunk"], r["roofline"]["achieved"], r["roofline"]["frac"], r["last_chunk"],
      r["decode"]["ms_per_token"], r["e2e"]["value"], r["parity_sample"]["ok"], r["cpu_baseline"]["value"], r["clocks"])
PY
