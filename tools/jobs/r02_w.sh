#!/bin/bash
# round-2 GPU job W: warp-issue default (prefill + GEMM): parity, GEMM vs cuBLAS, probe, default bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1 || { tail -30 gpurun_out/w_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_duo.py tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_layer_tp.py tests/test_gpu_fullsize.py -x -q > gpurun_out/w_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/w_tests.log
timeout 600 python tools/gemm_bench.py > gpurun_out/w_gemm.json 2> gpurun_out/w_gemm.err; tail -5 gpurun_out/w_gemm.err
timeout 300 python tools/prefill_probe.py --seconds 8 > gpurun_out/w_probe.json 2>> gpurun_out/w_probe.err; cat gpurun_out/w_probe.json
timeout 1500 python bench.py > gpurun_out/w_bench.json 2> gpurun_out/w_bench.err; tail -1 gpurun_out/w_bench.err
python - <<'PY'
import json
r = json.loads(open("gpurun_out/w_bench.json").read().strip().splitlines()[-1])
print(r["value"], r["roofline"]["achieved"], r["roofline"]["frac"], r["last_chunk"]["tok_s"], r["decode"]["ms_per_token"],
      r["e2e"]["value"], r["parity_sample"]["ok"], r["clocks"])
PY
