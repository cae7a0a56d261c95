#!/bin/bash
# round-2 GPU job L: re-run the fixed tests; NEXT-3 / NEXT-4 / configs[3] / configs[4] bench records
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1 || { tail -30 gpurun_out/l_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_bench.py -x -q -m gpu > gpurun_out/l_tests.log 2>&1; tail -4 gpurun_out/l_tests.log
summ() { python - "$1" <<'PY'
import json, sys
r = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], r["value"], r["config"]["workload"], r["roofline"]["achieved"], r["roofline"]["frac"], r.get("last_chunk", {}).get("tok_s"),
      r["decode"]["ms_per_token"], r.get("e2e", {}).get("value"), r.get("parity_sample", {}).get("ok"), r.get("model", {}).get("attention_share_of_prefill"))
PY
}
timeout 1500 python bench.py --steps 3 --warmup 3 --duo 0.5 > gpurun_out/l_duo.json 2> gpurun_out/l_duo.err; summ gpurun_out/l_duo.json
timeout 1500 python bench.py --steps 3 --warmup 3 --model > gpurun_out/l_model.json 2> gpurun_out/l_model.err; summ gpurun_out/l_model.json
timeout 1500 python bench.py --steps 3 --warmup 3 --workload 70B-1M --emulate-shard 0/8 > gpurun_out/l_70b.json 2> gpurun_out/l_70b.err; summ gpurun_out/l_70b.json
timeout 2400 python bench.py --steps 3 --warmup 3 --workload 8B-4M --emulate-shard 0/8 > gpurun_out/l_4m.json 2> gpurun_out/l_4m.err; summ gpurun_out/l_4m.json
