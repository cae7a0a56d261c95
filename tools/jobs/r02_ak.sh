#!/bin/bash
# round-2 GPU job AK: records on HEAD (K/V release + CTA-pair GEMM): full -m gpu suite, NEXT-4 whole-model bench,
# NEXT-3 duo 50 %, configs[4] 70B-1M and configs[3] 8B-4M as rank 0 of an 8-GPU head shard
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
r = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], r["value"], r["config"]["workload"], r["roofline"]["achieved"], r["roofline"]["frac"], r.get("last_chunk", {}).get("tok_s"),
      r["decode"]["ms_per_token"], r.get("e2e", {}).get("value"), r.get("parity_sample", {}).get("ok"), r.get("model", {}).get("attention_share_of_prefill"), r["clocks"]["sm_mhz"])
PY
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ak_build.log 2>&1 || { tail -30 gpurun_out/ak_build.log; exit 1; }
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/ak_gpu_tests.log 2>&1; tail -3 gpurun_out/ak_gpu_tests.log
timeout 1500 python bench.py --steps 3 --warmup 3 --model > gpurun_out/ak_model.json 2> gpurun_out/ak_model.err; summ gpurun_out/ak_model.json
timeout 1500 python bench.py --steps 3 --warmup 3 --duo 0.5 > gpurun_out/ak_duo.json 2> gpurun_out/ak_duo.err; summ gpurun_out/ak_duo.json
timeout 1500 python bench.py --steps 3 --warmup 3 --workload 70B-1M --emulate-shard 0/8 > gpurun_out/ak_70b.json 2> gpurun_out/ak_70b.err; summ gpurun_out/ak_70b.json
timeout 2400 python bench.py --steps 3 --warmup 3 --workload 8B-4M --emulate-shard 0/8 > gpurun_out/ak_4m.json 2> gpurun_out/ak_4m.err; summ gpurun_out/ak_4m.json
