#!/bin/bash
# round-2 GPU job BA: final checkpoint of the round-2 HEAD (final-O commit first, GEMM producer tail, sharded parity fix): smoke, full -m gpu suite,
# sustained probe, default bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ba_build.log 2>&1 || { tail -30 gpurun_out/ba_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ba_smoke.log 2>&1; tail -1 gpurun_out/ba_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/ba_gpu_tests.log 2>&1; tail -3 gpurun_out/ba_gpu_tests.log
timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/ba_probe.jsonl 2>> gpurun_out/ba_probe.err; tail -1 gpurun_out/ba_probe.jsonl
timeout 1500 python bench.py > gpurun_out/ba_bench.json 2> gpurun_out/ba_bench.err; tail -1 gpurun_out/ba_bench.err
python - <<'PY'
import json
r = json.loads(open("gpurun_out/ba_bench.json").read().strip().splitlines()[-1])
print(r["value"], r["roofline"]["achieved"], r["roofline"]["frac"], r["last_chunk"]["tok_s"], r["decode"]["ms_per_token"],
      r["e2e"]["value"], r["parity_sample"]["ok"], r["cpu_baseline"]["value"], r["gpu_launches"], r["clocks"])
PY
