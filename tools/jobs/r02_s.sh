#!/bin/bash
# round-2 GPU job S: checkpoint -- full -m gpu suite, smoke, default bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1 || { tail -30 gpurun_out/s_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1; tail -1 gpurun_out/s_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/s_gpu_tests.log 2>&1; tail -4 gpurun_out/s_gpu_tests.log
timeout 1500 python bench.py > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err; tail -1 gpurun_out/s_bench.err
python - <<'PY'
import json
r = json.loads(open("gpurun_out/s_bench.json").read().strip().splitlines()[-1])
print(r["value"], r["roofline"]["achieved"], r["roofline"]["frac"], r["last_chunk"]["tok_s"], r["decode"]["ms_per_token"],
      r["e2e"]["value"], r["parity_sample"]["ok"], r["cpu_baseline"]["value"], r["gpu_launches"], r["clocks"])
PY
