#!/bin/bash
# round-2 GPU job M: bench after the per-step timing + duo window restore; smoke
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1 || { tail -30 gpurun_out/m_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; tail -2 gpurun_out/m_smoke.log
timeout 900 python -m pytest tests/test_bench.py -x -q -m gpu > gpurun_out/m_tests.log 2>&1; tail -3 gpurun_out/m_tests.log
summ() { python - "$1" <<'PY'
import json, sys
r = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], r["value"], r["config"]["workload"], r["roofline"]["achieved"], r["roofline"]["frac"], r.get("last_chunk", {}).get("tok_s"),
      r["decode"]["ms_per_token"], r.get("e2e", {}).get("value"), r.get("parity_sample", {}).get("ok"), r["prefill_step_ms"])
PY
}
timeout 1500 python bench.py --steps 3 --warmup 3 --duo 0.5 > gpurun_out/m_duo.json 2> gpurun_out/m_duo.err; summ gpurun_out/m_duo.json
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; summ gpurun_out/m_bench.json
