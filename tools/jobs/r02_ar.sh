#!/bin/bash
# round-2 GPU job AR: final checkpoint of HEAD -- smoke, full -m gpu suite, default bench, ncu capture of the
# dominant prefill launch
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ar_build.log 2>&1 || { tail -30 gpurun_out/ar_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ar_smoke.log 2>&1; tail -1 gpurun_out/ar_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/ar_gpu_tests.log 2>&1; tail -3 gpurun_out/ar_gpu_tests.log
timeout 1500 python bench.py > gpurun_out/ar_bench.json 2> gpurun_out/ar_bench.err; tail -1 gpurun_out/ar_bench.err
python - <<'PY'
import json
r = json.loads(open("gpurun_out/ar_bench.json").read().strip().splitlines()[-1])
print(r["value"], r["roofline"]["achieved"], r["roofline"]["frac"], r["last_chunk"]["tok_s"], r["decode"]["ms_per_token"],
      r["e2e"]["value"], r["parity_sample"]["ok"], r["cpu_baseline"]["value"], r["gpu_launches"], r["clocks"])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 12 -c 1 \
  -o gpurun_out/prof_prefill_r02ar python tools/prefill_probe.py --seconds 1 > gpurun_out/ar_ncu_prefill.log 2>&1; tail -1 gpurun_out/ar_ncu_prefill.log
