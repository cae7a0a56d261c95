#!/bin/bash
# round-2 GPU job AG: checkpoint of HEAD (separate K/V release) -- smoke, full -m gpu suite, default bench, whole 1M
# prefill, ncu capture of the dominant launch, compute-sanitizer passes
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ag_build.log 2>&1 || { tail -30 gpurun_out/ag_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ag_smoke.log 2>&1; tail -1 gpurun_out/ag_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/ag_gpu_tests.log 2>&1; tail -3 gpurun_out/ag_gpu_tests.log
timeout 1500 python bench.py > gpurun_out/ag_bench.json 2> gpurun_out/ag_bench.err; tail -1 gpurun_out/ag_bench.err
python - <<'PY'
import json
r = json.loads(open("gpurun_out/ag_bench.json").read().strip().splitlines()[-1])
print(r["value"], r["roofline"]["achieved"], r["roofline"]["frac"], r["last_chunk"]["tok_s"], r["decode"]["ms_per_token"],
      r["e2e"]["value"], r["parity_sample"]["ok"], r["cpu_baseline"]["value"], r["gpu_launches"], r["clocks"])
PY
timeout 900 python tools/full_prefill.py > gpurun_out/ag_full_prefill.json 2> gpurun_out/ag_full_prefill.log; tail -c 300 gpurun_out/ag_full_prefill.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 12 -c 1 \
  -o gpurun_out/prof_prefill_r02ag python tools/prefill_probe.py --seconds 1 > gpurun_out/ag_ncu_prefill.log 2>&1; tail -1 gpurun_out/ag_ncu_prefill.log
bash tools/sanitize.sh; cat gpurun_out/sanitize_summary.txt
