#!/bin/bash
# round-2 GPU job I: the driver's default bench (8B-1M) at --steps 3 and 10, ncu evidence for the round
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1 || { tail -30 gpurun_out/i_build.log; exit 1; }
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/i_bench_s3.json 2> gpurun_out/i_bench_s3.err; tail -2 gpurun_out/i_bench_s3.err
timeout 1800 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/i_bench_s10.json 2> gpurun_out/i_bench_s10.err; tail -2 gpurun_out/i_bench_s10.err
python - <<'PY'
import json
for f in ("gpurun_out/i_bench_s3.json", "gpurun_out/i_bench_s10.json"):
    try:
        r = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, r["value"], r["steps"], r["roofline"]["achieved"], r["roofline"]["frac"], r["decode"]["ms_per_token"],
              r.get("e2e", {}).get("value"), r.get("parity_sample", {}).get("ok"), r["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
# ncu: one history-block launch of the bench configuration (1M, head group 2), full set, and the launch list
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_tc_kernel -s 12 -c 1 \
  -o gpurun_out/prof_prefill_r02 python tools/prefill_probe.py --seconds 1 > gpurun_out/i_ncu_prefill.log 2>&1; tail -3 gpurun_out/i_ncu_prefill.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches_r02_probe.csv python tools/prefill_probe.py --seconds 1 > gpurun_out/i_ncu_launches.log 2>&1; tail -2 gpurun_out/i_ncu_launches.log
timeout 900 ncu --set full --clock-control none -k regex:decode_partial_kernel -s 2 -c 1 \
  -o gpurun_out/prof_decode_resident_r02 python tools/decode_probe.py 1048576 2 -1 > gpurun_out/i_ncu_decode.log 2>&1; tail -3 gpurun_out/i_ncu_decode.log
