#!/bin/bash
# round-2 GPU job G: where the in-step prefill time goes -- offloaded vs resident (no H2D, one launch per unit),
# slot sizes; host-link probe; resident decode bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1 || { tail -30 gpurun_out/g_build.log; exit 1; }
for rep in 1 2; do
  timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/g_probe.jsonl 2>> gpurun_out/g_probe.err
  timeout 300 python tools/prefill_probe.py --seconds 8 --resident >> gpurun_out/g_probe.jsonl 2>> gpurun_out/g_probe.err
  timeout 300 python tools/prefill_probe.py --seconds 8 --slot-tokens 262144 >> gpurun_out/g_probe.jsonl 2>> gpurun_out/g_probe.err
done
cat gpurun_out/g_probe.jsonl
timeout 300 python tools/probe_link.py --gpus 1 > gpurun_out/g_link.json 2> gpurun_out/g_link.err; cat gpurun_out/g_link.json
timeout 1200 python bench.py --resident-heads -1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench_resident.json 2> gpurun_out/g_bench_resident.err; tail -2 gpurun_out/g_bench_resident.err; python -c "
import json; r=json.loads(open('gpurun_out/g_bench_resident.json').read().strip().splitlines()[-1]); print(r['value'], r['decode'], r['roofline'])"
