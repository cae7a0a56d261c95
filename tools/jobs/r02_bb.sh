#!/bin/bash
# round-2 GPU job BB: same-box sustained comparison on the dominant launch shape: cuDNN (torch SDPA) back to back for
# 8 s vs our kernel in the sustained 1M probe, interleaved twice
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bb_build.log 2>&1 || { tail -30 gpurun_out/bb_build.log; exit 1; }
for rep in 1 2; do
  timeout 600 python tools/ceiling_fmha.py --sustain 8 > gpurun_out/bb_ceiling_$rep.json 2> gpurun_out/bb_ceiling_$rep.err; tail -c 600 gpurun_out/bb_ceiling_$rep.json; echo
  timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/bb_probe.jsonl 2>> gpurun_out/bb_probe.err; tail -1 gpurun_out/bb_probe.jsonl
done
