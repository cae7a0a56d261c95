#!/bin/bash
# round-2 GPU job AV: the sharded decode parity fix (layer 0 re-gathered): the new multi-layer 2-rank test, the
# 8B-128K 2-rank torchrun run that exposed it, and the bench test file
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/av_build.log 2>&1 || { tail -30 gpurun_out/av_build.log; exit 1; }
timeout 1800 python -m pytest tests/test_bench.py -x -q -m gpu > gpurun_out/av_tests.log 2>&1; echo "bench tests rc=$?"; tail -3 gpurun_out/av_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --gpus 2 --steps 3 --warmup 3 --workload 8B-128K --ranks-share-gpu > gpurun_out/av_128k.json 2> gpurun_out/av_128k.err; echo "128k rc=$?"; python - <<'PY'
import json
r = json.loads(open("gpurun_out/av_128k.json").read().strip().splitlines()[-1])
print(r["n_gpus"], r["value"], r["roofline"]["frac"], r["decode"]["ms_per_token"], r["parity_sample"])
PY
