#!/bin/bash
# round-2 GPU job O: bench --model over 2 ranks sharing the GPU (TP + head sharding, gloo); Tab. 6/7 sweep on HEAD
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/o_build.log 2>&1 || { tail -30 gpurun_out/o_build.log; exit 1; }
timeout 900 python bench.py --workload 8B-128K --model --steps 2 --warmup 3 --gpus 2 --ranks-share-gpu --no-cpu-baseline > gpurun_out/o_tp2.json 2> gpurun_out/o_tp2.err; grep -v "NCCL INFO" gpurun_out/o_tp2.err | tail -3; head -c 400 gpurun_out/o_tp2.json; echo
TAB67_OUT=gpurun_out/tab67_r02.jsonl TAB67_CTX="1024 10240 102400 409600" bash tools/tab67_sweep.sh
TAB67_OUT=gpurun_out/tab67_r02_1m.jsonl TAB67_CTX="1048576" TAB67_G="8 -2" bash tools/tab67_sweep.sh
wc -l gpurun_out/tab67_r02*.jsonl
