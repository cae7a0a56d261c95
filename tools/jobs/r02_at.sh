#!/bin/bash
# round-2 GPU job AT: complete the Tab. 6/7 1M column (G = 4, 2, 1) on HEAD
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/at_build.log 2>&1 || { tail -30 gpurun_out/at_build.log; exit 1; }
TAB67_OUT=gpurun_out/tab67_r02b_1m_rest.jsonl TAB67_CTX="1048576" TAB67_G="4 2 1" bash tools/tab67_sweep.sh
wc -l gpurun_out/tab67_r02b_1m_rest.jsonl
