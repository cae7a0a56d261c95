#!/bin/bash
# round-2 GPU job AQ: the paper's Tab. 6/7 head-group sweep on HEAD (after the K/V release change), and an ncu capture
# of the CTA-pair NEXT-4 GEMM on the QKV shape
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aq_build.log 2>&1 || { tail -30 gpurun_out/aq_build.log; exit 1; }
timeout 600 ncu --set full --clock-control none -k regex:gemm_tc2_kernel -s 3 -c 1 -o gpurun_out/prof_gemm_pair_r02 \
  python tools/gemm_bench.py > gpurun_out/aq_ncu_gemm.log 2>&1; tail -1 gpurun_out/aq_ncu_gemm.log
TAB67_OUT=gpurun_out/tab67_r02b.jsonl TAB67_CTX="1024 10240 102400 409600" bash tools/tab67_sweep.sh
TAB67_OUT=gpurun_out/tab67_r02b_1m.jsonl TAB67_CTX="1048576" TAB67_G="8 -2" bash tools/tab67_sweep.sh
wc -l gpurun_out/tab67_r02b*.jsonl
