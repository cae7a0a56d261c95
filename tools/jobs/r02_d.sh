#!/bin/bash
# round-2 GPU job D: per-layer parity + host-KV probe after the write_host_kv ordering fix; resident decode
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1 || { tail -30 gpurun_out/d_build.log; exit 1; }
timeout 600 python tools/debug_layers.py --layers 32 > gpurun_out/d_dbg_plain.txt 2>&1; grep -v "qhead" gpurun_out/d_dbg_plain.txt | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or tiny or group" > gpurun_out/d_tests.log 2>&1; tail -5 gpurun_out/d_tests.log
