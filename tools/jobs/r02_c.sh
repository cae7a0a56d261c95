#!/bin/bash
# round-2 GPU job C: per-layer parity probe (race hunt), plain and serialized
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1 || { tail -30 gpurun_out/c_build.log; exit 1; }
timeout 600 python tools/debug_layers.py --layers 32 > gpurun_out/c_dbg_plain.txt 2>&1; tail -40 gpurun_out/c_dbg_plain.txt
timeout 600 python tools/debug_layers.py --layers 32 --flags 0x4 > gpurun_out/c_dbg_serial.txt 2>&1; tail -5 gpurun_out/c_dbg_serial.txt
timeout 600 python tools/debug_layers.py --layers 4 --group 1 > gpurun_out/c_dbg_g1.txt 2>&1; tail -8 gpurun_out/c_dbg_g1.txt
