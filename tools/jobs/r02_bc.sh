#!/bin/bash
# round-2 GPU job BC: ncu --set full of the cuDNN attention kernel on the dominant launch shape (diagnostic: its pipe
# utilisation, issue, registers, CTA shape next to ours; library code, not on our path)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bc_build.log 2>&1 || { tail -30 gpurun_out/bc_build.log; exit 1; }
timeout 900 ncu --set full --clock-control none -k regex:"cudnn|sm100|fmha|attention|flash" -s 2 -c 1 -o gpurun_out/prof_cudnn_fmha_r02 \
  python tools/ceiling_fmha.py --reps 3 > gpurun_out/bc_ncu.log 2>&1; tail -3 gpurun_out/bc_ncu.log
ncu -i gpurun_out/prof_cudnn_fmha_r02.ncu-rep --page raw --csv > gpurun_out/bc_raw.csv 2>/dev/null; head -c 300 gpurun_out/bc_raw.csv
