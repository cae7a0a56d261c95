#!/bin/bash
# round-2 GPU job A: build, sticky + parity smoke tests, library-FMHA ceiling diagnostic, quick perf probe
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/a_build.log 2>&1 || { tail -30 gpurun_out/a_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_sticky.py tests/test_gpu_contract.py -x -q > gpurun_out/a_tests.log 2>&1; tail -5 gpurun_out/a_tests.log
export FLASHINFER_CUDA_ARCH_LIST=10.0a
timeout 1200 python tools/ceiling_fmha.py > gpurun_out/ceiling_r02.json 2> gpurun_out/ceiling_r02.log; tail -8 gpurun_out/ceiling_r02.log
HI_QP_GROUP=2 timeout 600 python tools/quick_perf.py 1048576 1 18944 > gpurun_out/qp_r02.txt 2>&1; tail -8 gpurun_out/qp_r02.txt
