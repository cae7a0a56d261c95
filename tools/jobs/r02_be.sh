#!/bin/bash
# round-2 GPU job BE: the opt-in comparison-kernel parity suite (CTA pair, one tile, mma.sync, P in shared memory)
# after their issuers moved to the warp-converged form
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/be_build.log 2>&1 || { tail -30 gpurun_out/be_build.log; exit 1; }
HI_TEST_VARIANTS=1 timeout 2400 python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/be_tests.log 2>&1; echo "variant tests rc=$?"; tail -5 gpurun_out/be_tests.log
