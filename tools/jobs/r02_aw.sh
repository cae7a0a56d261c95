#!/bin/bash
# round-2 GPU job AW: the 2-rank multi-layer bench test (parity sample on)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aw_build.log 2>&1 || { tail -30 gpurun_out/aw_build.log; exit 1; }
timeout 1800 python -m pytest tests/test_bench.py -q -m gpu > gpurun_out/aw_tests.log 2>&1; echo "bench tests rc=$?"; tail -3 gpurun_out/aw_tests.log
