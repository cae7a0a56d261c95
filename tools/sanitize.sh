#!/bin/bash
# compute-sanitizer passes over small GPU parity cases (run under gpurun).  Writes gpurun_out/sanitize_*.log
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_parity.py::test_tiny_config_end_to_end tests/test_gpu_parity.py::test_block_and_slot_geometry"
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 --error-exitcode 99 \
      python -m pytest $SEL -x -q -k "P or S or 2-64" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
