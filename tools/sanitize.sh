#!/bin/bash
# compute-sanitizer passes over small GPU parity cases (run under gpurun).  Writes gpurun_out/sanitize_*.log
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_contract.py tests/test_gpu_parity.py tests/test_gpu_duo.py tests/test_gpu_layer.py tests/test_gpu_gemm.py tests/test_gpu_layer_tp.py"
K="timing_flag_reports_copy_engine_time or default_slots_keep_one_head or tiny_config_end_to_end and P or block_and_slot_geometry and 2-64 or resident_heads_next1 or llama8b_shape_small or duo_tiny_config and P or duo_sink_window_sweep and 16-300 or duo_with_groups_and_resident and 4-3 or layer_tiny_two_layers and opts0 or test_gemm_tc and 300-640 or test_gemm_tc and 2048 or gemv_decode and 64-8 or tp_layers_match_oracle and 2-opts0"
rm -f gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 20 --error-exitcode 99 \
      python -m pytest $SEL -x -q -k "$K" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY: 0 errors' gpurun_out/sanitize_$tool.log) clean-summaries, $(grep -E '[0-9]+ passed' -o gpurun_out/sanitize_$tool.log | tail -1)" >> gpurun_out/sanitize_summary.txt
done
