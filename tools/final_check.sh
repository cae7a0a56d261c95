# round-end check on one B200: GPU test tier, smoke, default bench (outputs under gpurun_out/)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout ${HI_TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -p no:cacheprovider ${HI_TEST_ARGS:-} > gpurun_out/r1_final_gputests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r1_final_gputests.log
if [ -z "${HI_SKIP_BENCH:-}" ]; then
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1_final_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r1_final_smoke.log
timeout 900 python bench.py > gpurun_out/r1_final_bench.json 2> gpurun_out/r1_final_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r1_final_bench.json
fi
