# ncu launch list of the NEXT-4 layer's own kernels (and the small path kernels) inside a 128K --model bench:
# per-launch duration and DRAM bytes -> HBM roofline fraction per kernel (tools/ncu_summary.py style)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 ncu --clock-control none -k regex:"rmsnorm|rope_split|swiglu|pack_kv|duo_append|decode_combine" -c 40 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/ncu_layer.csv \
  python bench.py --workload 8B-128K --model --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_layer_bench.log 2>&1
tail -3 gpurun_out/ncu_layer_bench.log; wc -l gpurun_out/ncu_layer.csv
