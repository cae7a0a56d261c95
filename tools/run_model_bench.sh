# NEXT-4 bench runs on one B200: tiny smoke of both modes, then the 1M whole-layer run
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python bench.py --workload tiny > gpurun_out/b_tiny.json 2> gpurun_out/b_tiny.log; tail -c 300 gpurun_out/b_tiny.json
timeout 300 python bench.py --workload tiny --model > gpurun_out/b_tiny_model.json 2> gpurun_out/b_tiny_model.log; tail -c 300 gpurun_out/b_tiny_model.json; tail -3 gpurun_out/b_tiny_model.log
timeout 1500 python bench.py --model > gpurun_out/b_1m_model.json 2> gpurun_out/b_1m_model.log; tail -c 900 gpurun_out/b_1m_model.json; tail -3 gpurun_out/b_1m_model.log
