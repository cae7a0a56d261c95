set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python bench.py --workload tiny --duo 0.5 --duo-sink 64 --duo-window 256 > gpurun_out/b_tiny_duo.json 2> gpurun_out/b_tiny_duo.log; tail -1 gpurun_out/b_tiny_duo.json
timeout 1200 python bench.py > gpurun_out/b_1m.json 2> gpurun_out/b_1m.log; tail -c 600 gpurun_out/b_1m.json
timeout 1200 python bench.py --duo 0.5 > gpurun_out/b_1m_duo.json 2> gpurun_out/b_1m_duo.log; tail -c 600 gpurun_out/b_1m_duo.json
