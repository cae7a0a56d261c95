# Whole-context 1M prefill through 32 synthetic Llama-3-8B layers (paper Tab. 6/7 comparison), with and without
# 50% duo streaming heads, and whole-layer decode with every KV head resident in HBM (NEXT-1 + NEXT-4)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python tools/full_prefill.py --model > gpurun_out/fp_model.json 2> gpurun_out/fp_model.log; tail -c 400 gpurun_out/fp_model.json
timeout 600 python tools/full_prefill.py --model --duo 0.5 > gpurun_out/fp_model_duo.json 2> gpurun_out/fp_model_duo.log; tail -c 400 gpurun_out/fp_model_duo.json
timeout 900 python bench.py --model --resident-heads -1 --no-e2e > gpurun_out/b_1m_model_res.json 2> gpurun_out/b_1m_model_res.log; tail -c 600 gpurun_out/b_1m_model_res.json
