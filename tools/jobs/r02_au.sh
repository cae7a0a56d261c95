#!/bin/bash
# round-2 GPU job AU: the driver's torchrun launch (not bench's self-launch) on one GPU with the ranks sharing it:
# ours arm and reference arm at N = 2, tiny and 8B-128K
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/au_build.log 2>&1 || { tail -30 gpurun_out/au_build.log; exit 1; }
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench.py --gpus 2 --steps 3 --warmup 3 --workload tiny --ranks-share-gpu > gpurun_out/au_tiny.json 2> gpurun_out/au_tiny.err; echo "tiny rc=$?"; tail -c 400 gpurun_out/au_tiny.json; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --gpus 2 --steps 3 --warmup 3 --workload 8B-128K --ranks-share-gpu > gpurun_out/au_128k.json 2> gpurun_out/au_128k.err; echo "128k rc=$?"; python - <<'PY'
import json
r = json.loads(open("gpurun_out/au_128k.json").read().strip().splitlines()[-1])
print(r["n_gpus"], r["value"], r["roofline"]["frac"], r["decode"]["ms_per_token"], r.get("sharded_parity", r.get("parity_sample", {})).get("ok") if isinstance(r.get("sharded_parity", r.get("parity_sample")), dict) else r.get("sharded_parity"), r.get("comm_nranks_ok"))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 --workload tiny > gpurun_out/au_ref.json 2> gpurun_out/au_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/au_ref.json; echo
