#!/bin/bash
# The paper's Tab. 6/7 (prefill latency in s, decode s/token, Llama-3-8B, per head-group granularity,
# P:L568-606) on one B200: whole-context prefill + 4 decode tokens through the attention path for
# G kv heads per offload unit in {8 (one unit per layer), 4, 2, 1 (head-wise)} and the paper's adaptive
# schedule (-2).  Writes gpurun_out/tab67.jsonl (one JSON line per run).
cd "$(dirname "$0")/.."
OUT=${TAB67_OUT:-gpurun_out/tab67.jsonl}; rm -f $OUT
for ctx in ${TAB67_CTX:-1024 10240 102400 409600 1048576}; do
  for G in ${TAB67_G:-8 4 2 1 -2}; do
    timeout 900 python tools/full_prefill.py --context $ctx --head-group $G --decode 4 2>/dev/null \
      | grep '^{' | python -c "import json,sys; r=json.loads(sys.stdin.read()); r.pop('chunk_ms'); r['head_group_arg']=$G; print(json.dumps(r))" \
      >> $OUT
  done
done
