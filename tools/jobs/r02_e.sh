#!/bin/bash
# round-2 GPU job E: prefill softmax A/B (polynomial exp2 masks) on the sustained 1M probe; cuDNN sustained ceiling
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1 || { tail -30 gpurun_out/e_build.log; exit 1; }
python - <<'PY' > gpurun_out/e_variants.log 2>&1
from paper_2502_12574_b200 import build as b
for name, defs in [("base", []), ("p52", ["HI_POLY_MASK8=0x52"]), ("p80", ["HI_POLY_MASK8=0x80"]), ("p22", ["HI_POLY_MASK8=0x22"])]:
    b.build_variant(name, defs)
PY
tail -3 gpurun_out/e_variants.log
for rep in 1 2; do
  for v in base p52 p80 p22; do
    HI_LIB_VARIANT=$v timeout 300 python tools/prefill_probe.py --seconds 8 >> gpurun_out/e_ab.jsonl 2>> gpurun_out/e_ab.err
  done
done
cat gpurun_out/e_ab.jsonl
timeout 600 python tools/ceiling_fmha.py --sustain 8 > gpurun_out/e_ceiling.json 2> gpurun_out/e_ceiling.log; grep -i "sustained\|cudnn" gpurun_out/e_ceiling.log | tail -3
