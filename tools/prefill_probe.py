"""Prefill kernel probe (not the bench): the bench's dominant launches in isolation or sustained.

One layer of the 8B shape (32 q / 8 kv heads, d = 128) at context S (default 1M), head group G (default 2 = the
bench's auto choice), chunk 18944: the history is placed untimed, then the last chunk is re-run back to back for
--seconds, so the clock settles where a long prefill step runs it (power cap).  Reports the attention kernels'
TFLOP/s from the library's HI_FLAG_TIMING events and the clocks seen.  Variants: HI_LIB_VARIANT=<name>.

    python tools/prefill_probe.py [--ctx 1048576] [--group 2] [--seconds 6] [--layers 1]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=1 << 20)
    ap.add_argument("--chunk", type=int, default=18944)
    ap.add_argument("--group", type=int, default=2)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--dist", default="U")
    ap.add_argument("--resident", action="store_true", help="every (layer, kv head) resident in HBM (no H2D)")
    ap.add_argument("--slot-tokens", type=int, default=0)
    ap.add_argument("--flags", type=lambda v: int(v, 0), default=0, help="extra hi_init flags (e.g. 0x20: CTA-pair kernel)")
    a = ap.parse_args()
    import bench
    from paper_2502_12574_b200._lib import HI_FLAG_TIMING
    from paper_2502_12574_b200.headinfer import HeadInfer
    from synth.cuda import fill_
    bench.DIST = a.dist
    L, hq, hkv, d, S, c = a.layers, 32, 8, 128, a.ctx, a.chunk
    p_last = S - c
    hi = HeadInfer(L, hq, hkv, d, S + 8, c, flags=HI_FLAG_TIMING | a.flags, head_group=a.group,
                   resident_kv_heads=-1 if a.resident else 0, slot_tokens=a.slot_tokens)
    bench.fill_history(hi, L, hkv, 0, d, p_last, torch, fill_)
    ins = [bench.gen_layer_inputs(l, p_last, c, hq, hkv, d, 0, 0, torch, fill_) for l in range(L)]
    out = torch.empty((c, hq, d), dtype=torch.bfloat16, device="cuda")

    def step():
        for l in range(L):
            hi.set_seq_len(l, p_last)
        for l in range(L):
            hi.prefill_chunk(l, *ins[l], out)

    step()
    hi.synchronize()
    st0 = hi.stats()
    steps = 0
    t0 = time.time()
    with bench.ClockSampler(torch.cuda.current_device()) as clk:
        while time.time() - t0 < a.seconds:
            step()
            steps += 1
        hi.synchronize()
    st1 = hi.stats()
    ms = st1["prefill_attn_ms"] - st0["prefill_attn_ms"]
    fl = st1["prefill_attn_flops"] - st0["prefill_attn_flops"]
    res = {"variant": os.environ.get("HI_LIB_VARIANT", "product") + (f"+0x{a.flags:x}" if a.flags else ""), "ctx": S, "group": a.group, "layers": L, "dist": a.dist,
           "resident": a.resident, "slot_tokens": hi.stats()["slot_tokens"],
           "steps": steps, "kernel_tflops": round(fl / ms / 1e9, 1), "kernel_ms_per_step": round(ms / steps, 2),
           "launches_per_step": (st1["prefill_attn_launches"] - st0["prefill_attn_launches"]) / steps,
           "clocks": clk.summary()}
    print(json.dumps(res), flush=True)
    hi.close()


if __name__ == "__main__":
    main()
