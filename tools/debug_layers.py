"""Debug probe: last-chunk prefill outputs of EVERY layer vs the oracle (relative L2 per (layer, q head)), as bench.py
runs them (history placed untimed, then one chunk through all layers back to back), with optional library flags.

    python tools/debug_layers.py [--layers 32] [--ctx 131072] [--chunk 18944] [--flags 0] [--group -1] [--rows 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--chunk", type=int, default=18944)
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
    ap.add_argument("--group", type=int, default=-1)
    ap.add_argument("--rows", type=int, default=4)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--dist", default="U")
    a = ap.parse_args()
    import bench
    import oracle
    import synth
    from paper_2502_12574_b200.headinfer import HeadInfer
    from synth.cuda import fill_
    bench.DIST = a.dist
    oracle.build()
    L, hq, hkv, d, S, c = a.layers, 32, 8, 128, a.ctx, a.chunk
    g = hq // hkv
    p_last = S - c
    hi = HeadInfer(L, hq, hkv, d, S + 8, c, flags=a.flags, head_group=a.group)
    bench.fill_history(hi, L, hkv, 0, d, p_last, torch, fill_)
    ins = [bench.gen_layer_inputs(l, p_last, c, hq, hkv, d, 0, 0, torch, fill_) for l in range(L)]
    outs = [torch.empty((c, hq, d), dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    for _ in range(a.steps):
        for l in range(L):
            hi.set_seq_len(l, p_last)
        for l in range(L):
            hi.prefill_chunk(l, *ins[l], outs[l])
    hi.synchronize()
    # host KV of the last layers vs the generator (localises a wrong history: fill / write-back vs kernel)
    for l in sorted({0, L - 3, L - 2, L - 1} & set(range(L))):
        bad = []
        for h in range(hkv):
            k, v = bench._oracle_kv(l, h, S, d, torch)
            hk, hv = hi.read_host_kv(l, h, 0, S)
            hk = hk.view(torch.int16).numpy().view(np.uint16)
            hv = hv.view(torch.int16).numpy().view(np.uint16)
            rows_bad = np.nonzero((hk != k).any(axis=1) | (hv != v).any(axis=1))[0]
            if len(rows_bad):
                bad.append((h, int(len(rows_bad)), int(rows_bad[0]), int(rows_bad[-1])))
        print(f"host KV layer {l}: {'bit-exact' if not bad else bad}", flush=True)
    toks = np.array(sorted(set([0, c // 2, c - 1] + list(np.random.default_rng(0).integers(0, c, a.rows)))))
    res = {}
    for l in range(L):
        got = outs[l][torch.tensor(toks, device="cuda")].float().cpu().numpy()
        q = synth.gen_block(bench.SEED, 0, a.dist, l, 0, hq, p_last, c, d)[toks]
        worst = 0.0
        for h in range(hkv):
            k = bench._oracle_kv(l, h, S, d, torch)
            for j in range(h * g, (h + 1) * g):
                ref = oracle.attention_rows(q[:, j], p_last + toks, *k)
                rel = float(np.linalg.norm(got[:, j] - ref) / np.linalg.norm(ref))
                worst = max(worst, rel)
                if rel > 1e-2:
                    print(f"layer {l} qhead {j}: rel {rel:.4f}; per row "
                          f"{[round(float(np.linalg.norm(got[i, j] - ref[i]) / np.linalg.norm(ref[i])), 4) for i in range(len(toks))]}",
                          flush=True)
        res[l] = round(worst, 5)
        print(f"layer {l}: worst rel-L2 {worst:.5f}", flush=True)
    print(json.dumps({"flags": a.flags, "group": a.group, "worst_per_layer": res, "rows": toks.tolist()}))
    hi.close()


if __name__ == "__main__":
    main()
