"""Whole-context prefill on one B200: every chunk from position 0 to S, through the attention path alone or
through 32 synthetic Llama-3-8B decoder layers (--model, NEXT-4), then a few decode tokens -- the quantity
the paper's Tab. 6/7 report for HeadInfer on an RTX 4090 (1M prefill 2054 s, decode 6.51 s/token, P:L582,
P:L602).  bench.py times the LAST chunks (the most expensive ones); this tool times all of them.

    python tools/full_prefill.py [--model] [--duo 0.5] [--context 1048576] [--resident-heads R]
    python tools/full_prefill.py --context 4194304 --emulate-shard 0/8           # configs[3]: rank 0 of 8
    python tools/full_prefill.py --shape 70B --chunk 9472 --emulate-shard 0/8    # configs[4]: rank 0 of 8

Each chunk's inputs are generated on the GPU outside its timed region (CUDA events around the layer calls
only); prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=1 << 20)
    ap.add_argument("--chunk", type=int, default=18944)
    ap.add_argument("--decode", type=int, default=4)
    ap.add_argument("--model", action="store_true")
    ap.add_argument("--duo", type=float, default=0.0)
    ap.add_argument("--resident-heads", type=int, default=0)
    ap.add_argument("--head-group", type=int, default=-1, help="kv heads per offload unit (NEXT-2; -1 auto, -2 paper)")
    ap.add_argument("--shape", choices=["8B", "70B"], default="8B", help="Llama-3-8B (32 L, 32 q / 8 kv) or 70B "
                    "(80 L, 64 q / 8 kv) attention shapes")
    ap.add_argument("--emulate-shard", type=lambda x: tuple(int(v) for v in x.split("/")), default=None,
                    metavar="R/W", help="rank R's head shard of a W-GPU job, alone on this GPU (as bench.py)")
    args = ap.parse_args()
    import torch

    import bench
    import synth
    from paper_2502_12574_b200.headinfer import HeadInfer
    from synth.cuda import fill_, fill_matrix_, gen_layer_weights_cuda

    L, hq, hkv, d = (32, 32, 8, 128) if args.shape == "8B" else (80, 64, 8, 128)
    S, c = args.context, args.chunk
    hr, hw = args.emulate_shard or (0, 1)
    if args.model and (hw != 1 or args.shape != "8B"):
        raise SystemExit("--model runs the 8B shape at world 1")
    hq_loc, hkv_loc = hq // hw, hkv // hw
    q0h, kv0h = hr * hq_loc, hr * hkv_loc
    opts = dict(head_group=args.head_group, resident_kv_heads=args.resident_heads)
    if args.duo > 0:
        opts.update(streaming_heads=synth.streaming_labels(bench.SEED, L, hkv, args.duo).tolist(), duo_sink=64,
                    duo_window=256)
    t0 = time.time()
    hi = HeadInfer(L, hq, hkv, d, S + args.decode, c, hr, hw, **opts)
    init_s = time.time() - t0
    model = weights = None
    if args.model:
        from paper_2502_12574_b200.layer import HeadInferLayer
        H, I = bench.MODEL_DIMS
        model = HeadInferLayer(hi, H, I, bench.MODEL_ROPE_THETA, bench.MODEL_RMS_EPS)
        weights = [gen_layer_weights_cuda(bench.SEED, l, H, I, hq, hkv, d) for l in range(L)]
    stream = torch.cuda.current_stream()
    out = torch.empty((c, hq_loc, d), dtype=torch.bfloat16, device="cuda")

    def inputs(pos, n):
        if model is not None:
            return fill_matrix_(torch.empty((n, bench.MODEL_DIMS[0]), dtype=torch.bfloat16, device="cuda"), bench.SEED,
                                synth.TENSOR_X, 0, row0=pos)
        return [bench.gen_layer_inputs(l, pos, n, hq_loc, hkv_loc, d, q0h, kv0h, torch, fill_) for l in range(L)]

    def step(x, n):
        for l in range(L):
            if model is not None:
                model.prefill_chunk(l, weights[l], x)
            else:
                hi.prefill_chunk(l, *x[l], out[:n])

    chunk_ms = []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for pos in range(0, S, c):
        n = min(c, S - pos)
        x = inputs(pos, n)
        ev[0].record(stream)
        step(x, n)
        hi.synchronize()   # the chunk's write-back has landed too
        ev[1].record(stream)
        torch.cuda.synchronize()
        chunk_ms.append(ev[0].elapsed_time(ev[1]))
        del x
        if len(chunk_ms) % 8 == 0:
            print(f"chunk {len(chunk_ms)} at {pos}: {chunk_ms[-1]:.0f} ms", file=sys.stderr, flush=True)
    dec_ms = []
    for t in range(args.decode):
        x = inputs(S + t, 1)
        ev[0].record(stream)
        for l in range(L):
            if model is not None:
                model.decode(l, weights[l], x[0])
            else:
                q, k, v = x[l]
                hi.decode(l, q[0], k[0], v[0], out[0])
        hi.synchronize()
        ev[1].record(stream)
        torch.cuda.synchronize()
        dec_ms.append(ev[0].elapsed_time(ev[1]))
    st = hi.stats()
    total_s = sum(chunk_ms) / 1e3
    res = {"tool": "full_prefill", "path": "decoder layers" if model is not None else "attention",
           "context": S, "chunk": c, "chunks": len(chunk_ms), "shape": args.shape,
           "shard": ({"rank": hr, "world": hw, "note": "one rank's heads alone on one GPU; every rank of the W-GPU "
                      "job does the same work on its own heads; the output all-gather is not timed"}
                     if hw > 1 else None), "prefill_s": round(total_s, 4),
           "prefill_tok_s": round(S / total_s, 1), "first_chunk_ms": round(chunk_ms[0], 1),
           "last_chunk_ms": round(chunk_ms[-1], 1),
           "decode_ms_per_token": round(sum(dec_ms[1:]) / max(1, len(dec_ms) - 1), 2) if dec_ms else None,
           "head_group": st["head_group"], "resident_kv_heads": st["resident_kv_heads"],
           "streaming_kv_heads": st["streaming_kv_heads"], "init_s": round(init_s, 1),
           "paper_rtx4090": {"prefill_1m_s": 2054, "decode_1m_s_per_token": 6.51, "prefill_4m_s": 27114,
                             "decode_4m_s_per_token": 27.2, "cite": "Tab. 6/7, P:L582-583, P:L602-603 (Llama-3-8B)"},
           "chunk_ms": [round(x, 1) for x in chunk_ms]}
    if model is not None:
        model.close()
    hi.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
