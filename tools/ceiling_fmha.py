"""Ceiling diagnostic (not a target, not on the product path): time library sm_100 attention kernels on
the exact shape of the bench's dominant prefill launch and report TFLOP/s next to ours.

Shape (8B-1M bench, head group 2, one-head staging ring): 18944 queries x 8 q heads (2 kv heads, g = 4),
131072 keys of history, d = 128, bf16, non-causal (a history block).  FLOPs = 4*d*n*nk*Hq.

    python tools/ceiling_fmha.py [--reps 10]

Libraries tried (each optional): torch SDPA on cuDNN, flashinfer's CUTLASS sm100a FMHA (fmha_varlen, JIT
compiled on first use), flashinfer's cute-dsl ragged prefill.  Ours: hi_prefill_chunk is not used here; the
same launch is timed through the library's HI_FLAG_TIMING counters by tools/quick_perf.py.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def sustained(fn, seconds, flops):
    """Back-to-back launches for `seconds` (power-capped regime, like a long prefill step), clocks sampled."""
    from bench import ClockSampler
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        n, t = 0, 0.0
        e0.record()
        while t < seconds * 1e3:
            for _ in range(20):
                fn()
            n += 20
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
    return {"ms": round(t / n, 3), "tflops": round(flops / (t / n) / 1e9, 1), "launches": n, "clocks": clk.summary()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sustain", type=float, default=0.0, help="also time cuDNN back to back for this many seconds")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--n", type=int, default=18944)
    ap.add_argument("--nk", type=int, default=131072)
    ap.add_argument("--hq", type=int, default=8)
    ap.add_argument("--hkv", type=int, default=2)
    a = ap.parse_args()
    n, nk, hq, hkv, d = a.n, a.nk, a.hq, a.hkv, 128
    flops = 4.0 * d * n * nk * hq
    torch.manual_seed(0)
    q = (torch.rand(n, hq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(nk, hkv, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(nk, hkv, d, device="cuda") * 2 - 1).bfloat16()
    res = {"shape": {"n": n, "nk": nk, "hq": hq, "hkv": hkv, "d": d}, "flops": flops}

    def report(name, ms):
        res[name] = {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1)}
        print(name, res[name], file=sys.stderr, flush=True)

    # torch SDPA, cuDNN backend (heads expanded: GQA -> MHA view)
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel
        qb = q.transpose(0, 1).unsqueeze(0)
        kb = k.repeat_interleave(hq // hkv, dim=1).transpose(0, 1).unsqueeze(0).contiguous()
        vb = v.repeat_interleave(hq // hkv, dim=1).transpose(0, 1).unsqueeze(0).contiguous()
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            fn = lambda: torch.nn.functional.scaled_dot_product_attention(qb, kb, vb)  # noqa: E731
            report("torch_sdpa_cudnn", timeit(fn, a.reps))
            if a.sustain > 0:
                res["torch_sdpa_cudnn_sustained"] = sustained(fn, a.sustain, flops)
                print("cudnn sustained", res["torch_sdpa_cudnn_sustained"], file=sys.stderr, flush=True)
        del kb, vb
    except Exception as e:  # noqa: BLE001
        res["torch_sdpa_cudnn"] = {"error": str(e)[:200]}
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel
        qb = q.transpose(0, 1).unsqueeze(0)
        kb = k.transpose(0, 1).unsqueeze(0)
        vb = v.transpose(0, 1).unsqueeze(0)
        with sdpa_kernel(SDPBackend.FLASH_ATTENTION):
            report("torch_sdpa_flash", timeit(lambda: torch.nn.functional.scaled_dot_product_attention(
                qb, kb, vb, enable_gqa=True), a.reps))
    except Exception as e:  # noqa: BLE001
        res["torch_sdpa_flash"] = {"error": str(e)[:200]}
    # flashinfer CUTLASS sm100a FMHA
    try:
        import flashinfer.prefill as fp
        qo = torch.tensor([0, n], dtype=torch.int32, device="cuda")
        kvo = torch.tensor([0, nk], dtype=torch.int32, device="cuda")
        out = torch.empty(n + 128, hq, d, dtype=torch.bfloat16, device="cuda")
        report("flashinfer_cutlass_fmha", timeit(lambda: fp.fmha_varlen(q, k, v, qo, kvo, max_qo_len=n, out=out), a.reps))
    except Exception as e:  # noqa: BLE001
        res["flashinfer_cutlass_fmha"] = {"error": str(e)[:300]}
    # flashinfer cute-dsl ragged prefill
    try:
        import flashinfer
        ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend="cute-dsl")
        qo = torch.tensor([0, n], dtype=torch.int32, device="cuda")
        kvo = torch.tensor([0, nk], dtype=torch.int32, device="cuda")
        w.plan(qo, kvo, hq, hkv, d, causal=False, q_data_type=torch.bfloat16)
        report("flashinfer_cute_dsl", timeit(lambda: w.run(q, k, v), a.reps))
    except Exception as e:  # noqa: BLE001
        res["flashinfer_cute_dsl"] = {"error": str(e)[:300]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
