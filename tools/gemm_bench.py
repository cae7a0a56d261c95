"""NEXT-4 GEMM shapes: this library's tcgen05 GEMM (hl_gemm) vs cuBLAS (torch.matmul) on the Llama-3-8B
projections at the bench chunk (18944 tokens), bf16, TFLOP/s from CUDA events (burst: 20 back-to-back launches
after warm-up).

    python tools/gemm_bench.py [--n 18944]   ->  one JSON line
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    from paper_2502_12574_b200.layer import hl_gemm
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=18944)
    a = ap.parse_args()
    H, I, d, hq, hkv = 4096, 14336, 128, 32, 8
    shapes = {"qkv": ((hq + 2 * hkv) * d, H), "o": (H, hq * d), "gate_up": (2 * I, H), "down": (H, I)}
    res = {"n": a.n}
    tot_ours = tot_cublas = flops_all = 0.0
    for name, (mo, kd) in shapes.items():
        x = torch.randn(a.n, kd, device="cuda").bfloat16()
        w = (torch.randn(mo, kd, device="cuda") / kd ** 0.5).bfloat16()
        y = torch.empty(a.n, mo, device="cuda", dtype=torch.bfloat16)
        flops = 2.0 * a.n * mo * kd
        t_ours = timed(lambda: hl_gemm(w, x, y))
        t_cub = timed(lambda: torch.matmul(x, w.T, out=y))
        res[name] = {"mo": mo, "kd": kd, "ours_tflops": round(flops / t_ours / 1e9, 1),
                     "cublas_tflops": round(flops / t_cub / 1e9, 1), "ratio": round(t_cub / t_ours, 3)}
        tot_ours += t_ours
        tot_cublas += t_cub
        flops_all += flops
        print(name, res[name], file=sys.stderr, flush=True)
    res["all"] = {"ours_tflops": round(flops_all / tot_ours / 1e9, 1), "cublas_tflops": round(flops_all / tot_cublas / 1e9, 1),
                  "ratio": round(tot_cublas / tot_ours, 3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
