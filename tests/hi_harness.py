"""Shared driver for GPU parity tests: run a prefill/decode sequence through the C ABI
(paper_2502_12574_b200.headinfer) on seeded synth inputs, and the fp64 oracle on the same
inputs regenerated on the CPU.  The two share only synth/ (no method arithmetic)."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

import synth
from synth.cuda import fill_

TOL_MAX_ABS = 2e-2   # north_star: max-abs 2e-2, mean-abs 2e-3 (fp32 accumulate, bf16 out)
TOL_MEAN_ABS = 2e-3
# reading R10: |o| shrinks like 1/sqrt(keys) under near-uniform attention (~1e-3 at 1M), where the
# absolute bounds cannot fail; the relative L2 error of every (layer, q head) is bounded too.  bf16 P and bf16
# output rounding give ~2^-9 relative, so 1e-2 leaves a 3-5x margin while a dropped history block or a 2%
# scale error fails it.
TOL_REL_L2 = 1e-2


def rel_l2_per_head(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """||got - ref|| / ||ref|| per q head over rows and dims; got/ref [rows, Hq, d]."""
    num = np.sqrt(((got - ref) ** 2).sum(axis=(0, 2)))
    den = np.sqrt((ref ** 2).sum(axis=(0, 2)))
    return num / np.maximum(den, 1e-300)


@dataclass
class Run:
    layers: int
    q_heads: int
    kv_heads: int
    d: int
    chunks: list            # prefill chunk sizes, in order
    n_decode: int
    dist: str = "P"
    seed: int = synth.BASE_SEED
    chunk_cap: int = 0      # hi_init chunk (default: max of chunks)
    opts: dict = field(default_factory=dict)

    @property
    def s_prefill(self):
        return sum(self.chunks)

    @property
    def s_total(self):
        return self.s_prefill + self.n_decode


def run_gpu(r: Run, ctx=None):
    """Returns (outputs [L] float32 CPU tensors [s_total, Hq, d] as bf16->f32, ctx)."""
    from paper_2502_12574_b200.headinfer import HeadInfer
    cap = r.chunk_cap or max(r.chunks + [1])
    if ctx is None:
        ctx = HeadInfer(r.layers, r.q_heads, r.kv_heads, r.d, r.s_total, cap, **r.opts)
    outs = [torch.empty((r.s_total, r.q_heads, r.d), dtype=torch.bfloat16, device="cuda") for _ in range(r.layers)]
    pos = 0
    for n in r.chunks:
        for layer in range(r.layers):
            Q = fill_(torch.empty((n, r.q_heads, r.d), dtype=torch.bfloat16, device="cuda"), r.seed, 0, r.dist, layer, 0, pos)
            K = fill_(torch.empty((n, r.kv_heads, r.d), dtype=torch.bfloat16, device="cuda"), r.seed, 1, r.dist, layer, 0, pos)
            V = fill_(torch.empty((n, r.kv_heads, r.d), dtype=torch.bfloat16, device="cuda"), r.seed, 2, r.dist, layer, 0, pos)
            ctx.prefill_chunk(layer, Q, K, V, outs[layer][pos:pos + n])
        pos += n
    for t in range(r.n_decode):
        for layer in range(r.layers):
            q = fill_(torch.empty((1, r.q_heads, r.d), dtype=torch.bfloat16, device="cuda"), r.seed, 0, r.dist, layer, 0, pos)
            k = fill_(torch.empty((1, r.kv_heads, r.d), dtype=torch.bfloat16, device="cuda"), r.seed, 1, r.dist, layer, 0, pos)
            v = fill_(torch.empty((1, r.kv_heads, r.d), dtype=torch.bfloat16, device="cuda"), r.seed, 2, r.dist, layer, 0, pos)
            ctx.decode(layer, q[0], k[0], v[0], outs[layer][pos])
        pos += 1
    torch.cuda.synchronize()
    return [o.float().cpu() for o in outs], ctx


def run_oracle(r: Run):
    """fp64 oracle outputs [L] of [s_total, Hq, d] plus the generated (q, k, v) per layer."""
    from oracle import gqa_attention
    res, inputs = [], []
    for layer in range(r.layers):
        q, k, v = synth.gen_qkv(r.seed, r.dist, layer, 0, r.s_total, r.q_heads, r.kv_heads, r.d)
        res.append(gqa_attention(q, k, v, 0))
        inputs.append((q, k, v))
    return res, inputs


def compare(gpu_outs, ref_outs, tol_max=TOL_MAX_ABS, tol_mean=TOL_MEAN_ABS, tol_rel=TOL_REL_L2):
    """Per layer: max-abs, mean-abs and the relative L2 error of every q head (R10); all three asserted."""
    worst = {"max_abs": 0.0, "mean_abs": 0.0, "rel_l2": 0.0}
    for g, ref in zip(gpu_outs, ref_outs):
        gd = g.double().numpy()
        err = np.abs(gd - ref)
        worst["max_abs"] = max(worst["max_abs"], float(err.max()))
        worst["mean_abs"] = max(worst["mean_abs"], float(err.mean()))
        worst["rel_l2"] = max(worst["rel_l2"], float(rel_l2_per_head(gd, ref).max()))
        assert np.all(np.isfinite(g.numpy())), "non-finite GPU output"
    assert worst["max_abs"] <= tol_max, worst
    assert worst["mean_abs"] <= tol_mean, worst
    assert worst["rel_l2"] <= tol_rel, worst
    return worst


def check_host_kv(ctx, r: Run, inputs, upto=None):
    """Host KV store must be bit-exact to the K/V fed in, for every (layer, head, pos)."""
    upto = r.s_total if upto is None else upto
    for layer in range(r.layers):
        _, k, v = inputs[layer]
        for h in range(r.kv_heads // ctx.world):
            hk, hv = ctx.read_host_kv(layer, h, 0, upto)
            hg = ctx.rank * (r.kv_heads // ctx.world) + h
            assert np.array_equal(hk.view(torch.int16).numpy().view(np.uint16), k[:upto, hg]), (layer, h)
            assert np.array_equal(hv.view(torch.int16).numpy().view(np.uint16), v[:upto, hg]), (layer, h)
