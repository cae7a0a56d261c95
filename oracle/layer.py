"""Oracle for NEXT-4: one synthetic Llama decoder layer around the attention path (TEST INFRASTRUCTURE:
only tests/, __graft_entry__.smoke() and bench.py's cpu legs may import it; the product path never does).

What it computes (include/hilayer.h; the paper's model family, Llama-3; its HF-style layer
code, App. E, is prior art), written out step by step in fp64 for hidden states x [S, H] at
positions 0 .. S-1 (the whole sequence at once: causal attention makes chunked prefill and decode the
same computation, Eq. 3 P:L161 / Eq. 9):

    xn   = rmsnorm(x) * attn_norm                  rmsnorm(x) = x / sqrt(mean(x^2) + eps)
    q|k|v = xn W_qkv^T
    q, k = rope(q), rope(k)                        rotate-half RoPE, inv_freq_i = theta^(-2i/d), angle = p * inv_freq_i
    a    = causal GQA attention(q, k, v)           (oracle.gqa_attention: the pinned attention oracle)
    x1   = x + a W_o^T
    xn2  = rmsnorm(x1) * mlp_norm
    g|u  = xn2 W_gate_up^T
    y    = x1 + (silu(g) * u) W_down^T             silu(g) = g / (1 + exp(-g))

With ``bf16_boundaries=True`` (the default, reading R19 in DESIGN.md) every line's result is rounded to
bf16 (round-to-nearest-even from the fp64 value), as the GPU stores it; the arithmetic inside each line
stays fp64.  With ``False`` nothing is rounded (pinned against transformers' LlamaDecoderLayer in fp64).
"""
from __future__ import annotations

import numpy as np

from synth import bf16_to_f64


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> nearest bf16 value (ties to even), returned as fp64.  x = m * 2^e with m in [0.5, 1):
    bf16 keeps 8 significant bits, so round m * 2^8 to the nearest integer (np.rint: ties to even)."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    return np.ldexp(np.rint(m * 256.0) / 256.0, e)


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Bit patterns of values that are already exactly bf16 (after bf16_round)."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)  # exact: a bf16 value is an fp32 value
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def rms_norm(x: np.ndarray, gamma: np.ndarray, eps: float) -> np.ndarray:
    """gamma * x / sqrt(mean(x^2) + eps), per row (RMSNorm, Llama)."""
    return gamma * x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """Rotate-half RoPE on x [S, heads, d] at positions pos [S]: pairs (i, i + d/2) rotated by
    pos * theta^(-2i/d)."""
    d = x.shape[-1]
    inv = theta ** (-(2.0 * np.arange(d // 2)) / d)
    ang = pos.astype(np.float64)[:, None] * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(g: np.ndarray) -> np.ndarray:
    return g / (1.0 + np.exp(-g))


def causal_gqa_f64(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Textbook causal GQA attention on fp64 arrays (full score matrix, explicit mask, row softmax) -- the
    unrounded variant's attention (the rounded variant uses the C oracle on bf16 bits)."""
    S, hq, d = q.shape
    g = hq // k.shape[1]
    kk, vv = np.repeat(k, g, axis=1), np.repeat(v, g, axis=1)
    sc = np.einsum("qhd,khd->hqk", q, kk) / np.sqrt(d)
    sc = np.where(np.tril(np.ones((S, S), dtype=bool))[None], sc, -np.inf)
    sc = sc - sc.max(axis=-1, keepdims=True)
    w = np.exp(sc)
    w = w / w.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", w, vv)


def layer_forward(x: np.ndarray, w: dict, q_heads: int, kv_heads: int, d: int, theta: float, eps: float,
                  bf16_boundaries: bool = True) -> np.ndarray:
    """One decoder layer over positions 0 .. S-1.  x: fp64 [S, H] (exact bf16 values when rounding);
    w: fp64 weights (see synth.gen_layer_weights for names / layouts).  Returns y [S, H] fp64."""
    from oracle import gqa_attention
    R = bf16_round if bf16_boundaries else (lambda a: a)
    S = x.shape[0]
    pos = np.arange(S)
    xn = R(rms_norm(x, w["attn_norm"], eps))
    qkv = R(xn @ w["w_qkv"].T)
    q = qkv[:, : q_heads * d].reshape(S, q_heads, d)
    k = qkv[:, q_heads * d:(q_heads + kv_heads) * d].reshape(S, kv_heads, d)
    v = qkv[:, (q_heads + kv_heads) * d:].reshape(S, kv_heads, d)
    q, k = R(rope(q, pos, theta)), R(rope(k, pos, theta))
    if bf16_boundaries:
        a = R(gqa_attention(f64_to_bf16_bits(q), f64_to_bf16_bits(k), f64_to_bf16_bits(v), 0))
    else:
        a = causal_gqa_f64(q, k, v)
    x1 = R(x + a.reshape(S, q_heads * d) @ w["w_o"].T)
    xn2 = R(rms_norm(x1, w["mlp_norm"], eps))
    gu = R(xn2 @ w["w_gate_up"].T)
    inter = gu.shape[1] // 2
    act = R(silu(gu[:, :inter]) * gu[:, inter:])
    return R(x1 + act @ w["w_down"].T)


def weights_f64(wbits: dict) -> dict:
    """bf16 bit weights (synth.gen_layer_weights) -> exact fp64 arrays."""
    return {k: bf16_to_f64(v) for k, v in wbits.items()}
