"""Seeded synthetic bf16 input generator (CPU/numpy twin).

This module is shared test/bench infrastructure: it holds NONE of the method's
arithmetic (no dot products, softmax, masking or accumulation) -- only the
counter-based hash that turns a coordinate into a bf16 value.  Both the fp64
oracle (``oracle/``) and the CUDA path consume its output; the CUDA twin lives
in ``synth/csrc/synth_kernel.cu`` and must produce identical bits
(``tests/test_synth.py`` pins this on the GPU).

Generator spec (SURVEY.md §8(d) "Synthetic inputs"), for coordinate
(seed, tensor, layer, head_global, pos, dim):

    key  = ((((tensor*128 + layer)*128 + head) << 23 | pos) << 8) | dim
    h    = splitmix64(key XOR (seed * 0x9E3779B97F4A7C15 mod 2^64))
    v    = (h >> 40) - 2^23                       # int24, in [-2^23, 2^23)
    x    = v * 2^-23 * scale                      # exact in fp32 (|v| < 2^24, scale = 2^k)
    bits = bf16_rne(x)

``head`` is the GLOBAL head index (q head for Q, kv head for K/V), so a head
shard on W GPUs sees exactly the data it would see at W=1.  ``pos`` is the
global token position; decode tokens continue it (prefill S, decode S, S+1, ...).

Value distributions:
  U    Q, K, V in U[-1, 1)                     near-uniform attention (throughput)
  P    Q * 16                                  peaked rows (main parity workload)
  S    K[pos 0] = +1.0, Q = |gen|             first-token "sink"
  ONE  V == 1.0                                exact-normalisation check
"""
from __future__ import annotations

import numpy as np

TENSOR_Q, TENSOR_K, TENSOR_V = 0, 1, 2
# NEXT-4 synthetic decoder layer: hidden-state input and the layer's random-init weights
TENSOR_X, TENSOR_ATTN_NORM, TENSOR_WQKV, TENSOR_WO, TENSOR_MLP_NORM, TENSOR_WGU, TENSOR_WDOWN = 3, 4, 5, 6, 7, 8, 9
DISTS = ("U", "P", "S", "ONE")
DIST_ID = {name: i for i, name in enumerate(DISTS)}
BASE_SEED = 0x48454144  # "HEAD"

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_BF16_ONE = np.uint16(0x3F80)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (inputs are finite)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bias = np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return ((u + bias) >> np.uint64(16)).astype(np.uint16)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact bf16 bits -> float64 (via fp32 bit shift)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def tensor_scale(tensor: int, dist: str) -> float:
    """Power-of-two scale applied to the raw int24/2^23 value."""
    if dist == "P" and tensor == TENSOR_Q:
        return 16.0
    return 1.0


def gen_block(seed: int, tensor: int, dist: str, layer: int, head0: int, n_heads: int,
              pos0: int, n_pos: int, d: int) -> np.ndarray:
    """bf16 bit patterns, shape [n_pos, n_heads, d] (token-major, like the ABI's Q/K/V).

    Heads head0 .. head0+n_heads-1 (GLOBAL indices), positions pos0 .. pos0+n_pos-1.
    """
    if dist not in DIST_ID:
        raise ValueError(f"unknown dist {dist!r}")
    if not (0 <= tensor < 16 and 0 <= layer < 128 and 0 <= head0 and head0 + n_heads <= 128
            and 0 <= pos0 and pos0 + n_pos <= (1 << 23) and 0 < d <= 256):
        raise ValueError("coordinate out of generator range")
    if dist == "ONE" and tensor == TENSOR_V:
        return np.full((n_pos, n_heads, d), _BF16_ONE, dtype=np.uint16)
    pos = np.arange(pos0, pos0 + n_pos, dtype=np.uint64)[:, None, None]
    head = np.arange(head0, head0 + n_heads, dtype=np.uint64)[None, :, None]
    dim = np.arange(d, dtype=np.uint64)[None, None, :]
    hi = np.uint64((tensor * 128 + layer) * 128)
    key = ((((hi + head) << np.uint64(23)) | pos) << np.uint64(8)) | dim
    with np.errstate(over="ignore"):
        seedmix = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _GOLDEN
    h = splitmix64(key ^ seedmix)
    v = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    x = v.astype(np.float32) * np.float32(2.0 ** -23) * np.float32(tensor_scale(tensor, dist))
    if dist == "S" and tensor == TENSOR_Q:
        x = np.abs(x)
    bits = f32_to_bf16_rne(x)
    if dist == "S" and tensor == TENSOR_K and pos0 == 0 and n_pos > 0:
        bits[0, :, :] = _BF16_ONE
    return bits


def gen_qkv(seed: int, dist: str, layer: int, pos0: int, n_pos: int,
            q_heads: int, kv_heads: int, d: int, q_head0: int = 0, kv_head0: int = 0):
    """(Q, K, V) bf16 bit arrays [n_pos, heads, d] for one layer and a position range."""
    q = gen_block(seed, TENSOR_Q, dist, layer, q_head0, q_heads, pos0, n_pos, d)
    k = gen_block(seed, TENSOR_K, dist, layer, kv_head0, kv_heads, pos0, n_pos, d)
    v = gen_block(seed, TENSOR_V, dist, layer, kv_head0, kv_heads, pos0, n_pos, d)
    return q, k, v


def gen_matrix(seed: int, tensor: int, layer: int, rows: int, cols: int, scale_log2: int = 0,
               row0: int = 0) -> np.ndarray:
    """bf16 bits [rows, cols] for the NEXT-4 layer tensors (distribution U): element (r, c) is the generator
    value at (tensor, layer, head = c // 128, pos = row0 + r, dim = c % 128), times 2^scale_log2 (a power of
    two: exact in bf16).  cols must be a multiple of 128 (at most 128 * 128)."""
    if cols % 128 or cols // 128 > 128:
        raise ValueError("cols must be a multiple of 128, at most 16384")
    b = gen_block(seed, tensor, "U", layer, 0, cols // 128, row0, rows, 128).reshape(rows, cols)
    if scale_log2:
        b = f32_to_bf16_rne(bf16_to_f32(b) * np.float32(2.0 ** scale_log2))
    return b


def layer_weight_scales(hidden: int, inter: int, q_dim: int) -> dict:
    """Power-of-two weight scales keeping the synthetic layer's activations O(1): 2^(1 - floor(log2(fan_in)/2))."""
    sc = lambda fan_in: 1 - (int(np.log2(fan_in)) // 2)
    return {"w_qkv": sc(hidden), "w_o": sc(q_dim), "w_gate_up": sc(hidden), "w_down": sc(inter)}


def gen_layer_weights(seed: int, layer: int, hidden: int, inter: int, q_heads: int, kv_heads: int, d: int) -> dict:
    """Random-init bf16 weights of one synthetic Llama decoder layer (include/hilayer.h layouts)."""
    sc = layer_weight_scales(hidden, inter, q_heads * d)
    return {
        "attn_norm": gen_matrix(seed, TENSOR_ATTN_NORM, layer, 1, hidden)[0],
        "w_qkv": gen_matrix(seed, TENSOR_WQKV, layer, (q_heads + 2 * kv_heads) * d, hidden, sc["w_qkv"]),
        "w_o": gen_matrix(seed, TENSOR_WO, layer, hidden, q_heads * d, sc["w_o"]),
        "mlp_norm": gen_matrix(seed, TENSOR_MLP_NORM, layer, 1, hidden)[0],
        "w_gate_up": gen_matrix(seed, TENSOR_WGU, layer, 2 * inter, hidden, sc["w_gate_up"]),
        "w_down": gen_matrix(seed, TENSOR_WDOWN, layer, hidden, inter, sc["w_down"]),
    }


def streaming_labels(seed: int, layers: int, kv_heads: int, frac: float = 0.5) -> np.ndarray:
    """Synthetic duo-attention head labels (NEXT-3; the paper's labels come from a trained model,
    App. D): uint8 [layers, kv_heads], 1 = streaming head.  Exactly round(frac * kv_heads)
    streaming heads per layer, chosen by ranking a counter hash of (seed, layer, head) -- a pure
    function of its arguments, no method arithmetic."""
    n_str = int(round(frac * kv_heads))
    lab = np.zeros((layers, kv_heads), dtype=np.uint8)
    for layer in range(layers):
        keys = np.array([(seed << 20) ^ (layer << 8) ^ h for h in range(kv_heads)], dtype=np.uint64)
        order = np.argsort(splitmix64(keys), kind="stable")
        lab[layer, order[:n_str]] = 1
    return lab
