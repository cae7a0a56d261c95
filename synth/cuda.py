"""GPU twin of synth.gen_block (libsynth.so): seeded bf16 inputs generated directly in HBM.

Test/bench infrastructure only (no method arithmetic).  Bit-identical to synth/gen.py."""
from __future__ import annotations

import ctypes
import os

import torch

from .gen import DIST_ID

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python -m paper_2502_12574_b200.build`")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.synth_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                   ctypes.c_int64, ctypes.c_void_p]
        lib.synth_fill.restype = ctypes.c_int
        _lib = lib
    return _lib


def fill_(out: torch.Tensor, seed: int, tensor: int, dist: str, layer: int, head0: int, pos0: int) -> torch.Tensor:
    """Fill a CUDA bf16 tensor shaped [n_pos, n_heads, d] (or a strided token-major view whose
    last two dims are contiguous) with generator values for heads head0.., positions pos0.."""
    if not out.is_cuda or out.dtype != torch.bfloat16 or out.dim() != 3:
        raise ValueError("out must be a 3-D CUDA bf16 tensor [n_pos, n_heads, d]")
    n_pos, n_heads, d = out.shape
    if out.stride(2) != 1 or out.stride(1) != d:
        raise ValueError("heads/dims of out must be contiguous")
    rc = _load().synth_fill(out.data_ptr(), seed & 0xFFFFFFFFFFFFFFFF, tensor, DIST_ID[dist], layer, head0, n_heads,
                            pos0, n_pos, d, out.stride(0), torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill failed: cudaError {rc}")
    return out


def gen_block_cuda(seed: int, tensor: int, dist: str, layer: int, head0: int, n_heads: int, pos0: int, n_pos: int,
                   d: int, device=None) -> torch.Tensor:
    out = torch.empty((n_pos, n_heads, d), dtype=torch.bfloat16, device=device or "cuda")
    return fill_(out, seed, tensor, dist, layer, head0, pos0)


def fill_matrix_(out: torch.Tensor, seed: int, tensor: int, layer: int, scale_log2: int = 0, row0: int = 0) -> torch.Tensor:
    """GPU twin of synth.gen_matrix: fill a contiguous CUDA bf16 [rows, cols] (or [cols]) tensor."""
    flat = out.view(-1, out.shape[-1]) if out.dim() == 2 else out.view(1, -1)
    rows, cols = flat.shape
    if cols % 128:
        raise ValueError("cols must be a multiple of 128")
    fill_(flat.view(rows, cols // 128, 128), seed, tensor, "U", layer, 0, row0)
    if scale_log2:
        out.mul_(2.0 ** scale_log2)  # a power of two: exact in bf16
    return out


def gen_layer_weights_cuda(seed: int, layer: int, hidden: int, inter: int, q_heads: int, kv_heads: int, d: int) -> dict:
    """GPU twin of synth.gen_layer_weights (same bits)."""
    from .gen import (TENSOR_ATTN_NORM, TENSOR_MLP_NORM, TENSOR_WDOWN, TENSOR_WGU, TENSOR_WO, TENSOR_WQKV,
                      layer_weight_scales)
    sc = layer_weight_scales(hidden, inter, q_heads * d)
    e = lambda *shape: torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    return {
        "attn_norm": fill_matrix_(e(hidden), seed, TENSOR_ATTN_NORM, layer),
        "w_qkv": fill_matrix_(e((q_heads + 2 * kv_heads) * d, hidden), seed, TENSOR_WQKV, layer, sc["w_qkv"]),
        "w_o": fill_matrix_(e(hidden, q_heads * d), seed, TENSOR_WO, layer, sc["w_o"]),
        "mlp_norm": fill_matrix_(e(hidden), seed, TENSOR_MLP_NORM, layer),
        "w_gate_up": fill_matrix_(e(2 * inter, hidden), seed, TENSOR_WGU, layer, sc["w_gate_up"]),
        "w_down": fill_matrix_(e(hidden, inter), seed, TENSOR_WDOWN, layer, sc["w_down"]),
    }
