"""Thin Python binding of the NEXT-4 layer ABI (include/hilayer.h) -- argument marshalling only.

``HeadInferLayer`` wraps an ``hl_model`` around a ``HeadInfer`` context: every step of the layer
(RMSNorm, GEMMs, RoPE, SwiGLU, the offloaded attention) runs in libheadinfer.so on the caller's stream.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from ._lib import HIError, hl_weights
from .headinfer import HeadInfer, _dev_tensor, _stream_ptr

WEIGHT_NAMES = ("attn_norm", "w_qkv", "w_o", "mlp_norm", "w_gate_up", "w_down")


class HeadInferLayer:
    """Synthetic Llama decoder layers (weights supplied per call) around one HeadInfer context."""

    def __init__(self, hi: HeadInfer, hidden: int, inter: int, rope_theta: float = 500000.0, rms_eps: float = 1e-5):
        self.hi, self.hidden, self.inter = hi, hidden, inter
        lib = _lib.load()
        h = ctypes.c_void_p()
        st = lib.hl_create(hi.handle, hidden, inter, rope_theta, rms_eps, ctypes.byref(h))
        if st != _lib.HI_OK:
            raise HIError(st, lib.hl_last_error(None).decode(errors="replace"))
        self._m = h.value
        self._wcache = {}

    def _weights(self, w: dict) -> hl_weights:
        hq, hkv, d, H, I = self.hi.hq_loc, self.hi.hkv_loc, self.hi.head_dim, self.hidden, self.inter // self.hi.world
        shapes = {"attn_norm": (H,), "w_qkv": ((hq + 2 * hkv) * d, H), "w_o": (H, hq * d), "mlp_norm": (H,),
                  "w_gate_up": (2 * I, H), "w_down": (H, I)}
        return hl_weights(**{k: _dev_tensor(w[k], shapes[k], k) for k in WEIGHT_NAMES})

    def _check(self, st: int) -> None:
        if st != _lib.HI_OK:
            raise HIError(st, _lib.load().hl_last_error(self._m).decode(errors="replace"))

    def prefill_chunk(self, layer: int, w: dict, x: torch.Tensor, stream: Optional[torch.cuda.Stream] = None):
        """x [n, hidden] bf16, updated in place to the layer's output."""
        n = x.shape[0]
        ptr = _dev_tensor(x, (n, self.hidden), "x")
        ws = self._weights(w)
        self._check(_lib.load().hl_prefill_chunk(self._m, layer, ctypes.byref(ws), ptr, n, _stream_ptr(stream)))
        return x

    def decode(self, layer: int, w: dict, x: torch.Tensor, stream: Optional[torch.cuda.Stream] = None):
        """x [hidden] bf16 (one token), updated in place."""
        ptr = _dev_tensor(x, (self.hidden,), "x")
        ws = self._weights(w)
        self._check(_lib.load().hl_decode(self._m, layer, ctypes.byref(ws), ptr, _stream_ptr(stream)))
        return x

    # -- tensor parallel (context world > 1; include/hilayer.h): the caller all-reduces y and z between the calls
    def attn_partial(self, layer: int, w: dict, x: torch.Tensor, decode: bool = False, y: Optional[torch.Tensor] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """x [n, hidden] bf16 (read); returns y [n, hidden] fp32 = this rank's attention output times W_o^T."""
        n = 1 if decode else x.shape[0]
        xp = _dev_tensor(x, (n, self.hidden) if not decode or x.dim() == 2 else (self.hidden,), "x")
        if y is None:
            y = torch.empty((n, self.hidden), dtype=torch.float32, device=x.device)
        ws = self._weights(w)
        self._check(_lib.load().hl_attn_partial(self._m, layer, ctypes.byref(ws), xp, n, 1 if decode else 0,
                                                y.data_ptr(), _stream_ptr(stream)))
        return y

    def mlp_partial(self, layer: int, w: dict, x: torch.Tensor, y: torch.Tensor, z: Optional[torch.Tensor] = None,
                    stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """x = bf16(x + y) in place (y: the all-reduced attention partials); returns z fp32 = this rank's MLP partial."""
        n = y.shape[0]
        xp = _dev_tensor(x, (n, self.hidden) if x.dim() == 2 else (self.hidden,), "x")
        if y.dtype != torch.float32 or not y.is_contiguous() or tuple(y.shape) != (n, self.hidden):
            raise ValueError("y must be contiguous fp32 [n, hidden]")
        if z is None:
            z = torch.empty_like(y)
        ws = self._weights(w)
        self._check(_lib.load().hl_mlp_partial(self._m, layer, ctypes.byref(ws), xp, y.data_ptr(), n, z.data_ptr(),
                                               _stream_ptr(stream)))
        return z

    def residual_add(self, x: torch.Tensor, z: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """x = bf16(x + z) (z: the all-reduced MLP partials)."""
        n = z.shape[0]
        xp = _dev_tensor(x, (n, self.hidden) if x.dim() == 2 else (self.hidden,), "x")
        self._check(_lib.load().hl_residual_add(self._m, xp, z.data_ptr(), n, _stream_ptr(stream)))
        return x

    def close(self) -> None:
        if getattr(self, "_m", None):
            _lib.load().hl_free(self._m)
            self._m = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hl_gemm(w: torch.Tensor, x: torch.Tensor, y: torch.Tensor, beta: bool = False,
            stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """include/hilayer.h hl_gemm: y[n, mo] = (beta ? y : 0) + x[n, kd] w[mo, kd]^T (bf16, fp32 accumulate, one
    rounding).  Argument marshalling only."""
    mo, kd = w.shape
    n = x.shape[0]
    for t, shp, name in ((w, (mo, kd), "w"), (x, (n, kd), "x"), (y, (n, mo), "y")):
        if not t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous() or tuple(t.shape) != shp:
            raise ValueError(f"{name} must be a contiguous CUDA bf16 tensor of shape {shp}")
    s = stream if stream is not None else torch.cuda.current_stream()
    st = _lib.load().hl_gemm(w.data_ptr(), x.data_ptr(), y.data_ptr(), mo, n, kd, 1 if beta else 0, s.cuda_stream)
    if st != _lib.HI_OK:
        raise _lib.HIError(st, _lib.load().hl_last_error(None).decode(errors="replace"))
    return y


def shard_layer_weights(w: dict, q_heads: int, kv_heads: int, head_dim: int, inter: int, rank: int, world: int) -> dict:
    """Rank `rank`'s tensor-parallel shard of one layer's full weights (include/hilayer.h): the q/k/v rows and
    W_o columns of its head shard (parallel.shard), its inter/world gate, up and down columns; norms replicated.
    Slicing only (copies), no arithmetic."""
    from .parallel import shard
    sh = shard(q_heads, kv_heads, rank, world)
    (q0, q1), (k0, k1) = sh["q"], sh["kv"]
    d = head_dim
    qkv = w["w_qkv"]
    ko = q_heads * d
    vo = ko + kv_heads * d
    il = inter // world
    i0 = rank * il
    return {
        "attn_norm": w["attn_norm"], "mlp_norm": w["mlp_norm"],
        "w_qkv": torch.cat([qkv[q0 * d:q1 * d], qkv[ko + k0 * d:ko + k1 * d], qkv[vo + k0 * d:vo + k1 * d]]).contiguous(),
        "w_o": w["w_o"][:, q0 * d:q1 * d].contiguous(),
        "w_gate_up": torch.cat([w["w_gate_up"][i0:i0 + il], w["w_gate_up"][inter + i0:inter + i0 + il]]).contiguous(),
        "w_down": w["w_down"][:, i0:i0 + il].contiguous(),
    }
