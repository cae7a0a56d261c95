"""Thin Python binding of libheadinfer.so -- argument marshalling only.

Every step of the hot path (write-back, prefetch, attention, combine) runs in the native
library's kernels and copy streams; this module only checks tensor metadata and passes raw
pointers plus torch's current CUDA stream.  Names follow the C ABI (include/headinfer.h):
``hi_init``, ``hi_prefill_chunk``, ``hi_decode``, ``hi_free`` (+ introspection helpers), and the
``HeadInfer`` class wraps a context handle.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from ._lib import HIError, hi_options, hi_stats


def _check(ctx, status: int) -> None:
    if status != _lib.HI_OK:
        msg = _lib.load().hi_last_error(ctx).decode(errors="replace")
        raise HIError(status, msg)


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev_tensor(t: torch.Tensor, shape, name: str) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.bfloat16:
        raise ValueError(f"{name} must be bfloat16, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.data_ptr() % 16:
        raise ValueError(f"{name} must be 16-byte aligned")
    return t.data_ptr()


def hi_init(layers: int, q_heads: int, kv_heads: int, head_dim: int, max_ctx: int, chunk: int,
            rank: int = 0, world: int = 1, n_slots: int = 0, slot_tokens: int = 0, flags: int = 0,
            device: Optional[int] = None, numa_policy: int = 0, numa_node: int = 0,
            resident_kv_heads: int = 0, head_group: int = 1, streaming_heads=None, duo_sink: int = 0,
            duo_window: int = 0) -> int:
    """hi_init / hi_init_ex.  Returns the opaque context handle (an int).

    ``streaming_heads``: optional [layers, kv_heads] array-like of 0/1 (global kv heads), NEXT-3."""
    lib = _lib.load()
    handle = ctypes.c_void_p()
    lab = None
    if streaming_heads is not None:
        lab = (ctypes.c_ubyte * (layers * kv_heads))()
        flat = [int(x) for row in streaming_heads for x in row]
        if len(flat) != layers * kv_heads:
            raise ValueError(f"streaming_heads must be [layers={layers}, kv_heads={kv_heads}]")
        for i, x in enumerate(flat):
            lab[i] = 1 if x else 0
    opt = hi_options(n_slots=n_slots, slot_tokens=slot_tokens,
                     device=torch.cuda.current_device() if device is None else device,
                     flags=flags, numa_policy=numa_policy, numa_node=numa_node,
                     resident_kv_heads=resident_kv_heads, head_group=head_group,
                     streaming_heads=ctypes.cast(lab, ctypes.c_void_p) if lab is not None else None,
                     duo_sink=duo_sink, duo_window=duo_window)
    st = lib.hi_init_ex(layers, q_heads, kv_heads, head_dim, max_ctx, chunk, rank, world,
                        ctypes.byref(opt), ctypes.byref(handle))
    if st != _lib.HI_OK:
        raise HIError(st, lib.hi_last_error(None).decode(errors="replace"))
    return handle.value


def hi_prefill_chunk(ctx: int, layer: int, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                     out: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> None:
    n, hq, d = Q.shape
    hkv = K.shape[1]
    args = (_dev_tensor(Q, (n, hq, d), "Q"), _dev_tensor(K, (n, hkv, d), "K"),
            _dev_tensor(V, (n, hkv, d), "V"), _dev_tensor(out, (n, hq, d), "out"))
    _check(ctx, _lib.load().hi_prefill_chunk(ctx, layer, *args, n, _stream_ptr(stream)))


def hi_decode(ctx: int, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
              stream: Optional[torch.cuda.Stream] = None) -> None:
    hq, d = q.shape
    hkv = k.shape[0]
    args = (_dev_tensor(q, (hq, d), "q"), _dev_tensor(k, (hkv, d), "k"), _dev_tensor(v, (hkv, d), "v"),
            _dev_tensor(out, (hq, d), "out"))
    _check(ctx, _lib.load().hi_decode(ctx, layer, *args, _stream_ptr(stream)))


def hi_free(ctx: Optional[int]) -> None:
    _lib.load().hi_free(ctx)


class HeadInfer:
    """One head-shard context: host KV store + staging + streams on the current device.

    Local head counts: Hq_loc = q_heads // world, Hkv_loc = kv_heads // world; Q/out tensors
    carry the shard's q heads, K/V the shard's kv heads (see include/headinfer.h)."""

    def __init__(self, layers: int, q_heads: int, kv_heads: int, head_dim: int, max_ctx: int, chunk: int,
                 rank: int = 0, world: int = 1, **opts):
        self.layers, self.q_heads, self.kv_heads, self.head_dim = layers, q_heads, kv_heads, head_dim
        self.max_ctx, self.chunk, self.rank, self.world = max_ctx, chunk, rank, world
        self.hq_loc, self.hkv_loc = q_heads // world, kv_heads // world
        self._ctx = hi_init(layers, q_heads, kv_heads, head_dim, max_ctx, chunk, rank, world, **opts)

    # -- hot path ---------------------------------------------------------------------------
    def prefill_chunk(self, layer: int, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(Q)
        hi_prefill_chunk(self._ctx, layer, Q, K, V, out)
        return out

    def decode(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
               out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(q)
        hi_decode(self._ctx, layer, q, k, v, out)
        return out

    # -- introspection / preparation ----------------------------------------------------------
    def seq_len(self, layer: int) -> int:
        return int(_lib.load().hi_seq_len(self._ctx, layer))

    def set_seq_len(self, layer: int, s: int) -> None:
        _check(self._ctx, _lib.load().hi_set_seq_len(self._ctx, layer, s))

    def read_host_kv(self, layer: int, kv_head_local: int, pos: int, n: int):
        k = torch.empty((n, self.head_dim), dtype=torch.bfloat16)
        v = torch.empty((n, self.head_dim), dtype=torch.bfloat16)
        _check(self._ctx, _lib.load().hi_read_host_kv(self._ctx, layer, kv_head_local, pos, n,
                                                      k.data_ptr(), v.data_ptr()))
        return k, v

    def write_host_kv(self, layer: int, kv_head_local: int, pos: int, k: torch.Tensor, v: torch.Tensor) -> None:
        n = k.shape[0]
        if k.shape != (n, self.head_dim) or v.shape != k.shape or k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
            raise ValueError("k, v must be bf16 [n, head_dim]")
        k, v = k.contiguous(), v.contiguous()
        _check(self._ctx, _lib.load().hi_write_host_kv(self._ctx, layer, kv_head_local, pos, n, k.data_ptr(),
                                                       v.data_ptr(), 1 if k.is_cuda else 0))

    def synchronize(self) -> None:
        _check(self._ctx, _lib.load().hi_synchronize(self._ctx))

    def stats(self) -> dict:
        s = hi_stats()
        _check(self._ctx, _lib.load().hi_get_stats(self._ctx, ctypes.byref(s)))
        return s.as_dict()

    @property
    def handle(self) -> int:
        return self._ctx

    def close(self) -> None:
        if self._ctx:
            hi_free(self._ctx)
            self._ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
