"""Head sharding across GPUs.

Heads are the natural shard: attention is independent per head ("embarrassingly parallel",
App. D; head-wise independence, §5), so rank r of W owns kv heads
[r*H_kv/W, (r+1)*H_kv/W) and the q heads of their groups; each rank streams only its own
heads' K/V from its own pinned host store, and no K/V ever crosses GPUs.  The only
collective is one all-gather of the per-head outputs after each layer call (the "Concatenate"
of Alg. 1 line 15), NCCL over NVLink on a GPU box, gloo in the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(q_heads: int, kv_heads: int, rank: int, world: int) -> dict:
    """Head ranges owned by `rank` (global indices, half-open)."""
    if kv_heads % world or q_heads % kv_heads:
        raise ValueError("world must divide kv_heads and kv_heads must divide q_heads")
    hkv = kv_heads // world
    g = q_heads // kv_heads
    return {"kv": (rank * hkv, (rank + 1) * hkv), "q": (rank * hkv * g, (rank + 1) * hkv * g),
            "kv_local": hkv, "q_local": hkv * g}


def gather_heads(out_local: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather the rank-local outputs [..., Hq_loc, d] into a rank-major [W, ..., Hq_loc, d]
    tensor (one collective, no permute: rank-major IS global q-head order per token once the
    W axis is moved next to the head axis, see ``to_token_major``)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world, *out_local.shape), dtype=out_local.dtype, device=out_local.device)
    if out_local.is_cuda and dist.get_backend(group) == "gloo":
        # validation mode (several ranks sharing one GPU, e.g. bench.py --ranks-share-gpu): gloo has no
        # CUDA all-gather, so stage through host memory.  The NCCL path below is the product path.
        parts = [torch.empty(out_local.shape, dtype=out_local.dtype) for _ in range(world)]
        dist.all_gather(parts, out_local.cpu(), group=group)
        out.copy_(torch.stack(parts))
        return out
    dist.all_gather_into_tensor(out.view(-1), out_local.contiguous().view(-1), group=group)
    return out


def to_token_major(gathered: torch.Tensor) -> torch.Tensor:
    """[W, n, Hq_loc, d] (or [W, Hq_loc, d]) -> [n, Hq, d] (or [Hq, d]): global q head
    r*Hq_loc + j sits at gathered[r, ..., j, :]."""
    if gathered.dim() == 4:
        w, n, hq_loc, d = gathered.shape
        return gathered.permute(1, 0, 2, 3).reshape(n, w * hq_loc, d)
    w, hq_loc, d = gathered.shape
    return gathered.reshape(w * hq_loc, d)


def all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over the group (NCCL over NVLink on a GPU box; through host memory when the group is gloo
    and the tensor lives on a GPU -- the ranks-share-one-GPU validation mode)."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, group=group)
    return t


def tp_layer_step(layer, idx: int, w: dict, x: torch.Tensor, group=None, decode: bool = False,
                  bufs: dict | None = None) -> torch.Tensor:
    """One tensor-parallel decoder layer (include/hilayer.h): the library computes this rank's fp32 partials of
    the O and down projections; the two all-reduces between its three calls are the only collectives."""
    y = layer.attn_partial(idx, w, x, decode=decode, y=None if bufs is None else bufs.get("y"))
    all_reduce_sum(y, group)
    z = layer.mlp_partial(idx, w, x, y, z=None if bufs is None else bufs.get("z"))
    all_reduce_sum(z, group)
    layer.residual_add(x, z)
    return x
