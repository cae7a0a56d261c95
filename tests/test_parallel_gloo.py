"""N>1 host logic on CPU: head sharding + the output all-gather (world_size 2, gloo).

Each rank computes ITS shard's outputs with the fp64 oracle on the shard's heads (the
attention is per head, so that is exactly what the rank's GPU would produce up to rounding);
after gather_heads + to_token_major every rank must hold the full-model oracle output
bit-for-bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2502_12574_b200.parallel import gather_heads, shard, to_token_major


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, hq, hkv, d, n, q0, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import gqa_attention
        sh = shard(hq, hkv, rank, world)
        q, k, v = synth.gen_qkv(7, "P", 0, 0, n, hq, hkv, d)
        (q_lo, q_hi), (k_lo, k_hi) = sh["q"], sh["kv"]
        local = gqa_attention(q[q0:, q_lo:q_hi], k[:, k_lo:k_hi], v[:, k_lo:k_hi], q0)
        gathered = gather_heads(torch.from_numpy(local))
        full = to_token_major(gathered).numpy()
        ref = gqa_attention(q[q0:], k, v, q0)
        result[rank] = bool(np.array_equal(full, ref))
        # decode-shaped gather: [Hq_loc, d] per rank
        g1 = to_token_major(gather_heads(torch.from_numpy(local[-1])))
        result[world + rank] = bool(np.array_equal(g1.numpy(), ref[-1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("hq,hkv,world", [(8, 4, 2), (32, 8, 2), (32, 8, 4)])
def test_two_rank_head_shard_gather_equals_full(hq, hkv, world):
    """W = 2 (and W = 4: two kv heads per rank, the 4-GPU row of configs[2]) head shards gathered."""
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), hq, hkv, 16, 40, 10, result), nprocs=world, join=True)
    assert all(result[i] for i in range(2 * world)), dict(result)


def test_shard_ranges_cover_heads():
    seen_q, seen_kv = [], []
    for r in range(4):
        sh = shard(32, 8, r, 4)
        seen_q += list(range(*sh["q"]))
        seen_kv += list(range(*sh["kv"]))
        # every local q head's kv head is local (GQA groups never straddle ranks)
        for j in range(*sh["q"]):
            assert sh["kv"][0] <= j // 4 < sh["kv"][1]
    assert seen_q == list(range(32)) and seen_kv == list(range(8))
    with pytest.raises(ValueError):
        shard(32, 8, 0, 3)
