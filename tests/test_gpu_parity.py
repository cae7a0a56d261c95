"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same seeded inputs.

Bar (BASELINE.json north_star): attention outputs within max-abs 2e-2 / mean-abs 2e-3 of the
oracle; host KV bytes bit-exact to the K/V fed in; special cases exact where the arithmetic
makes them exact (single key -> V[0]; V == 1 -> 1.0)."""
import numpy as np
import pytest
import torch

import synth
from conftest import cuda_available
from hi_harness import Run, check_host_kv, compare, run_gpu, run_oracle

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]

TINY = dict(layers=1, q_heads=4, kv_heads=2, d=64)  # BASELINE.json configs[0]


@pytest.mark.parametrize("dist", ["U", "P", "S", "ONE"])
def test_tiny_config_end_to_end(dist):
    """configs[0]: 1 layer, 4q/2kv, d64, 1024-token prefill in chunks of 256, then 16 decodes."""
    r = Run(**TINY, chunks=[256] * 4, n_decode=16, dist=dist)
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    st = ctx.stats()
    assert st["staging_bytes"] <= st["staging_bound_bytes"]
    assert ctx.seq_len(0) == 1040
    ctx.close()


@pytest.mark.parametrize("chunk", [64, 128, 256, 1024])
def test_chunk_size_sweep(chunk):
    r = Run(**TINY, chunks=[chunk] * (1024 // chunk), n_decode=4, dist="P")
    gpu, ctx = run_gpu(r)
    ref, _ = run_oracle(r)
    compare(gpu, ref)
    ctx.close()


@pytest.mark.parametrize("slots,slot_tokens", [(2, 64), (3, 96), (2, 1000), (5, 128)])
def test_block_and_slot_geometry(slots, slot_tokens):
    """Many / ragged history blocks per head and slot reuse across heads and calls."""
    r = Run(**TINY, chunks=[200, 300, 77, 256], n_decode=6, dist="S", chunk_cap=300,
            opts=dict(n_slots=slots, slot_tokens=slot_tokens))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()


@pytest.mark.parametrize("g", [1, 2, 4, 8])
@pytest.mark.parametrize("d", [64, 128])
def test_group_size_and_head_dim(g, d):
    """GQA packing of g q heads per 128-row tile; d in {64,128}; a ragged last chunk."""
    r = Run(layers=2, q_heads=2 * g, kv_heads=2, d=d, chunks=[250, 250, 100], n_decode=3, dist="P",
            opts=dict(slot_tokens=192))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()


def test_llama8b_shape_small_context():
    """Llama-3-8B head geometry (32q/8kv, d128) at a short context, 2 layers."""
    r = Run(layers=2, q_heads=32, kv_heads=8, d=128, chunks=[512, 512, 300], n_decode=4, dist="U",
            opts=dict(slot_tokens=512))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()


def test_v_one_gives_exactly_one():
    r = Run(**TINY, chunks=[256, 256], n_decode=5, dist="ONE", opts=dict(n_slots=2, slot_tokens=64))
    gpu, ctx = run_gpu(r)
    assert torch.all(gpu[0] == 1.0), "normalisation across blocks/splits must be exact with V == 1"
    ctx.close()


def test_first_row_equals_v0_exactly():
    r = Run(**TINY, chunks=[256], n_decode=0, dist="P")
    gpu, ctx = run_gpu(r)
    _, k, v = synth.gen_qkv(r.seed, r.dist, 0, 0, 1, 4, 2, 64)
    v0 = torch.from_numpy(synth.bf16_to_f32(v[0]))
    for j in range(4):
        assert torch.equal(gpu[0][0, j], v0[j // 2])
    ctx.close()


def test_decode_matches_prefill_of_one_more_token():
    """decode after prefill(S) ~= prefill(S+1)'s last row, on two contexts."""
    a = Run(**TINY, chunks=[256, 256, 100], n_decode=1, dist="P", chunk_cap=256)
    b = Run(**TINY, chunks=[256, 256, 101], n_decode=0, dist="P", chunk_cap=256)
    ga, ca = run_gpu(a)
    gb, cb = run_gpu(b)
    diff = (ga[0][612] - gb[0][612]).abs().max().item()
    assert diff <= 2e-2
    ca.close()
    cb.close()


def test_decode_from_empty_context_returns_v():
    r = Run(**TINY, chunks=[], n_decode=3, dist="U", chunk_cap=16)
    gpu, ctx = run_gpu(r)
    ref, _ = run_oracle(r)
    _, _, v = synth.gen_qkv(r.seed, r.dist, 0, 0, 1, 4, 2, 64)
    for j in range(4):
        assert torch.equal(gpu[0][0, j], torch.from_numpy(synth.bf16_to_f32(v[0, j // 2])))
    compare(gpu, ref)
    ctx.close()


def test_poison_mode_is_bit_identical():
    """Poisoning every slot with NaN before each H2D must not change a single output bit
    (a stale read would surface as NaN)."""
    base = Run(**TINY, chunks=[256] * 4, n_decode=8, dist="S", opts=dict(n_slots=2, slot_tokens=128))
    pois = Run(**TINY, chunks=[256] * 4, n_decode=8, dist="S",
               opts=dict(n_slots=2, slot_tokens=128, flags=0x1))
    g1, c1 = run_gpu(base)
    g2, c2 = run_gpu(pois)
    assert torch.equal(g1[0], g2[0])
    c1.close()
    c2.close()


def test_deterministic():
    r = Run(**TINY, chunks=[256] * 2, n_decode=4, dist="P")
    g1, c1 = run_gpu(r)
    g2, c2 = run_gpu(r)
    assert torch.equal(g1[0], g2[0])
    c1.close()
    c2.close()


def test_gpu_generator_matches_cpu_bits():
    from synth.cuda import gen_block_cuda
    for dist in synth.DISTS:
        for t in range(3):
            a = gen_block_cuda(99, t, dist, 3, 1, 5, 0, 300, 128).cpu().view(torch.int16).numpy().view(np.uint16)
            b = synth.gen_block(99, t, dist, 3, 1, 5, 0, 300, 128)
            assert np.array_equal(a, b), (dist, t)


@pytest.mark.parametrize("resident", [1, 3, 8, -1])
def test_resident_heads_next1(resident):
    """NEXT-1 (Alg. 1 H_on branch): the first R (layer, kv head) pairs keep their KV in HBM; results and
    the KV store contents must not depend on R (R = -1: as many as fit)."""
    r = Run(layers=2, q_heads=8, kv_heads=4, d=128, chunks=[300, 300, 100], n_decode=4, dist="P",
            opts=dict(slot_tokens=128, resident_kv_heads=resident))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    st = ctx.stats()
    assert st["resident_kv_heads"] == (8 if resident == -1 else resident)
    if st["resident_kv_heads"] == 8:
        assert st["host_store_bytes"] == 0 and st["h2d_bytes"] == 0
    ctx.close()


@pytest.mark.parametrize("group,resident,flags", [(2, 0, 0), (4, 0, 0), (8, 0, 0), (2, 3, 0), (-1, 0, 0)])
def test_head_groups_next2(group, resident, flags):
    """NEXT-2 (§4 adaptive head-wise offloading, Tab. 5-7): `group` kv heads per H2D block and per
    kernel launch; results and host KV must not depend on the group size, with resident heads in front
    (the groups start after them)."""
    r = Run(layers=2, q_heads=16, kv_heads=8, d=128, chunks=[300, 300, 100], n_decode=4, dist="P",
            opts=dict(slot_tokens=128, head_group=group, resident_kv_heads=resident, flags=flags))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    st = ctx.stats()
    assert st["head_group"] == (8 if group == -1 else group)  # auto: 5 tiles per head -> all 8 heads
    assert st["staging_bytes"] <= st["staging_bound_bytes"]
    ctx.close()


def test_head_groups_bit_identical_to_group1():
    """The per-head prefill arithmetic does not change with the grouping: prefill rows are bit-identical
    for G = 1, 4 (decode rows may differ in the last bits: the split-K partition depends on how many heads
    share a launch)."""
    outs = []
    for group in (1, 4):
        r = Run(layers=1, q_heads=32, kv_heads=8, d=128, chunks=[256, 256, 77], n_decode=3, dist="U",
                opts=dict(slot_tokens=192, head_group=group))
        gpu, ctx = run_gpu(r)
        outs.append(gpu[0][:589])
        ctx.close()
    assert torch.equal(outs[0], outs[1])
