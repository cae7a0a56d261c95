"""C-ABI contract on a GPU: error paths are atomic (no state change), capacity is enforced,
seq_len bookkeeping, stats, hi_set_seq_len rewinds."""
import pytest
import torch

from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]


def _ctx(**kw):
    from paper_2502_12574_b200.headinfer import HeadInfer
    return HeadInfer(2, 4, 2, 64, 300, 128, **kw)


def _qkv(n, hq=4, hkv=2, d=64):
    mk = lambda h: torch.randn(n, h, d, device="cuda").clamp(-1, 1).to(torch.bfloat16)
    return mk(hq), mk(hkv), mk(hkv)


def test_error_paths_leave_state_unchanged():
    from paper_2502_12574_b200._lib import HIError
    ctx = _ctx()
    Q, K, V = _qkv(128)
    ctx.prefill_chunk(0, Q, K, V)
    assert ctx.seq_len(0) == 128 and ctx.seq_len(1) == 0
    with pytest.raises(HIError) as e:
        ctx.prefill_chunk(2, Q, K, V)  # layer out of range
    assert e.value.status == 2
    Q2, K2, V2 = _qkv(129)
    with pytest.raises(HIError) as e:
        ctx.prefill_chunk(0, Q2, K2, V2)  # n > chunk
    assert e.value.status == 2
    ctx.prefill_chunk(0, Q, K, V)  # 256
    with pytest.raises(HIError) as e:
        ctx.prefill_chunk(0, Q, K, V)  # 384 > max_ctx 300
    assert e.value.status == 3
    assert ctx.seq_len(0) == 256
    Q3, K3, V3 = _qkv(44)
    ctx.prefill_chunk(0, Q3, K3, V3)  # exactly max_ctx
    assert ctx.seq_len(0) == 300
    q, k, v = _qkv(1)
    with pytest.raises(HIError) as e:
        ctx.decode(0, q[0], k[0], v[0])
    assert e.value.status == 3
    ctx.decode(1, q[0], k[0], v[0])
    assert ctx.seq_len(1) == 1
    st = ctx.stats()
    assert st["prefill_calls"] == 3 and st["decode_calls"] == 1
    assert st["d2h_bytes"] == (300 + 1) * 2 * 2 * 64 * 2
    ctx.set_seq_len(0, 128)
    assert ctx.seq_len(0) == 128
    ctx.close()


def test_bad_tensor_metadata_rejected_by_binding():
    ctx = _ctx()
    Q, K, V = _qkv(16)
    with pytest.raises(ValueError):
        ctx.prefill_chunk(0, Q.float(), K, V)
    with pytest.raises(ValueError):
        ctx.prefill_chunk(0, Q.cpu(), K, V)
    with pytest.raises(ValueError):
        ctx.prefill_chunk(0, Q, K[:, :1], V)
    assert ctx.seq_len(0) == 0
    ctx.close()


def test_init_reports_host_store_and_residency():
    ctx = _ctx(n_slots=3)
    st = ctx.stats()
    assert st["host_store_bytes"] == 2 * 2 * 2 * 300 * 64 * 2
    # one head would give 300/3 -> 64-token slots; the minimum block min(max_ctx/2, 32768) -> 128 tokens
    assert st["n_slots"] == 3 and st["slot_tokens"] == 128
    assert st["staging_bytes"] == 3 * 128 * 4 * 64 == st["staging_bound_bytes"]
    ctx.close()


@pytest.mark.parametrize("group", [2, -1])
def test_default_slots_keep_one_head_resident_with_head_groups(group):
    """Eq. 11 (reading R8): with the default slot size the staging ring holds at most one head's K+V
    at max_ctx whatever the head group (NEXT-2): slots shrink instead of the ring growing (long contexts,
    where the 32768-token minimum block does not bind)."""
    from paper_2502_12574_b200.headinfer import HeadInfer
    max_ctx, d = 1 << 20, 64
    ctx = HeadInfer(1, 32, 8, d, max_ctx, 1024, head_group=group)
    st = ctx.stats()
    one_head = 4 * d * max_ctx
    assert st["head_group"] == (2 if group == 2 else 8)
    assert st["staging_bound_bytes"] == one_head
    assert st["staging_bytes"] <= one_head
    assert st["slot_tokens"] * st["n_slots"] * st["head_group"] <= max_ctx
    ctx.close()


def test_timing_flag_reports_copy_engine_time():
    """HI_FLAG_TIMING brackets every history H2D block and every prefill write-back D2H with events on the
    copy streams: busy time > 0 and a rate below the host link's physical ceiling (PCIe 5 x16: 64 GB/s)."""
    from paper_2502_12574_b200._lib import HI_FLAG_TIMING
    from paper_2502_12574_b200.headinfer import HeadInfer
    from synth.cuda import fill_
    L, hq, hkv, d, c = 2, 32, 8, 128, 4096
    ctx = HeadInfer(L, hq, hkv, d, 4 * c, c, flags=HI_FLAG_TIMING)
    for i in range(4):
        for l in range(L):
            Q = fill_(torch.empty((c, hq, d), dtype=torch.bfloat16, device="cuda"), 1, 0, "U", l, 0, i * c)
            K = fill_(torch.empty((c, hkv, d), dtype=torch.bfloat16, device="cuda"), 1, 1, "U", l, 0, i * c)
            V = fill_(torch.empty((c, hkv, d), dtype=torch.bfloat16, device="cuda"), 1, 2, "U", l, 0, i * c)
            ctx.prefill_chunk(l, Q, K, V)
    ctx.synchronize()
    st = ctx.stats()
    assert st["h2d_bytes"] == L * hkv * 4 * d * c * (0 + 1 + 2 + 3)
    assert st["d2h_bytes"] == L * hkv * 4 * d * c * 4
    assert st["h2d_copy_ms"] > 0 and st["d2h_copy_ms"] > 0
    assert st["h2d_bytes"] / (st["h2d_copy_ms"] / 1e3) < 64e9
    assert st["d2h_bytes"] / (st["d2h_copy_ms"] / 1e3) < 64e9
    ctx.close()


@pytest.mark.parametrize("max_ctx,world,want", [(4096, 1, 8), (600_000, 1, 4), (1_048_704, 1, 4), (1_500_000, 1, 2),
                                                 (3_000_000, 1, 1), (600_000, 2, 4), (600_000, 8, 1),
                                                 (1_500_000, 2, 2)])
def test_paper_adaptive_head_groups(max_ctx, world, want):
    """HI_GROUP_PAPER: §4 "Adaptive Head-wise Offloading" -- all heads fused up to 500K, two groups to
    1M, four to 2M, eight (head-wise) beyond, for Llama-3-8B's 8 kv heads; a unit never spans ranks."""
    from paper_2502_12574_b200._lib import HI_GROUP_PAPER
    from paper_2502_12574_b200.headinfer import HeadInfer
    ctx = HeadInfer(1, 32, 8, 64, max_ctx, 256, 0, world, head_group=HI_GROUP_PAPER, numa_policy=1)
    st = ctx.stats()
    assert st["head_group"] == want
    # default slot size: one head's K+V (Eq. 11), unless the minimum block min(max_ctx/2, 32768) binds
    # (short contexts, DESIGN.md §4 "Short contexts"), where the ring is n_slots blocks of `want` heads
    min_blk = min((max_ctx // 2) // 64 * 64, 32768)
    ring_at_min = st["n_slots"] * want * min_blk * 4 * 64
    assert st["staging_bytes"] <= max(4 * 64 * max_ctx, ring_at_min)
    if max_ctx >= 1_000_000:
        assert st["staging_bytes"] <= 4 * 64 * max_ctx  # long contexts: one head, the rule unchanged
    ctx.close()


def test_short_context_blocks_are_long():
    """Short contexts: blocks of at least min(max_ctx/2, 32768) tokens, so a head's history is 2 copies, not
    n_slots * group of them; the bound reports the (small) ring."""
    from paper_2502_12574_b200.headinfer import HeadInfer
    max_ctx, d = 10240, 128
    ctx = HeadInfer(1, 32, 8, d, max_ctx, 1024, head_group=8)
    st = ctx.stats()
    assert st["slot_tokens"] == 5120
    assert st["staging_bytes"] == 4 * 8 * 5120 * 4 * d
    assert st["staging_bytes"] <= st["staging_bound_bytes"]
    ctx.close()
