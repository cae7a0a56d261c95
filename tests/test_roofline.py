"""Work counters pinned to the paper's printed App. C values (RTX-4090 table)
and to the paper's memory tables, in the paper's conventions."""
import pytest

from paper_2502_12574_b200 import roofline as rf

S8B = rf.LLAMA3_8B


@pytest.mark.parametrize("S,ops,mem,kv", [
    (1024, 17e9, 21e6, 4.2e6),        # flashattention (1k)
    (10240, 1.7e12, 209e6, 42e6),     # flashattention (10k)
    (102400, 172e12, 2.1e9, 419e6),   # flashattention (100k) P:L849
])
def test_app_c_prefill_full_layer(S, ops, mem, kv):
    r = rf.paper_prefill(S8B, S)
    assert r["ops"] == pytest.approx(ops, rel=0.03)
    assert r["memory"] == pytest.approx(mem, rel=0.03)
    assert r["kv_memory"] == pytest.approx(kv, rel=0.03)


@pytest.mark.parametrize("S,ops,mem,kv", [
    (1024, 2.1e9, 2.6e6, 0.5e6),      # head-wise (1k)
    (10240, 215e9, 26e6, 5.2e6),      # head-wise (10k)
    (102400, 21e12, 262e6, 52e6),     # head-wise (100k) P:L852
])
def test_app_c_prefill_headwise(S, ops, mem, kv):
    r = rf.paper_prefill(S8B, S, heads=1)
    assert r["ops"] == pytest.approx(ops, rel=0.05)
    assert r["memory"] == pytest.approx(mem, rel=0.05)
    assert r["kv_memory"] == pytest.approx(kv, rel=0.05)


@pytest.mark.parametrize("S,val,heads", [
    (1024, 17e6, None), (10240, 168e6, None), (102400, 1.7e9, None),
    (1024, 2.1e6, 1), (10240, 21e6, 1), (102400, 210e6, 1),
])
def test_app_c_decode(S, val, heads):
    r = rf.paper_decode(S8B, S, heads)
    assert r["ops"] == pytest.approx(val, rel=0.03)
    assert r["memory"] == pytest.approx(val, rel=0.03)


def test_kv_sizes_match_memory_tables():
    # "Total KV cache" 128 GB at 1M, Llama-3-8B (Tab. P:L738); per-head on-GPU = 128/256 GiB
    total = S8B.layers * S8B.kv_heads * rf.kv_bytes(S8B.head_dim, 1 << 20)
    assert total == 128 * 2**30
    assert rf.kv_bytes(128, 1 << 20) == 512 * 2**20  # one head's K+V (Eq. 11 with H = kv heads, R5)
    # HeadInfer-4000K on-GPU KV 3.91 GB = 2 ping-pong heads at 4,096,000 tokens
    assert 2 * rf.kv_bytes(128, 4_096_000) / 2**30 == pytest.approx(3.91, abs=0.01)
    # Layer-wise offload 45K: 5.63 GB total KV
    assert S8B.layers * S8B.kv_heads * rf.kv_bytes(128, 45 * 1024) / 2**30 == pytest.approx(5.63, abs=0.01)


def test_algorithmic_counters_exact_causal_pairs():
    # brute-force pair count: sum over new tokens t of (s + t + 1) visible keys
    d, g, s, n = 64, 2, 37, 11
    pairs = sum(s + t + 1 for t in range(n))
    assert rf.prefill_flops(d, g, s, n) == 4 * d * g * pairs
    assert rf.decode_flops(d, g, s) == 4 * d * g * (s + 1)
    step = rf.prefill_step(S8B, 1 << 20, 16384)
    assert step["h2d_bytes"] == 32 * 8 * 512 * (1 << 20)


def test_step_roofline_bound():
    peaks = {"bf16_tflops": 1000.0, "hbm_gbs": 5000.0, "h2d_gbs": 50.0, "d2h_gbs": 50.0}
    dec = rf.step_roofline_seconds(rf.decode_step(S8B, 1 << 20), peaks)
    assert dec["bound"] == "h2d"
    pre = rf.step_roofline_seconds(rf.prefill_step(S8B, 1 << 20, 16384), peaks)
    assert pre["bound"] == "tensor"


def test_duo_counters_brute_force():
    """NEXT-3 counters: duo_keys / duo_pairs against a direct enumeration of the visible key set
    {i <= p : i < n_sink or i > p - win} (reading R18), across the sink / window regimes."""
    for n_sink, win in [(0, 1), (3, 5), (64, 256), (10, 4), (7, 100)]:
        for s in [0, 1, 5, 60, 300]:
            for n in [1, 7, 130]:
                brute = sum(1 for p in range(s, s + n) for i in range(p + 1) if i < n_sink or i > p - win)
                assert rf.duo_pairs(s, n, n_sink, win) == brute, (n_sink, win, s, n)
                assert rf.duo_keys(s + n - 1, n_sink, win) == sum(
                    1 for i in range(s + n) if i < n_sink or i > s + n - 1 - win)


def test_duo_step_reduces_to_plain_without_streaming():
    a = rf.prefill_step(S8B, 4096, 1024, 1, 3)
    b = rf.prefill_step(S8B, 4096, 1024, 1, 3, streaming=0)
    assert a == b
    # a window covering the context makes a streaming head cost what a resident head costs in FLOPs
    c = rf.prefill_step(S8B, 4096, 1024, 1, 0, streaming=S8B.layers * S8B.kv_heads, n_sink=0, win=1 << 30)
    assert c["flops"] == pytest.approx(a["flops"])
    assert c["h2d_bytes"] == 0 and c["d2h_bytes"] == 0
