"""GPU parity for NEXT-3, head-wise sparsity (duo-attention streaming heads; §4, App. D
L916-1000; reading R18 in DESIGN.md): streaming heads keep only the attention-sink rows and a window of
recent rows on the GPU and attend exactly those keys; retrieval heads keep (and offload) the full cache.
The CUDA path through the C ABI is compared with oracle.duo_gqa_attention (fp64) on the same seeded
inputs and synthetic labels (synth.streaming_labels -- the paper's labels need a trained model)."""
import numpy as np
import pytest
import torch

import synth
from conftest import cuda_available
from hi_harness import Run, compare, run_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]

TINY = dict(layers=1, q_heads=4, kv_heads=2, d=64)  # BASELINE.json configs[0]


def duo_run(r: Run, frac=0.5, n_sink=64, win=256, labels=None):
    if labels is None:
        labels = synth.streaming_labels(r.seed, r.layers, r.kv_heads, frac)
    r.opts = dict(r.opts, streaming_heads=labels.tolist(), duo_sink=n_sink if n_sink > 0 else -1, duo_window=win)
    return r, labels


def oracle_duo(r: Run, labels, n_sink, win):
    from oracle import duo_gqa_attention
    res, inputs = [], []
    for layer in range(r.layers):
        q, k, v = synth.gen_qkv(r.seed, r.dist, layer, 0, r.s_total, r.q_heads, r.kv_heads, r.d)
        res.append(duo_gqa_attention(q, k, v, 0, [bool(x) for x in labels[layer]], n_sink, win))
        inputs.append((q, k, v))
    return res, inputs


def check_kv(ctx, r: Run, inputs, labels, n_sink, win):
    """Retrieval heads: every cached row bit-exact.  Streaming heads: the sink rows and the last `win`
    rows bit-exact, any other row refused (HI_ESTATE) -- they were never kept."""
    from paper_2502_12574_b200._lib import HI_ESTATE, HIError
    s = r.s_total
    for layer in range(r.layers):
        _, k, v = inputs[layer]
        for h in range(r.kv_heads):
            u16 = lambda t: t.view(torch.int16).numpy().view(np.uint16)
            if not labels[layer][h]:
                hk, hv = ctx.read_host_kv(layer, h, 0, s)
                assert np.array_equal(u16(hk), k[:s, h]) and np.array_equal(u16(hv), v[:s, h]), (layer, h)
                continue
            ns = min(n_sink, s)
            if ns:
                hk, hv = ctx.read_host_kv(layer, h, 0, ns)
                assert np.array_equal(u16(hk), k[:ns, h]) and np.array_equal(u16(hv), v[:ns, h])
            lo = max(ns, s - win)
            if lo < s:
                hk, hv = ctx.read_host_kv(layer, h, lo, s - lo)
                assert np.array_equal(u16(hk), k[lo:s, h]) and np.array_equal(u16(hv), v[lo:s, h])
            if lo > ns:
                with pytest.raises(HIError) as e:
                    ctx.read_host_kv(layer, h, lo - 1, 1)
                assert e.value.status == HI_ESTATE


@pytest.mark.parametrize("dist", ["U", "P", "S", "ONE"])
def test_duo_tiny_config(dist):
    """configs[0] with 50% streaming heads (one of the two kv heads), sink 64 + window 256, 1024-token
    prefill in chunks of 256, then 16 decodes."""
    r, lab = duo_run(Run(**TINY, chunks=[256] * 4, n_decode=16, dist=dist))
    gpu, ctx = run_gpu(r)
    if dist == "ONE":
        assert torch.all(gpu[0] == 1.0), "normalisation over sink + window segments must be exact"
    ref, inputs = oracle_duo(r, lab, 64, 256)
    compare(gpu, ref)
    check_kv(ctx, r, inputs, lab, 64, 256)
    st = ctx.stats()
    assert st["streaming_kv_heads"] == int(lab.sum()) == 1
    # only the retrieval head is offloaded: host store and write-back hold one head
    assert st["host_store_bytes"] == 1 * 2 * r.s_total * 64 * 2
    ctx.close()


@pytest.mark.parametrize("n_sink,win", [(0, 1), (1, 7), (64, 256), (16, 300), (300, 100), (100, 1000), (0, 5000)])
def test_duo_sink_window_sweep(n_sink, win):
    """Ragged chunks and windows smaller / larger than a chunk, sinks that straddle chunk boundaries
    (300 with 200-token chunks), a window reaching back past the sink, one larger than the context (the
    streaming head is then plain causal attention), win = 1 with no sink (a row attends only itself)."""
    r, lab = duo_run(Run(**TINY, chunks=[200, 300, 77, 256], n_decode=6, dist="S", chunk_cap=300,
                         opts=dict(n_slots=2, slot_tokens=128)), n_sink=n_sink, win=win)
    gpu, ctx = run_gpu(r)
    ref, inputs = oracle_duo(r, lab, n_sink, win)
    compare(gpu, ref)
    check_kv(ctx, r, inputs, lab, n_sink, win)
    if n_sink == 0 and win == 1:  # each row is its own value, exactly
        _, _, v = inputs[0]
        h = int(np.flatnonzero(lab[0])[0])
        vv = torch.from_numpy(synth.bf16_to_f32(v[:, h]))
        for j in range(2 * h, 2 * h + 2):
            assert torch.equal(gpu[0][:, j], vv)
    ctx.close()


@pytest.mark.parametrize("g,d", [(1, 64), (4, 128), (8, 128), (2, 64)])
def test_duo_gqa_and_head_dim(g, d):
    r, lab = duo_run(Run(layers=2, q_heads=4 * g, kv_heads=4, d=d, chunks=[250, 250, 100], n_decode=3, dist="P",
                         opts=dict(slot_tokens=192)), n_sink=32, win=128)
    gpu, ctx = run_gpu(r)
    ref, inputs = oracle_duo(r, lab, 32, 128)
    compare(gpu, ref)
    check_kv(ctx, r, inputs, lab, 32, 128)
    ctx.close()


@pytest.mark.parametrize("group,resident", [(1, 0), (2, 0), (4, 3), (-1, 0), (2, -1)])
def test_duo_with_groups_and_resident(group, resident):
    """Streaming heads interleaved with resident (NEXT-1) and grouped offloaded (NEXT-2) retrieval heads:
    the unit lists are not contiguous in head order, so head maps carry the q/out columns per launch."""
    r, lab = duo_run(Run(layers=2, q_heads=32, kv_heads=8, d=128, chunks=[512, 512, 300], n_decode=4, dist="U",
                         opts=dict(slot_tokens=256, head_group=group, resident_kv_heads=resident)),
                     n_sink=64, win=256)
    gpu, ctx = run_gpu(r)
    ref, inputs = oracle_duo(r, lab, 64, 256)
    compare(gpu, ref)
    check_kv(ctx, r, inputs, lab, 64, 256)
    st = ctx.stats()
    assert st["streaming_kv_heads"] == int(lab.sum()) == 8
    ctx.close()


@pytest.mark.parametrize("frac", [0.0, 1.0])
def test_duo_all_or_no_streaming(frac):
    """frac 0: identical to plain head-wise offload.  frac 1: nothing offloaded (no host store, no H2D)."""
    r, lab = duo_run(Run(layers=2, q_heads=8, kv_heads=4, d=128, chunks=[300, 300, 100], n_decode=4, dist="P",
                         opts=dict(slot_tokens=128)), frac=frac, n_sink=16, win=100)
    gpu, ctx = run_gpu(r)
    ref, inputs = oracle_duo(r, lab, 16, 100)
    compare(gpu, ref)
    st = ctx.stats()
    if frac == 1.0:
        assert st["host_store_bytes"] == 0 and st["h2d_bytes"] == 0 and st["d2h_bytes"] == 0
    else:
        assert st["streaming_kv_heads"] == 0
    ctx.close()


def test_duo_window_covering_context_equals_full_attention():
    """A window longer than the whole context keeps every key: the streaming head is then plain causal
    attention, within tolerance of the same head without labels (its history is split differently)."""
    base = Run(**TINY, chunks=[256, 256], n_decode=3, dist="P", opts=dict(n_slots=2, slot_tokens=128))
    g0, c0 = run_gpu(base)
    c0.close()
    r, lab = duo_run(Run(**TINY, chunks=[256, 256], n_decode=3, dist="P", opts=dict(n_slots=2, slot_tokens=128)),
                     labels=np.ones((1, 2), dtype=np.uint8), n_sink=0, win=100000)
    g1, c1 = run_gpu(r)
    c1.close()
    ref, _ = oracle_duo(r, lab, 0, 100000)
    compare(g1, ref)
    assert (g0[0] - g1[0]).abs().max().item() <= 2e-2


def test_duo_decode_matches_prefill_of_one_more_token():
    a, lab = duo_run(Run(**TINY, chunks=[256, 256, 100], n_decode=1, dist="P", chunk_cap=256), n_sink=8, win=50)
    b, _ = duo_run(Run(**TINY, chunks=[256, 256, 101], n_decode=0, dist="P", chunk_cap=256), n_sink=8, win=50)
    ga, ca = run_gpu(a)
    gb, cb = run_gpu(b)
    assert (ga[0][612] - gb[0][612]).abs().max().item() <= 2e-2
    ca.close()
    cb.close()


def test_duo_deterministic_and_write_kv_prepares_history():
    """hi_write_host_kv fills a streaming head's sink + ring (the bench's way of preparing a long context);
    decoding after it equals decoding after a real prefill, bit for bit."""
    r, lab = duo_run(Run(**TINY, chunks=[256, 256], n_decode=0, dist="P"), labels=np.array([[1, 0]], np.uint8),
                     n_sink=16, win=64)
    from paper_2502_12574_b200.headinfer import HeadInfer
    from synth.cuda import fill_
    outs = []
    for prep in ("prefill", "write"):
        ctx = HeadInfer(1, 4, 2, 64, 520, 256, **r.opts)
        if prep == "prefill":
            run_gpu(r, ctx)
        else:
            q, k, v = synth.gen_qkv(r.seed, r.dist, 0, 0, 512, 4, 2, 64)
            for h in range(2):
                kt = torch.from_numpy(np.ascontiguousarray(k[:, h]).view(np.int16)).view(torch.bfloat16)
                vt = torch.from_numpy(np.ascontiguousarray(v[:, h]).view(np.int16)).view(torch.bfloat16)
                ctx.write_host_kv(0, h, 0, kt, vt)
            ctx.set_seq_len(0, 512)
        o = []
        for t in range(3):
            q = fill_(torch.empty((1, 4, 64), dtype=torch.bfloat16, device="cuda"), r.seed, 0, r.dist, 0, 0, 512 + t)
            k = fill_(torch.empty((1, 2, 64), dtype=torch.bfloat16, device="cuda"), r.seed, 1, r.dist, 0, 0, 512 + t)
            v = fill_(torch.empty((1, 2, 64), dtype=torch.bfloat16, device="cuda"), r.seed, 2, r.dist, 0, 0, 512 + t)
            o.append(ctx.decode(0, q[0], k[0], v[0]).float().cpu())
        outs.append(torch.stack(o))
        ctx.close()
    assert torch.equal(outs[0], outs[1])
