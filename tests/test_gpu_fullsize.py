"""Full-size parity: the Llama-3-8B head geometry at the 128K context of BASELINE.json configs[1],
in bench.py's launch configuration (chunk 18944, 4 staging slots of max_ctx/4 tokens, head groups as
bench.py picks them; also with 50% duo streaming heads, NEXT-3), on sampled
rows the oracle computes one by one, plus a bit-exact host-KV scan.  Layers are reduced to 2 (every
layer call runs the identical launch sequence)."""
import numpy as np
import pytest
import torch

import synth
from conftest import cuda_available
from hi_harness import TOL_MAX_ABS, TOL_MEAN_ABS, TOL_REL_L2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]

SEED = synth.BASE_SEED


def _gen(tensor, dist, layer, head0, nh, pos0, n, d):
    from synth.cuda import gen_block_cuda
    return gen_block_cuda(SEED, tensor, dist, layer, head0, nh, pos0, n, d)


def assert_parity(e):
    assert e["max_abs"] <= TOL_MAX_ABS and e["mean_abs"] <= TOL_MEAN_ABS, e
    assert e["rel_l2_max"] <= TOL_REL_L2, e


@pytest.mark.parametrize("dist,opts", [
    ("U", {}),
    ("P", {}),
    ("P", {"head_group": -1}),                                                 # bench.py's default unit size
    ("S", {"head_group": -1, "duo": 0.5}),                                     # NEXT-3 at full size
])
def test_llama8b_128k_sampled_rows_and_host_kv(dist, opts):
    assert_parity(_sampled_rows_and_host_kv(2, 32, 8, 128, 131072, 18944, dist, opts))


def test_llama8b_1m_headline_geometry_peaked():
    """The HEADLINE geometry (bench.py's 8B-1M launch configuration): 32 q / 8 kv heads (g = 4), head group 2,
    the default one-head staging ring (4 slots of 131072-key blocks per 2-head unit), chunk 18944 (the 1M
    context ends in a ragged 6464-token chunk), the whole 1M context prefilled for 2 layers, under the peaked
    distribution P (max-dominated rows: online-softmax rescaling across the 8 history blocks and the chunk
    segment), then 3 decode steps; sampled rows of EVERY q head against the oracle (max-abs, mean-abs,
    relative L2 per (layer, q head)) and a bit-exact scan of the whole host KV store."""
    e = _sampled_rows_and_host_kv(2, 32, 8, 128, 1 << 20, 18944, "P", {"head_group": 2}, n_rand=16,
                                  expect_slot_tokens=131072)
    assert_parity(e)


def test_llama70b_1m_rank0_of_8_sampled_rows_and_host_kv():
    """configs[4] (Llama-3-70B heads, 1M context, head-sharded over 8 GPUs) as bench.py --emulate-shard 0/8
    runs it: rank 0's kv head 0 and q heads 0-7 (g = 8), chunk 9472, the whole 1M context prefilled."""
    assert_parity(_sampled_rows_and_host_kv(2, 64, 8, 128, 1 << 20, 9472, "P", {}, rank=0, world=8, n_rand=8))


def test_negative_control_scaled_output_fails_only_relative_bar():
    """Negative control (SPEC.md S:L401 idea): the GPU rows at U/128K, scaled by 0.98, still pass the absolute
    bounds (|o| ~ 2e-3 there) but must FAIL the relative-L2 bar -- the check the round-1 tests lacked."""
    e = _sampled_rows_and_host_kv(1, 32, 8, 128, 131072, 18944, "U", {}, n_rand=8, scale=0.98)
    assert e["max_abs"] <= TOL_MAX_ABS and e["mean_abs"] <= TOL_MEAN_ABS, e
    assert e["rel_l2_max"] > TOL_REL_L2, e


def test_negative_control_dropped_history_block_fails():
    """Negative control: HI_FLAG_FAULT_SKIP_BLOCK drops the attention launch over the first history block of
    every unit (a mis-merge of whole blocks).  At U/128K the absolute bounds cannot see it; the relative-L2 bar
    must."""
    from paper_2502_12574_b200._lib import HI_FLAG_FAULT_SKIP_BLOCK
    e = _sampled_rows_and_host_kv(1, 32, 8, 128, 131072, 18944, "U", {"flags": HI_FLAG_FAULT_SKIP_BLOCK}, n_rand=8,
                                  check_decode=False)
    assert e["rel_l2_max"] > TOL_REL_L2, e


def _sampled_rows_and_host_kv(L, hq, hkv, d, S, c, dist, opts, rank=0, world=1, n_rand=24, scale=1.0,
                              check_decode=True, expect_slot_tokens=None):
    from oracle import attention_rows, attention_rows_duo
    from paper_2502_12574_b200.headinfer import HeadInfer
    n_dec = 3
    g = hq // hkv
    hkv_loc, hq_loc = hkv // world, hq // world
    kv0, q0 = rank * hkv_loc, rank * hq_loc   # global head indices of this rank's shard
    opts = dict(opts)
    labels = None
    n_sink, win = 64, 256
    if opts.pop("duo", 0):
        labels = synth.streaming_labels(SEED, L, hkv, 0.5)
        opts.update(streaming_heads=labels.tolist(), duo_sink=n_sink, duo_window=win)
    hi = HeadInfer(L, hq, hkv, d, S + n_dec, c, rank, world, **opts)
    sample = {}  # (layer) -> list of (pos, out row [hq_loc, d])
    rng = np.random.default_rng(0)
    chunk_starts = list(range(0, S, c))
    want = set()
    for s0 in chunk_starts:  # first/last row of every chunk, plus random rows
        want.update([s0, min(S, s0 + c) - 1])
    want.update(rng.integers(0, S, n_rand).tolist())
    for s0 in chunk_starts:
        n = min(c, S - s0)
        for layer in range(L):
            Q, K, V = (_gen(t, dist, layer, h0, h, s0, n, d) for t, h0, h in ((0, q0, hq_loc), (1, kv0, hkv_loc),
                                                                               (2, kv0, hkv_loc)))
            out = hi.prefill_chunk(layer, Q, K, V)
            rows = [p for p in want if s0 <= p < s0 + n]
            if rows:
                o = out[torch.tensor([p - s0 for p in rows], device="cuda")].float().cpu().numpy()
                for p, r in zip(rows, o):
                    sample.setdefault(layer, []).append((p, r))
    for t in range(n_dec if check_decode else 0):
        p = S + t
        for layer in range(L):
            q, k, v = (_gen(tt, dist, layer, h0, h, p, 1, d)[0] for tt, h0, h in ((0, q0, hq_loc), (1, kv0, hkv_loc),
                                                                                 (2, kv0, hkv_loc)))
            o = hi.decode(layer, q, k, v).float().cpu().numpy()
            sample.setdefault(layer, []).append((p, o))
    hi.synchronize()
    if not check_decode:
        n_dec = 0
    maxerr, sumerr, cnt = 0.0, 0.0, 0
    rel = {}
    for layer in range(L):
        pos = np.array([p for p, _ in sample[layer]])
        got = np.stack([r for _, r in sample[layer]]) * scale  # [R, hq_loc, d]
        qpos = np.concatenate([synth.gen_block(SEED, 0, dist, layer, q0, hq_loc, int(p), 1, d) for p in pos])
        for hl in range(hkv_loc):
            h = kv0 + hl   # global kv head
            k = _gen(1, dist, layer, h, 1, 0, S + n_dec, d)[:, 0].cpu().view(torch.int16).numpy().view(np.uint16)
            v = _gen(2, dist, layer, h, 1, 0, S + n_dec, d)[:, 0].cpu().view(torch.int16).numpy().view(np.uint16)
            streaming = labels is not None and labels[layer][h]
            # host KV store must hold exactly these bytes (a streaming head: its sink and its window)
            spans = [(0, n_sink), (S + n_dec - win, S + n_dec)] if streaming else [(0, S + n_dec)]
            for lo, hi_ in spans:
                hk, hv = hi.read_host_kv(layer, hl, lo, hi_ - lo)
                assert np.array_equal(hk.view(torch.int16).numpy().view(np.uint16), k[lo:hi_]), (layer, h)
                assert np.array_equal(hv.view(torch.int16).numpy().view(np.uint16), v[lo:hi_]), (layer, h)
            for jl in range(hl * g, (hl + 1) * g):   # local q head; global q head q0 + jl
                if streaming:
                    ref = attention_rows_duo(qpos[:, jl], pos, k, v, n_sink, win)
                else:
                    ref = attention_rows(qpos[:, jl], pos, k, v)
                err = np.abs(got[:, jl] - ref)
                maxerr = max(maxerr, float(err.max()))
                sumerr += float(err.sum())
                cnt += err.size
                rel[(layer, q0 + jl)] = float(np.linalg.norm(got[:, jl] - ref) / max(np.linalg.norm(ref), 1e-300))
    st = hi.stats()
    hi.close()
    assert st["staging_bytes"] <= st["staging_bound_bytes"]
    if expect_slot_tokens is not None:
        assert st["slot_tokens"] == expect_slot_tokens, st
    worst = max(rel, key=rel.get)
    assert len({k[1] for k in rel}) == hq_loc   # every q head of the shard checked
    return {"max_abs": maxerr, "mean_abs": sumerr / cnt, "rel_l2_max": rel[worst], "worst": worst,
            "rows": int(cnt // d)}
