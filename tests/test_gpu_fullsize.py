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

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]

SEED = synth.BASE_SEED


def _gen(tensor, dist, layer, head0, nh, pos0, n, d):
    from synth.cuda import gen_block_cuda
    return gen_block_cuda(SEED, tensor, dist, layer, head0, nh, pos0, n, d)


@pytest.mark.parametrize("dist,opts", [
    ("U", {}),
    ("P", {}),
    ("P", {"head_group": -1}),                                                 # bench.py's default unit size
    ("S", {"head_group": -1, "duo": 0.5}),                                     # NEXT-3 at full size
])
def test_llama8b_128k_sampled_rows_and_host_kv(dist, opts):
    _sampled_rows_and_host_kv(2, 32, 8, 128, 131072, 18944, dist, opts)


def test_llama70b_1m_rank0_of_8_sampled_rows_and_host_kv():
    """configs[4] (Llama-3-70B heads, 1M context, head-sharded over 8 GPUs) as bench.py --emulate-shard 0/8
    runs it: rank 0's kv head 0 and q heads 0-7 (g = 8), chunk 9472, the whole 1M context prefilled."""
    _sampled_rows_and_host_kv(2, 64, 8, 128, 1 << 20, 9472, "P", {}, rank=0, world=8, n_rand=8)


def _sampled_rows_and_host_kv(L, hq, hkv, d, S, c, dist, opts, rank=0, world=1, n_rand=24):
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
    for t in range(n_dec):
        p = S + t
        for layer in range(L):
            q, k, v = (_gen(tt, dist, layer, h0, h, p, 1, d)[0] for tt, h0, h in ((0, q0, hq_loc), (1, kv0, hkv_loc),
                                                                                 (2, kv0, hkv_loc)))
            o = hi.decode(layer, q, k, v).float().cpu().numpy()
            sample.setdefault(layer, []).append((p, o))
    hi.synchronize()
    maxerr, sumerr, cnt = 0.0, 0.0, 0
    for layer in range(L):
        pos = np.array([p for p, _ in sample[layer]])
        got = np.stack([r for _, r in sample[layer]])  # [R, hq_loc, d]
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
    st = hi.stats()
    hi.close()
    assert maxerr <= 2e-2 and sumerr / cnt <= 2e-3, (maxerr, sumerr / cnt)
    assert st["staging_bytes"] <= st["staging_bound_bytes"]
