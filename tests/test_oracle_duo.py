"""Pins for the duo-attention (NEXT-3) oracle: streaming heads attend the sink tokens and a window of
recent tokens (§4, App. D; reading R18 in DESIGN.md).  Pinned against
things other than the oracle itself:

* textbook brute force (dense_attention_np: full score matrix, explicit sink|window & causal mask,
  row softmax) and torch SDPA (fp64, the same boolean mask, enable_gqa);
* explicit gather: a streaming row equals plain attention of the same query over the gathered key
  list (the keys it keeps, in order) -- the definition of truncating a head's cache;
* closed forms: n_sink = 0, win = 1 -> each row returns its own value exactly; V == 1 -> exactly 1;
  a window covering the whole context reduces to full causal attention; retrieval heads unchanged.
"""
import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import synth
from oracle import attention_rows, attention_rows_duo, dense_attention_np, duo_gqa_attention, gqa_attention


@settings(max_examples=40, deadline=None)
@given(hkv=st.sampled_from([1, 2, 4]), g=st.sampled_from([1, 2, 4]), d=st.sampled_from([8, 16, 64]),
       n=st.integers(1, 48), q0frac=st.floats(0, 1), n_sink=st.integers(0, 6), win=st.integers(1, 20),
       dist=st.sampled_from(["U", "P", "S"]), seed=st.integers(0, 2**31), lab=st.integers(0, 15))
def test_duo_vs_dense_bruteforce(hkv, g, d, n, q0frac, n_sink, win, dist, seed, lab):
    hq = hkv * g
    q, k, v = synth.gen_qkv(seed, dist, 0, 0, n, hq, hkv, d)
    q0 = int(q0frac * (n - 1))
    streaming = [(lab >> h) & 1 == 1 for h in range(hkv)]
    got = duo_gqa_attention(q[q0:], k, v, q0, streaming, n_sink, win)
    ref = dense_attention_np(q[q0:], k, v, q0, streaming, n_sink, win)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n_sink,win", [(4, 16), (0, 7), (64, 960)])
def test_duo_vs_torch_sdpa_fp64(n_sink, win):
    n, hq, hkv, d, q0 = 1100, 4, 2, 64, 1000
    q, k, v = synth.gen_qkv(7, "S", 0, 0, n, hq, hkv, d)
    got = duo_gqa_attention(q[q0:], k, v, q0, [True, True], n_sink, win)
    qt = torch.from_numpy(synth.bf16_to_f64(q[q0:])).permute(1, 0, 2)[None]
    kt = torch.from_numpy(synth.bf16_to_f64(k)).permute(1, 0, 2)[None]
    vt = torch.from_numpy(synth.bf16_to_f64(v)).permute(1, 0, 2)[None]
    kp, qp = torch.arange(n)[None, :], torch.arange(q0, n)[:, None]
    mask = (kp <= qp) & ((kp < n_sink) | (kp > qp - win))
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask, enable_gqa=True)
    np.testing.assert_allclose(got, ref[0].permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)


def test_streaming_row_equals_attention_over_kept_keys():
    n, d, n_sink, win = 300, 64, 5, 30
    q, k, v = synth.gen_qkv(9, "U", 0, 0, n, 1, 1, d)
    rows = np.array([0, 3, 4, 5, 34, 35, 36, 299], dtype=np.int64)
    got = attention_rows_duo(q[rows, 0], rows, k[:, 0], v[:, 0], n_sink, win)
    for r, p in enumerate(rows):
        keep = [i for i in range(p + 1) if i < n_sink or i > p - win]
        ref = attention_rows(q[p:p + 1, 0], np.array([len(keep) - 1]), k[keep, 0], v[keep, 0])
        np.testing.assert_array_equal(got[r], ref[0])


def test_window_one_no_sink_returns_own_value_exactly():
    n, d = 50, 64
    q, k, v = synth.gen_qkv(2, "P", 0, 0, n, 2, 1, d)
    out = duo_gqa_attention(q, k, v, 0, [True], 0, 1)
    for p in range(n):
        for j in range(2):
            assert np.array_equal(out[p, j], synth.bf16_to_f64(v[p, 0]))


def test_v_one_gives_exactly_one():
    q, k, v = synth.gen_qkv(5, "ONE", 0, 0, 200, 4, 2, 64)
    out = duo_gqa_attention(q, k, v, 0, [True, False], 3, 17)
    assert np.all(out == 1.0)


def test_full_window_reduces_to_causal_and_retrieval_heads_unchanged():
    n, q0 = 120, 40
    q, k, v = synth.gen_qkv(4, "S", 0, 0, n, 4, 2, 32)
    full = gqa_attention(q[q0:], k, v, q0)
    np.testing.assert_array_equal(duo_gqa_attention(q[q0:], k, v, q0, [True, True], 0, n), full)
    np.testing.assert_array_equal(duo_gqa_attention(q[q0:], k, v, q0, [False, False], 4, 8), full)
    mixed = duo_gqa_attention(q[q0:], k, v, q0, [False, True], 4, 8)
    np.testing.assert_array_equal(mixed[:, :2], full[:, :2])
    assert not np.allclose(mixed[:, 2:], full[:, 2:])
