"""Pins for the fp64 oracle (oracle/): against things other than itself.

* textbook brute force (full score matrix + mask + softmax, numpy fp64) and the
  library routine torch SDPA (fp64, explicit bottom-right bool mask, enable_gqa)
* closed forms: single key, uniform scores -> prefix mean,
  two keys -> logistic weights, V == 1 -> exactly 1 (normalisation)
* invariants the paper relies on: chunk invariance, decode(S) ==
  prefill(S+1) last row, kv-head permutation equivariance,
  head-wise == monolithic.
"""
import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import synth
from oracle import attention_rows, dense_attention_np, gqa_attention


def _inputs(seed, dist, n, hq, hkv, d, layer=0):
    return synth.gen_qkv(seed, dist, layer, 0, n, hq, hkv, d)


@settings(max_examples=40, deadline=None)
@given(hkv=st.sampled_from([1, 2, 4]), g=st.sampled_from([1, 2, 4, 8]), d=st.sampled_from([8, 16, 64]),
       n=st.integers(1, 40), q0frac=st.floats(0, 1), dist=st.sampled_from(["U", "P", "S"]),
       seed=st.integers(0, 2**31))
def test_oracle_vs_dense_bruteforce(hkv, g, d, n, q0frac, dist, seed):
    hq = hkv * g
    q, k, v = _inputs(seed, dist, n, hq, hkv, d)
    q0 = int(q0frac * (n - 1))
    got = gqa_attention(q[q0:], k, v, q0)
    ref = dense_attention_np(q[q0:], k, v, q0)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dist", ["U", "P", "S"])
@pytest.mark.parametrize("hq,hkv,d,n,q0", [(4, 2, 64, 48, 0), (8, 2, 32, 33, 17), (32, 8, 128, 20, 5)])
def test_oracle_vs_torch_sdpa_fp64(dist, hq, hkv, d, n, q0):
    q, k, v = _inputs(11, dist, n, hq, hkv, d)
    got = gqa_attention(q[q0:], k, v, q0)
    qt = torch.from_numpy(synth.bf16_to_f64(q[q0:])).permute(1, 0, 2)[None]
    kt = torch.from_numpy(synth.bf16_to_f64(k)).permute(1, 0, 2)[None]
    vt = torch.from_numpy(synth.bf16_to_f64(v)).permute(1, 0, 2)[None]
    # bottom-right (global-position) causal mask, reading R2; NOT is_causal (top-left when Lq != Lk)
    mask = torch.arange(n)[None, :] <= torch.arange(q0, n)[:, None]
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask, enable_gqa=True)
    np.testing.assert_allclose(got, ref[0].permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)


def test_single_key_returns_v0_exactly():
    q, k, v = _inputs(3, "P", 5, 4, 2, 64)
    out = gqa_attention(q[:1], k, v, 0)
    for j in range(4):
        assert np.array_equal(out[0, j], synth.bf16_to_f64(v[0, j // 2]))


def test_v_one_gives_exactly_one():
    q, k, v = _inputs(5, "ONE", 300, 4, 2, 64)
    out = gqa_attention(q, k, v, 0)
    assert np.all(out == 1.0)


def test_uniform_scores_give_prefix_mean():
    q, k, v = _inputs(9, "U", 64, 4, 2, 32)
    q[:] = 0  # q = 0 -> every score 0 -> uniform weights
    out = gqa_attention(q, k, v, 0)
    vf = synth.bf16_to_f64(v)
    prefix_mean = np.cumsum(vf, axis=0) / np.arange(1, 65)[:, None, None]
    for j in range(4):
        np.testing.assert_allclose(out[:, j], prefix_mean[:, j // 2], rtol=0, atol=1e-14)


def test_two_keys_logistic_closed_form():
    q, k, v = _inputs(21, "P", 2, 1, 1, 16)
    qf, kf, vf = (synth.bf16_to_f64(x)[:, 0] for x in (q, k, v))
    s0, s1 = qf[1] @ kf[0] / 4.0, qf[1] @ kf[1] / 4.0
    a1 = 1.0 / (1.0 + np.exp(s0 - s1))
    expect = (1 - a1) * vf[0] + a1 * vf[1]
    got = attention_rows(q[1:2, 0], np.array([1]), k[:, 0], v[:, 0])[0]
    np.testing.assert_allclose(got, expect, rtol=0, atol=1e-15)


def test_dominant_key_selects_its_value():
    d = 64
    q, k, v = _inputs(4, "U", 50, 1, 1, d)
    k[17, 0] = synth.f32_to_bf16_rne(np.full(d, 1.0, np.float32))
    q[:, 0] = synth.f32_to_bf16_rne(np.full(d, 8.0, np.float32))  # logit gap >= 8*64*(1-1)/8 ... >> 1
    out = gqa_attention(q[40:41], k, v, 40)[0, 0]
    np.testing.assert_allclose(out, synth.bf16_to_f64(v[17, 0]), atol=1e-12)


def test_chunk_invariance_bit_exact():
    n, hq, hkv, d = 97, 4, 2, 32
    q, k, v = _inputs(13, "P", n, hq, hkv, d)
    whole = gqa_attention(q, k, v, 0)
    for c in (1, 7, 32, 64):
        parts = [gqa_attention(q[s:s + c], k[:min(n, s + c)], v[:min(n, s + c)], s) for s in range(0, n, c)]
        assert np.array_equal(np.concatenate(parts), whole)


def test_decode_equals_prefill_last_row():
    n, hq, hkv, d = 65, 8, 2, 64
    q, k, v = _inputs(17, "S", n, hq, hkv, d)
    pre = gqa_attention(q, k, v, 0)
    dec = gqa_attention(q[n - 1:], k, v, n - 1)  # decode token at position n-1 attends itself (R3)
    assert np.array_equal(dec[0], pre[n - 1])


def test_kv_head_permutation_equivariance():
    n, hkv, g, d = 40, 4, 2, 16
    q, k, v = _inputs(23, "P", n, hkv * g, hkv, d)
    perm = np.array([2, 0, 3, 1])
    qperm = q.reshape(n, hkv, g, d)[:, perm].reshape(n, hkv * g, d)
    out = gqa_attention(q, k, v, 0)
    outp = gqa_attention(qperm, k[:, perm], v[:, perm], 0)
    assert np.array_equal(outp.reshape(n, hkv, g, d), out.reshape(n, hkv, g, d)[:, perm])


def test_headwise_equals_monolithic():
    # Eq. 9 + concat == one all-heads matrix computation ("exact mathematical equivalence")
    n, hq, hkv, d = 48, 8, 2, 64
    q, k, v = _inputs(29, "P", n, hq, hkv, d)
    headwise = gqa_attention(q, k, v, 0)
    mono = dense_attention_np(q, k, v, 0)
    np.testing.assert_allclose(headwise, mono, rtol=0, atol=1e-12)


def test_bad_arguments_rejected():
    q, k, v = _inputs(1, "U", 4, 1, 1, 8)
    with pytest.raises(RuntimeError):
        attention_rows(q[:1, 0], np.array([4]), k[:, 0], v[:, 0])  # key index out of range
    with pytest.raises(ValueError):
        gqa_attention(q, k[:2], v[:2], 0)
    assert attention_rows(q[:0, 0], np.zeros(0, np.int64), k[:, 0], v[:, 0]).shape == (0, 8)
