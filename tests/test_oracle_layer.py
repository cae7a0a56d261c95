"""Pins for the NEXT-4 layer oracle (oracle/layer.py), each against something other than the oracle:

* transformers' LlamaDecoderLayer (library routine), fp64, SDPA attention, torch's rms_norm, same
  weights, with fp64 RoPE tables passed in (HF computes its own in fp32, and its RMSNorm / eager softmax
  upcast to fp32) -- the unrounded oracle must agree to 1e-11;
* closed forms: RMSNorm of a constant row is gamma * sign(c) (eps -> 0); RoPE is a rotation (norms kept)
  and q_m . k_n depends only on m - n; RoPE at position 0 is the identity; silu(0) = 0;
* bf16_round against torch's bf16 conversion (an independent RNE implementation) on fp32-exact inputs
  and on hand-made ties;
* the bf16-boundary variant stays within the bf16 error bound of the unrounded one.
"""
import numpy as np
import pytest
import torch

import synth
from oracle.layer import bf16_round, layer_forward, rms_norm, rope, silu, weights_f64

CFG = dict(hidden=256, inter=512, q_heads=4, kv_heads=2, d=64, theta=10000.0, eps=1e-5)


def _inputs(S, cfg=CFG, seed=11, layer=0):
    wb = synth.gen_layer_weights(seed, layer, cfg["hidden"], cfg["inter"], cfg["q_heads"], cfg["kv_heads"], cfg["d"])
    x = synth.bf16_to_f64(synth.gen_matrix(seed, synth.TENSOR_X, 0, S, cfg["hidden"]))
    return x, weights_f64(wb)


def test_unrounded_layer_matches_transformers_llama_decoder_layer():
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaDecoderLayer
    c = CFG
    S = 48
    x, w = _inputs(S)
    conf = LlamaConfig(hidden_size=c["hidden"], intermediate_size=c["inter"], num_attention_heads=c["q_heads"],
                       num_key_value_heads=c["kv_heads"], head_dim=c["d"], rms_norm_eps=c["eps"],
                       rope_theta=c["theta"], attention_bias=False, mlp_bias=False, hidden_act="silu")
    conf._attn_implementation = "sdpa"   # torch SDPA: fp64 throughout (eager's softmax runs in fp32)
    lay = LlamaDecoderLayer(conf, layer_idx=0).double().eval()
    # LlamaRMSNorm upcasts to fp32 internally; use torch's own rms_norm (a library routine) in fp64 instead
    for norm in (lay.input_layernorm, lay.post_attention_layernorm):
        norm.forward = (lambda n: lambda h: torch.nn.functional.rms_norm(h, (h.shape[-1],), n.weight,
                                                                         n.variance_epsilon))(norm)
    qd, kd = c["q_heads"] * c["d"], c["kv_heads"] * c["d"]
    with torch.no_grad():
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        lay.input_layernorm.weight.copy_(T(w["attn_norm"]))
        lay.post_attention_layernorm.weight.copy_(T(w["mlp_norm"]))
        lay.self_attn.q_proj.weight.copy_(T(w["w_qkv"][:qd]))
        lay.self_attn.k_proj.weight.copy_(T(w["w_qkv"][qd:qd + kd]))
        lay.self_attn.v_proj.weight.copy_(T(w["w_qkv"][qd + kd:]))
        lay.self_attn.o_proj.weight.copy_(T(w["w_o"]))
        lay.mlp.gate_proj.weight.copy_(T(w["w_gate_up"][:c["inter"]]))
        lay.mlp.up_proj.weight.copy_(T(w["w_gate_up"][c["inter"]:]))
        lay.mlp.down_proj.weight.copy_(T(w["w_down"]))
        inv = c["theta"] ** (-(2.0 * np.arange(c["d"] // 2)) / c["d"])
        ang = np.arange(S)[:, None] * inv[None, :]
        emb = np.concatenate([ang, ang], axis=-1)
        cos, sin = T(np.cos(emb))[None], T(np.sin(emb))[None]
        mask = torch.full((S, S), float("-inf"), dtype=torch.float64).triu(1)[None, None]
        out = lay(T(x)[None], attention_mask=mask, position_embeddings=(cos, sin))
        out = out[0] if isinstance(out, tuple) else out
    ref = out[0].numpy()
    got = layer_forward(x, w, c["q_heads"], c["kv_heads"], c["d"], c["theta"], c["eps"], bf16_boundaries=False)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-11)


def test_rmsnorm_constant_row_and_scaling():
    g = np.linspace(-1, 1, 64)
    for cval in (3.0, -0.25):
        out = rms_norm(np.full((1, 64), cval), g, 0.0)[0]
        np.testing.assert_allclose(out, g * np.sign(cval), rtol=0, atol=1e-15)
        # eps inside the root: a constant row c gives gamma * c / sqrt(c^2 + eps)
        out = rms_norm(np.full((1, 64), cval), g, 0.5)[0]
        np.testing.assert_allclose(out, g * cval / np.sqrt(cval * cval + 0.5), rtol=0, atol=1e-15)
    x = np.random.default_rng(0).standard_normal((5, 64))
    np.testing.assert_allclose(rms_norm(7.0 * x, g, 0.0), rms_norm(x, g, 0.0), atol=1e-13)


def test_rope_is_a_relative_rotation():
    rng = np.random.default_rng(1)
    d, theta = 64, 500000.0
    q = rng.standard_normal((1, 1, d))
    k = rng.standard_normal((1, 1, d))
    np.testing.assert_array_equal(rope(q, np.array([0]), theta), q)       # position 0: identity
    for p in (1, 17, 1 << 20):                                          # a rotation keeps norms
        assert np.linalg.norm(rope(q, np.array([p]), theta)) == pytest.approx(np.linalg.norm(q), rel=1e-13)
    dots = []
    for m in (5, 1000, 123456):                                          # q_m . k_n depends on m - n only
        qm, kn = rope(q, np.array([m]), theta), rope(k, np.array([m - 3]), theta)
        dots.append(float((qm * kn).sum()))
    np.testing.assert_allclose(dots, dots[0], rtol=0, atol=1e-9)


def test_silu_closed_forms():
    assert silu(np.array(0.0)) == 0.0
    np.testing.assert_allclose(silu(np.array([40.0, -40.0])), [40.0, -40.0 * np.exp(-40.0)], rtol=1e-12)


def test_bf16_round_matches_torch_rne():
    rng = np.random.default_rng(2)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 20, 100000))).astype(np.float32).astype(np.float64)
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(bf16_round(x), ref)
    # ties: 1 + 2^-8 sits halfway between 1 and 1 + 2^-7 -> even (1); 1 + 3*2^-8 -> 1 + 2^-6
    np.testing.assert_array_equal(bf16_round(np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8)])),
                                  [1.0, 1 + 2 ** -6, -1.0])


def test_bf16_boundaries_stay_within_rounding_error():
    c = CFG
    x, w = _inputs(64)
    a = layer_forward(x, w, c["q_heads"], c["kv_heads"], c["d"], c["theta"], c["eps"], bf16_boundaries=True)
    b = layer_forward(x, w, c["q_heads"], c["kv_heads"], c["d"], c["theta"], c["eps"], bf16_boundaries=False)
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert 1e-4 < rel < 2e-2, rel  # rounding happened, and stays of the order of a few bf16 ulps


def test_layer_is_causal_and_chunk_free():
    """Outputs of the first rows do not depend on later rows (what lets the GPU run it chunk by chunk)."""
    c = CFG
    x, w = _inputs(40)
    full = layer_forward(x, w, c["q_heads"], c["kv_heads"], c["d"], c["theta"], c["eps"])
    part = layer_forward(x[:25], w, c["q_heads"], c["kv_heads"], c["d"], c["theta"], c["eps"])
    np.testing.assert_array_equal(full[:25], part)


def test_gpu_weight_twin_is_pinned_to_gen_matrix_layout():
    """gen_matrix(r, c) is the generator coordinate (head = c // 128, pos = r, dim = c % 128), scaled by an
    exact power of two."""
    m = synth.gen_matrix(5, synth.TENSOR_X, 2, 3, 256, -5, row0=7)
    blk = synth.gen_block(5, synth.TENSOR_X, "U", 2, 0, 2, 7, 3, 128)
    np.testing.assert_array_equal(synth.bf16_to_f64(m), synth.bf16_to_f64(blk.reshape(3, 256)) * 2.0 ** -5)
