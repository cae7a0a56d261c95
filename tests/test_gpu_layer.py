"""GPU parity for NEXT-4: synthetic Llama decoder layers (include/hilayer.h) around the offloaded attention
path, through the C ABI, against oracle/layer.py (fp64 arithmetic, bf16 storage at the op boundaries,
reading R19) on the same seeded weights and inputs.

Tolerance: both sides round to bf16 at the same nine points; inside an op the GPU accumulates in fp32
(GEMM K up to 14336, attention over the context) where the oracle uses fp64, so a stored value may land one
bf16 ulp away (2^-8 relative) and such flips propagate through the following ops; the attention step also
rounds P to bf16 for its PV MMA (reading R9).  Bound used: relative L2 error <= 1e-2 over the whole output
(observed 3.7e-3 - 5.7e-3 on B200), max-abs <= 1/16 at |y| up to ~7 (2 ulps of the [4, 8) binade;
observed 3/64)."""
import numpy as np
import pytest
import torch

import synth
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]

SEED = 0x4C415952  # "LAYR"
REL_L2, MAX_ABS = 1e-2, 1.0 / 16


def run_layers_gpu(cfg, chunks, n_decode, opts=None):
    from paper_2502_12574_b200.headinfer import HeadInfer
    from paper_2502_12574_b200.layer import HeadInferLayer
    from synth.cuda import fill_matrix_, gen_layer_weights_cuda
    L, H, I, hq, hkv, d = cfg["layers"], cfg["hidden"], cfg["inter"], cfg["q_heads"], cfg["kv_heads"], cfg["d"]
    S = sum(chunks) + n_decode
    hi = HeadInfer(L, hq, hkv, d, S, max(chunks), **(opts or {}))
    lay = HeadInferLayer(hi, H, I, cfg["theta"], cfg["eps"])
    ws = [gen_layer_weights_cuda(SEED, l, H, I, hq, hkv, d) for l in range(L)]
    out = torch.empty((S, H), dtype=torch.bfloat16, device="cuda")
    pos = 0
    for n in chunks:
        x = fill_matrix_(torch.empty((n, H), dtype=torch.bfloat16, device="cuda"), SEED, synth.TENSOR_X, 0, row0=pos)
        for l in range(L):
            lay.prefill_chunk(l, ws[l], x)
        out[pos:pos + n] = x
        pos += n
    for _ in range(n_decode):
        x = fill_matrix_(torch.empty((1, H), dtype=torch.bfloat16, device="cuda"), SEED, synth.TENSOR_X, 0, row0=pos)[0]
        for l in range(L):
            lay.decode(l, ws[l], x)
        out[pos] = x
        pos += 1
    torch.cuda.synchronize()
    st = hi.stats()
    lay.close()
    hi.close()
    return out.float().cpu().numpy().astype(np.float64), st


def run_layers_oracle(cfg, S):
    from oracle.layer import layer_forward, weights_f64
    x = synth.bf16_to_f64(synth.gen_matrix(SEED, synth.TENSOR_X, 0, S, cfg["hidden"]))
    for l in range(cfg["layers"]):
        w = weights_f64(synth.gen_layer_weights(SEED, l, cfg["hidden"], cfg["inter"], cfg["q_heads"], cfg["kv_heads"],
                                                cfg["d"]))
        x = layer_forward(x, w, cfg["q_heads"], cfg["kv_heads"], cfg["d"], cfg["theta"], cfg["eps"])
    return x


def check(got, ref):
    assert np.all(np.isfinite(got))
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    mx = float(np.abs(got - ref).max())
    print(f"rel_l2={rel:.3e} max_abs={mx:.3e} max|ref|={np.abs(ref).max():.2f}")
    assert rel <= REL_L2, rel
    assert mx <= MAX_ABS, mx
    return rel, mx


TINY = dict(layers=2, hidden=256, inter=512, q_heads=4, kv_heads=2, d=64, theta=10000.0, eps=1e-5)


@pytest.mark.parametrize("opts", [dict(), dict(n_slots=2, slot_tokens=64), dict(resident_kv_heads=2),
                                  dict(head_group=2)])
def test_layer_tiny_two_layers(opts):
    """Two stacked layers (layer 1 eats layer 0's GPU output): ragged chunks, then decodes; offloaded with
    several slot geometries, partially resident, grouped."""
    chunks, nd = [128, 128, 37], 3
    got, st = run_layers_gpu(TINY, chunks, nd, opts)
    ref = run_layers_oracle(TINY, sum(chunks) + nd)
    check(got, ref)


@pytest.mark.parametrize("g,d", [(1, 64), (8, 128)])
def test_layer_gqa_and_head_dim(g, d):
    cfg = dict(layers=1, hidden=512, inter=768, q_heads=2 * g, kv_heads=2, d=d, theta=500000.0, eps=1e-6)
    got, _ = run_layers_gpu(cfg, [200, 100], 2)
    ref = run_layers_oracle(cfg, 302)
    check(got, ref)


def test_layer_llama8b_shape():
    """One Llama-3-8B-shaped layer (4096 hidden, 14336 inter, 32q/8kv, d128, theta 5e5)."""
    cfg = dict(layers=1, hidden=4096, inter=14336, q_heads=32, kv_heads=8, d=128, theta=500000.0, eps=1e-5)
    got, _ = run_layers_gpu(cfg, [384, 256], 2)
    ref = run_layers_oracle(cfg, 642)
    check(got, ref)


def test_layer_rejects_bad_arguments():
    from paper_2502_12574_b200._lib import HIError
    from paper_2502_12574_b200.headinfer import HeadInfer
    from paper_2502_12574_b200.layer import HeadInferLayer
    hi = HeadInfer(1, 4, 2, 64, 256, 64)
    with pytest.raises(HIError):
        HeadInferLayer(hi, 100, 512)          # hidden not a multiple of 64
    lay = HeadInferLayer(hi, 256, 512)
    w = {k: torch.zeros(1, dtype=torch.bfloat16, device="cuda") for k in ("attn_norm",)}
    with pytest.raises((ValueError, KeyError)):
        lay.prefill_chunk(0, w, torch.zeros((8, 256), dtype=torch.bfloat16, device="cuda"))
    lay.close()
    hi.close()
