"""GPU parity for NEXT-4 tensor parallelism ("70B via TP"): W head-sharded contexts, each with its
shard of every layer's weights (paper_2502_12574_b200.layer.shard_layer_weights), run the layer as the three
include/hilayer.h calls hl_attn_partial -> [all-reduce] -> hl_mlp_partial -> [all-reduce] -> hl_residual_add.
The W ranks run one after another in this process (the logical-rank method of tests/test_gpu_hazards.py); the
all-reduce is the test's fp32 sum of the ranks' partials (bench.py uses NCCL / gloo).  Checked: every rank ends
with the same x; the result matches oracle/layer.py (same bar as tests/test_gpu_layer.py); at W = 1 the three
calls are bit-identical to hl_prefill_chunk / hl_decode."""
import numpy as np
import pytest
import torch

import synth
from conftest import cuda_available
from test_gpu_layer import SEED, TINY, check, run_layers_gpu, run_layers_oracle

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]


def run_tp(cfg, chunks, n_decode, world, opts=None):
    from paper_2502_12574_b200.headinfer import HeadInfer
    from paper_2502_12574_b200.layer import HeadInferLayer, shard_layer_weights
    from synth.cuda import fill_matrix_, gen_layer_weights_cuda
    L, H, I, hq, hkv, d = cfg["layers"], cfg["hidden"], cfg["inter"], cfg["q_heads"], cfg["kv_heads"], cfg["d"]
    S = sum(chunks) + n_decode
    his = [HeadInfer(L, hq, hkv, d, S, max(chunks), r, world, **(opts or {})) for r in range(world)]
    lays = [HeadInferLayer(hi, H, I, cfg["theta"], cfg["eps"]) for hi in his]
    full = [gen_layer_weights_cuda(SEED, l, H, I, hq, hkv, d) for l in range(L)]
    ws = [[shard_layer_weights(full[l], hq, hkv, d, I, r, world) for l in range(L)] for r in range(world)]
    out = torch.empty((S, H), dtype=torch.bfloat16, device="cuda")

    def step(xs, decode):
        for l in range(L):
            y = sum(lays[r].attn_partial(l, ws[r][l], xs[r], decode=decode) for r in range(world))
            z = sum(lays[r].mlp_partial(l, ws[r][l], xs[r], y) for r in range(world))
            for r in range(world):
                lays[r].residual_add(xs[r], z)
        for r in range(1, world):
            assert torch.equal(xs[r], xs[0]), "ranks disagree on the replicated hidden states"
        return xs[0]

    pos = 0
    for n in chunks:
        x = fill_matrix_(torch.empty((n, H), dtype=torch.bfloat16, device="cuda"), SEED, synth.TENSOR_X, 0, row0=pos)
        out[pos:pos + n] = step([x.clone() for _ in range(world)], False)
        pos += n
    for _ in range(n_decode):
        x = fill_matrix_(torch.empty((1, H), dtype=torch.bfloat16, device="cuda"), SEED, synth.TENSOR_X, 0, row0=pos)
        out[pos] = step([x.clone() for _ in range(world)], True)[0]
        pos += 1
    torch.cuda.synchronize()
    for lay in lays:
        lay.close()
    for hi in his:
        hi.close()
    return out.float().cpu().numpy().astype(np.float64)


TP = dict(TINY, q_heads=8, kv_heads=4)   # 4 q / 2 kv heads and inter/2 columns per rank at W = 2


@pytest.mark.parametrize("world,opts", [(2, {}), (4, {}), (2, dict(n_slots=2, slot_tokens=64)),
                                        (2, dict(resident_kv_heads=1))])
def test_tp_layers_match_oracle(world, opts):
    chunks, nd = [128, 96, 37], 3
    got = run_tp(TP, chunks, nd, world, opts)
    check(got, run_layers_oracle(TP, sum(chunks) + nd))


def test_tp_world1_bit_identical_to_fused_layer():
    """At W = 1 the three-call form rounds at the same points as the fused GEMM epilogues."""
    chunks, nd = [128, 64], 2
    fused, _ = run_layers_gpu(TP, chunks, nd)
    split = run_tp(TP, chunks, nd, 1)
    assert np.array_equal(fused, split)


def test_tp_llama8b_shape_two_ranks():
    """One Llama-3-8B-shaped layer split over 2 ranks (16 q / 4 kv heads and 7168 intermediate columns each)."""
    cfg = dict(layers=1, hidden=4096, inter=14336, q_heads=32, kv_heads=8, d=128, theta=500000.0, eps=1e-5)
    got = run_tp(cfg, [384, 128], 2, 2)
    check(got, run_layers_oracle(cfg, 514))
