"""Seeded generator: numpy twin vs the pure-Python-int golden bits (CPU)."""
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "synth_golden.txt")


def _cases():
    out = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            s, t, dist, layer, head, pos, dim, bits = line.split()
            out.append((int(s), int(t), dist, int(layer), int(head), int(pos), int(dim), int(bits, 16)))
    return out


@pytest.mark.parametrize("case", _cases())
def test_numpy_generator_matches_golden(case):
    seed, t, dist, layer, head, pos, dim, bits = case
    blk = synth.gen_block(seed, t, dist, layer, head, 1, pos, 1, max(dim + 1, 1))
    assert int(blk[0, 0, dim]) == bits


def test_generator_block_consistency():
    # a sub-block equals the matching slice of a larger block (pure coordinate function)
    big = synth.gen_block(7, synth.TENSOR_K, "U", 3, 0, 8, 100, 50, 64)
    sub = synth.gen_block(7, synth.TENSOR_K, "U", 3, 2, 3, 120, 10, 64)
    assert np.array_equal(big[20:30, 2:5], sub)


def test_generator_range_and_distribution():
    x = synth.bf16_to_f64(synth.gen_block(1, synth.TENSOR_Q, "U", 0, 0, 4, 0, 4096, 128))
    assert x.min() >= -1.0 and x.max() <= 1.0
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1 / np.sqrt(3)) < 0.01
    xp = synth.bf16_to_f64(synth.gen_block(1, synth.TENSOR_Q, "P", 0, 0, 4, 0, 4096, 128))
    assert np.array_equal(xp, 16 * x)  # power-of-two scale commutes with RNE
    xs = synth.bf16_to_f64(synth.gen_block(1, synth.TENSOR_Q, "S", 0, 0, 4, 0, 64, 128))
    assert xs.min() >= 0.0
    ks = synth.bf16_to_f64(synth.gen_block(1, synth.TENSOR_K, "S", 0, 0, 4, 0, 4, 128))
    assert np.all(ks[0] == 1.0) and not np.all(ks[1] == 1.0)
    v1 = synth.bf16_to_f64(synth.gen_block(1, synth.TENSOR_V, "ONE", 0, 0, 2, 0, 8, 64))
    assert np.all(v1 == 1.0)


def test_bf16_rne_ties():
    # 1 + 2^-8 is a tie between 1.0 and 1+2^-7: RNE keeps the even mantissa (1.0)
    f = np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -1.5], dtype=np.float32)
    assert list(synth.f32_to_bf16_rne(f)) == [0x3F80, 0x3F82, 0xBFC0]


def test_streaming_labels_deterministic_and_balanced():
    a = synth.streaming_labels(7, 32, 8, 0.5)
    b = synth.streaming_labels(7, 32, 8, 0.5)
    assert a.dtype == np.uint8 and a.shape == (32, 8)
    assert np.array_equal(a, b)
    assert np.all(a.sum(axis=1) == 4)
    assert not np.array_equal(a, synth.streaming_labels(8, 32, 8, 0.5))
    assert synth.streaming_labels(1, 2, 8, 0.0).sum() == 0 and synth.streaming_labels(1, 2, 8, 1.0).sum() == 16
