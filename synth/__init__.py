"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic)."""
from .gen import (BASE_SEED, DISTS, TENSOR_K, TENSOR_Q, TENSOR_V, TENSOR_X, bf16_to_f32, bf16_to_f64,
                  f32_to_bf16_rne, gen_block, gen_layer_weights, gen_matrix, gen_qkv, layer_weight_scales,
                  splitmix64, streaming_labels)

__all__ = ["BASE_SEED", "DISTS", "TENSOR_Q", "TENSOR_K", "TENSOR_V", "TENSOR_X", "bf16_to_f32", "bf16_to_f64",
           "f32_to_bf16_rne", "gen_block", "gen_layer_weights", "gen_matrix", "gen_qkv", "layer_weight_scales",
           "splitmix64", "streaming_labels"]
