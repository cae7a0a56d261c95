"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY -- never imported by the product path)."""
from .oracle import attention_rows, build, dense_attention_np, gqa_attention, num_threads

__all__ = ["attention_rows", "build", "dense_attention_np", "gqa_attention", "num_threads"]
