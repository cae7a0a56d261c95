"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY -- never imported by the product path)."""
from .oracle import (attention_rows, attention_rows_duo, build, dense_attention_np, duo_gqa_attention,
                     gqa_attention, num_threads)

__all__ = ["attention_rows", "attention_rows_duo", "build", "dense_attention_np", "duo_gqa_attention",
           "gqa_attention", "num_threads"]
