"""ctypes loader for libheadinfer.so (the C ABI declared in include/headinfer.h).

Fails loudly when the native library is missing: there is no CPU or eager fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libheadinfer.so")
# experiments only (tools/ab_prefill.sh): load a variant build of the same sources instead
if os.environ.get("HI_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, "build", "variants", f"libheadinfer_{os.environ['HI_LIB_VARIANT']}.so")

HI_OK, HI_EINVAL, HI_ESHAPE, HI_ECAPACITY, HI_ENOMEM_HOST, HI_ENOMEM_DEV, HI_ECUDA, HI_ESTATE = range(8)
STATUS_NAMES = ["HI_OK", "HI_EINVAL", "HI_ESHAPE", "HI_ECAPACITY", "HI_ENOMEM_HOST", "HI_ENOMEM_DEV",
                "HI_ECUDA", "HI_ESTATE"]
HI_FLAG_POISON_SLOTS = 0x1
HI_FLAG_NO_HUGEPAGE = 0x2
HI_FLAG_SERIALIZE = 0x4
HI_FLAG_TIMING = 0x8
HI_FLAG_MMA_SYNC_PREFILL = 0x10
HI_FLAG_PREFILL_2CTA = 0x20
HI_FLAG_PREFILL_TC1 = 0x40
HI_FLAG_JITTER = 0x80
HI_FLAG_FAULT_SKIP_RAW = 0x100
HI_FLAG_FAULT_LAUNCH = 0x200
HI_FLAG_FAULT_TRAP = 0x400
HI_FLAG_FAULT_SKIP_BLOCK = 0x800
HI_FLAG_PREFILL_PSMEM = 0x1000
HI_RESIDENT_AUTO = -1
HI_GROUP_AUTO = -1
HI_GROUP_PAPER = -2

# every symbol include/headinfer.h and include/hilayer.h declare (checked by tests/test_abi.py)
EXPORTS = ["hi_init", "hi_init_ex", "hi_prefill_chunk", "hi_decode", "hi_free", "hi_read_host_kv",
           "hi_write_host_kv", "hi_seq_len", "hi_set_seq_len", "hi_get_stats", "hi_synchronize",
           "hi_status_str", "hi_last_error",
           "hl_create", "hl_prefill_chunk", "hl_decode", "hl_free", "hl_last_error", "hl_gemm",
           "hl_attn_partial", "hl_mlp_partial", "hl_residual_add"]


class hi_options(ctypes.Structure):
    _fields_ = [("n_slots", ctypes.c_int), ("slot_tokens", ctypes.c_int64), ("device", ctypes.c_int),
                ("flags", ctypes.c_int), ("numa_policy", ctypes.c_int), ("numa_node", ctypes.c_int),
                ("resident_kv_heads", ctypes.c_int), ("head_group", ctypes.c_int),
                ("streaming_heads", ctypes.c_void_p), ("duo_sink", ctypes.c_int), ("duo_window", ctypes.c_int)]


class hl_weights(ctypes.Structure):
    """include/hilayer.h: one decoder layer's weights (device pointers, bf16, row-major [out, in])."""
    _fields_ = [("attn_norm", ctypes.c_void_p), ("w_qkv", ctypes.c_void_p), ("w_o", ctypes.c_void_p),
                ("mlp_norm", ctypes.c_void_p), ("w_gate_up", ctypes.c_void_p), ("w_down", ctypes.c_void_p)]


class hi_stats(ctypes.Structure):
    _fields_ = [("host_store_bytes", ctypes.c_int64), ("staging_bytes", ctypes.c_int64),
                ("staging_bound_bytes", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("prefill_calls", ctypes.c_int64), ("decode_calls", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64),
                ("prefill_attn_ms", ctypes.c_double), ("prefill_attn_flops", ctypes.c_double),
                ("prefill_attn_launches", ctypes.c_int64), ("decode_attn_ms", ctypes.c_double),
                ("decode_attn_bytes", ctypes.c_double), ("decode_attn_launches", ctypes.c_int64),
                ("init_seconds", ctypes.c_double),
                ("numa_node", ctypes.c_int), ("n_slots", ctypes.c_int), ("slot_tokens", ctypes.c_int64),
                ("resident_kv_heads", ctypes.c_int), ("resident_bytes", ctypes.c_int64),
                ("head_group", ctypes.c_int),
                ("streaming_kv_heads", ctypes.c_int), ("streaming_bytes", ctypes.c_int64),
                ("h2d_copy_ms", ctypes.c_double), ("d2h_copy_ms", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load libheadinfer.so (raises if it was not built -- run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2502_12574_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64, VP = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
    lib.hi_init.argtypes = [I, I, I, I, I64, I, I, I, ctypes.POINTER(P)]
    lib.hi_init_ex.argtypes = [I, I, I, I, I64, I, I, I, ctypes.POINTER(hi_options), ctypes.POINTER(P)]
    lib.hi_prefill_chunk.argtypes = [P, I, VP, VP, VP, VP, I, VP]
    lib.hi_decode.argtypes = [P, I, VP, VP, VP, VP, VP]
    lib.hi_free.argtypes = [P]
    lib.hi_read_host_kv.argtypes = [P, I, I, I64, I64, VP, VP]
    lib.hi_write_host_kv.argtypes = [P, I, I, I64, I64, VP, VP, I]
    lib.hi_seq_len.argtypes = [P, I]
    lib.hi_seq_len.restype = I64
    lib.hi_set_seq_len.argtypes = [P, I, I64]
    lib.hi_get_stats.argtypes = [P, ctypes.POINTER(hi_stats)]
    lib.hi_synchronize.argtypes = [P]
    lib.hi_status_str.argtypes = [I]
    lib.hi_status_str.restype = ctypes.c_char_p
    lib.hi_last_error.argtypes = [P]
    lib.hi_last_error.restype = ctypes.c_char_p
    lib.hl_create.argtypes = [P, I, I, ctypes.c_double, ctypes.c_float, ctypes.POINTER(P)]
    lib.hl_prefill_chunk.argtypes = [P, I, ctypes.POINTER(hl_weights), VP, I, VP]
    lib.hl_decode.argtypes = [P, I, ctypes.POINTER(hl_weights), VP, VP]
    lib.hl_free.argtypes = [P]
    lib.hl_gemm.argtypes = [VP, VP, VP, I, I, I, I, VP]
    lib.hl_gemm.restype = I
    lib.hl_attn_partial.argtypes = [P, I, ctypes.POINTER(hl_weights), VP, I, I, VP, VP]
    lib.hl_mlp_partial.argtypes = [P, I, ctypes.POINTER(hl_weights), VP, VP, I, VP, VP]
    lib.hl_residual_add.argtypes = [P, VP, VP, I, VP]
    for name in ["hl_attn_partial", "hl_mlp_partial", "hl_residual_add"]:
        getattr(lib, name).restype = I
    lib.hl_last_error.argtypes = [P]
    lib.hl_last_error.restype = ctypes.c_char_p
    for name in ["hl_create", "hl_prefill_chunk", "hl_decode", "hl_free"]:
        getattr(lib, name).restype = I
    if hasattr(lib, "hi_debug_prefill_trace"):  # HI_TRACE variant builds only
        lib.hi_debug_prefill_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        lib.hi_debug_prefill_trace.restype = ctypes.c_int
    for name in ["hi_init", "hi_init_ex", "hi_prefill_chunk", "hi_decode", "hi_free", "hi_read_host_kv",
                 "hi_write_host_kv", "hi_set_seq_len", "hi_get_stats", "hi_synchronize"]:
        getattr(lib, name).restype = I
    _lib = lib
    return lib


class HIError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
