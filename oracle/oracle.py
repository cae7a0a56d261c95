"""fp64 CPU oracle for HeadInfer's head-wise causal GQA attention.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  It shares no
code with the CUDA path (paper_2502_12574_b200/); inputs come from synth/.

Two independent formulations, both from the paper's definition:

* ``gqa_attention`` / ``attention_rows`` -- the C oracle (oracle/attention.c):
  per query row, step by step in the order of SURVEY.md §8(c):
  s_i = q.k_i/sqrt(d); m = max s_i; w_i = exp(s_i - m); o = sum w_i v_i / sum w_i.
  Head-wise (Eq. 9): each q head j reads kv head kv(j) = j // g
  (reading R4); outputs concatenated in q-head order.
* ``dense_attention_np`` -- textbook brute force: the full [n_q, n_k] score
  matrix per head, an explicit bottom-right causal mask (reading R2) and a
  row softmax (Eq. 3), in numpy float64.  Used only to pin the
  C oracle in tests.

The query at global position p attends keys 0..p (p = q_pos0 + t); decode
tokens are appended before they attend (reading R3), so a decode at position p
is the row p of a prefill over p+1 tokens.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attention.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/attention.c -> oracle/liboracle.so (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_attention_rows.restype = ctypes.c_int
        lib.oracle_attention_rows.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int, ctypes.c_void_p]
        lib.oracle_attention_rows_duo.restype = ctypes.c_int
        lib.oracle_attention_rows_duo.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_int, ctypes.c_void_p]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def attention_rows(q_rows: np.ndarray, last_key: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Rows of ONE kv head.  q_rows [R, d] bf16 bits; last_key [R] (row attends keys 0..p);
    k, v [n_k, d] bf16 bits (or any 2-D view with unit inner stride).  Returns [R, d] float64."""
    lib = _load()
    q_rows = np.ascontiguousarray(q_rows, dtype=np.uint16)
    last_key = np.ascontiguousarray(last_key, dtype=np.int64)
    if k.dtype != np.uint16 or v.dtype != np.uint16 or k.shape != v.shape or k.ndim != 2:
        raise ValueError("k, v must be uint16 [n_k, d] arrays of equal shape")
    if k.strides[1] != 2 or v.strides != k.strides:
        k = np.ascontiguousarray(k)
        v = np.ascontiguousarray(v)
    n_rows, d = q_rows.shape
    n_k = k.shape[0]
    if k.shape[1] != d:
        raise ValueError("head_dim mismatch")
    out = np.empty((n_rows, d), dtype=np.float64)
    rc = lib.oracle_attention_rows(q_rows.ctypes.data, n_rows, d, last_key.ctypes.data,
                                   k.ctypes.data, v.ctypes.data, n_k, k.strides[0] // 2, d,
                                   out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"oracle_attention_rows failed: {rc}")
    return out


def attention_rows_duo(q_rows: np.ndarray, last_key: np.ndarray, k: np.ndarray, v: np.ndarray,
                       n_sink: int, win: int) -> np.ndarray:
    """attention_rows for a duo-attention streaming head: row p attends keys i <= p with i < n_sink or
    i > p - win (oracle_attention_rows_duo; win <= 0 = no truncation)."""
    lib = _load()
    q_rows = np.ascontiguousarray(q_rows, dtype=np.uint16)
    last_key = np.ascontiguousarray(last_key, dtype=np.int64)
    k = np.ascontiguousarray(k, dtype=np.uint16)
    v = np.ascontiguousarray(v, dtype=np.uint16)
    n_rows, d = q_rows.shape
    out = np.empty((n_rows, d), dtype=np.float64)
    rc = lib.oracle_attention_rows_duo(q_rows.ctypes.data, n_rows, d, last_key.ctypes.data, int(n_sink), int(win),
                                       k.ctypes.data, v.ctypes.data, k.shape[0], d, d, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"oracle_attention_rows_duo failed: {rc}")
    return out


def duo_gqa_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_pos0: int, streaming,
                      n_sink: int, win: int) -> np.ndarray:
    """gqa_attention with duo-attention head-wise sparsity (NEXT-3): kv heads h with streaming[h]
    true attend the sink + recent-window key set; the others (retrieval heads) full causal."""
    n_q, hq, d = q.shape
    n_k, hkv, _ = k.shape
    g = hq // hkv
    out = np.empty((n_q, hq, d), dtype=np.float64)
    last = np.arange(q_pos0, q_pos0 + n_q, dtype=np.int64)
    for j in range(hq):
        h = j // g
        if streaming[h]:
            out[:, j, :] = attention_rows_duo(q[:, j, :], last, k[:, h, :], v[:, h, :], n_sink, win)
        else:
            out[:, j, :] = attention_rows(q[:, j, :], last, k[:, h, :], v[:, h, :])
    return out


def gqa_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_pos0: int) -> np.ndarray:
    """Head-wise causal GQA attention (Eq. 9 + concat).

    q [n_q, H_q, d] bf16 bits at global positions q_pos0 .. q_pos0+n_q-1;
    k, v [n_k, H_kv, d] bf16 bits at positions 0 .. n_k-1 (n_k >= q_pos0 + n_q).
    Returns [n_q, H_q, d] float64."""
    n_q, hq, d = q.shape
    n_k, hkv, _ = k.shape
    if hq % hkv:
        raise ValueError("q_heads % kv_heads != 0")
    if q_pos0 + n_q > n_k:
        raise ValueError("queries beyond the key range")
    g = hq // hkv
    out = np.empty((n_q, hq, d), dtype=np.float64)
    last = np.arange(q_pos0, q_pos0 + n_q, dtype=np.int64)
    for j in range(hq):
        h = j // g  # reading R4: contiguous groups
        out[:, j, :] = attention_rows(q[:, j, :], last, k[:, h, :], v[:, h, :])
    return out


def dense_attention_np(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_pos0: int, streaming=None,
                       n_sink: int = 0, win: int = 0) -> np.ndarray:
    """Textbook brute force (Eq. 3): full score matrix, bottom-right causal mask, row softmax.
    Same shapes/semantics as gqa_attention; float64 numpy throughout.  With ``streaming`` (per kv
    head) the streaming heads' mask is additionally restricted to keys < n_sink or > p - win."""
    from synth import bf16_to_f64
    qf, kf, vf = bf16_to_f64(q), bf16_to_f64(k), bf16_to_f64(v)
    n_q, hq, d = qf.shape
    n_k, hkv, _ = kf.shape
    g = hq // hkv
    kf = np.repeat(kf, g, axis=1)  # repeat_kv: q head j reads kv head j // g
    vf = np.repeat(vf, g, axis=1)
    scores = np.einsum("qhd,khd->hqk", qf, kf) / np.sqrt(d)
    qpos = np.arange(q_pos0, q_pos0 + n_q)[:, None]
    kpos = np.arange(n_k)[None, :]
    mask = np.broadcast_to((kpos <= qpos)[None], scores.shape).copy()
    if streaming is not None and win > 0:
        duo = (kpos < n_sink) | (kpos > qpos - win)
        for j in range(hq):
            if streaming[j // g]:
                mask[j] &= duo
    scores = np.where(mask, scores, -np.inf)
    scores = scores - scores.max(axis=-1, keepdims=True)
    w = np.exp(scores)
    w = w / w.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", w, vf)
