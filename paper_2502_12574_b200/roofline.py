"""Analytic work counters and roofline denominators for the head-wise offloaded path.

Two conventions:

* ``algorithmic`` (SURVEY.md §8(d) "Algorithmic work per unit"): exact causal pair counts,
  GQA K/V bytes -- what the method must compute / move.  Used for every reported fraction.
* ``paper`` (App. C tables): no causal halving, Q+O+K+V bytes for prefill,
  full-D (MHA-convention) K+V bytes for decode.  Only used to pin the counters against the
  paper's printed values (tests/test_roofline.py).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@dataclass(frozen=True)
class Shape:
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int

    @property
    def g(self) -> int:
        return self.q_heads // self.kv_heads


LLAMA3_8B = Shape(32, 32, 8, 128)
LLAMA3_70B = Shape(80, 64, 8, 128)
TINY = Shape(1, 4, 2, 64)             # BASELINE.json configs[0]


# ---- algorithmic convention (per layer-call, per local kv head) ---------------------------
def prefill_flops(d: int, g: int, s: int, n: int) -> float:
    """4*d*g*(s*n + n(n+1)/2): QK^T and PV over history s and the causal chunk n."""
    return 4.0 * d * g * (s * n + n * (n + 1) / 2.0)


def decode_flops(d: int, g: int, s: int) -> float:
    """4*d*g*(s+1): one query row per q head over s history keys + itself."""
    return 4.0 * d * g * (s + 1)


def kv_bytes(d: int, tokens: int) -> int:
    """K+V bytes of one head over `tokens` rows (bf16): 4*d per token."""
    return 4 * d * tokens


def duo_keys(p: int, n_sink: int, win: int) -> int:
    """Keys a duo-attention streaming head's query at position p attends (NEXT-3, reading R18):
    |{i <= p : i < n_sink or i > p - win}| = min(p+1, n_sink) + max(0, p + 1 - max(n_sink, p - win + 1))."""
    return min(p + 1, n_sink) + max(0, p + 1 - max(n_sink, p - win + 1))


def duo_pairs(s: int, n: int, n_sink: int, win: int) -> int:
    """Visible (query, key) pairs of a streaming head over chunk rows p in [s, s+n) (exact sum of duo_keys,
    summed in closed form over the three regimes of p)."""
    tot = 0
    p, end = s, s + n
    while p < end:
        if p + 1 <= n_sink:                      # every key is a sink key: p + 1 keys
            q = min(end, n_sink)
            tot += (p + 1 + q) * (q - p) // 2    # sum_{x=p}^{q-1} (x+1)
        elif p - win + 1 <= n_sink:              # window reaches into the sink: all p + 1 keys visible
            q = min(end, n_sink + win)
            tot += (p + 1 + q) * (q - p) // 2
        else:                                    # sink + a full window
            q = end
            tot += (q - p) * (n_sink + win)
        p = q
    return tot


def prefill_step(shape: Shape, s: int, n: int, world: int = 1, resident: int = 0, streaming: int = 0,
                 n_sink: int = 64, win: int = 256) -> dict:
    """One prefill chunk over all layers on one rank (H_kv/world local heads); `resident` of the
    rank's retrieval (layer, kv head) pairs keep their KV in HBM (NEXT-1): no link traffic, one HBM read;
    `streaming` pairs are duo streaming heads (NEXT-3): sink + window keys only, all in HBM."""
    pairs = shape.layers * (shape.kv_heads // world)
    retr = pairs - streaming
    off = retr - resident
    d, g = shape.head_dim, shape.g
    kept = min(s, n_sink + win)
    return {
        "flops": retr * prefill_flops(d, g, s, n) + streaming * 4.0 * d * g * duo_pairs(s, n, n_sink, win),
        "h2d_bytes": off * kv_bytes(d, s),
        "d2h_bytes": off * kv_bytes(d, n),
        "hbm_bytes": off * 2 * kv_bytes(d, s) + resident * kv_bytes(d, s) + streaming * kv_bytes(d, kept)
        + pairs * (kv_bytes(d, n) + 4 * d * g * n),
    }


def decode_step(shape: Shape, s: int, world: int = 1, resident: int = 0, streaming: int = 0,
                n_sink: int = 64, win: int = 256) -> dict:
    pairs = shape.layers * (shape.kv_heads // world)
    retr = pairs - streaming
    off = retr - resident
    d, g = shape.head_dim, shape.g
    keys = duo_keys(s, n_sink, win)   # history keys + the new one
    return {
        "flops": retr * decode_flops(d, g, s) + streaming * 4.0 * d * g * keys,
        "h2d_bytes": off * kv_bytes(d, s),
        "d2h_bytes": off * kv_bytes(d, 1),
        "hbm_bytes": off * 2 * kv_bytes(d, s) + resident * kv_bytes(d, s) + streaming * kv_bytes(d, keys),
    }


def step_roofline_seconds(work: dict, peaks: dict) -> dict:
    """T_roof = max over resources (SURVEY.md §8(d) 'Per-step roofline')."""
    t = {
        "tensor": work["flops"] / (peaks["bf16_tflops"] * 1e12),
        "hbm": work["hbm_bytes"] / (peaks["hbm_gbs"] * 1e9),
        "h2d": work["h2d_bytes"] / (peaks["h2d_gbs"] * 1e9),
        "d2h": work["d2h_bytes"] / (peaks["d2h_gbs"] * 1e9),
    }
    if peaks.get("bidir_gbs"):
        t["bidir"] = (work["h2d_bytes"] + work["d2h_bytes"]) / (peaks["bidir_gbs"] * 1e9)
    bound = max(t, key=t.get)
    return {"seconds": t[bound], "bound": bound, "terms": t}


# ---- paper convention (App. C, one Llama-3-8B layer, D = H_q * d) ----------------------------
def paper_prefill(shape: Shape, S: int, heads: int | None = None) -> dict:
    """App. C 'flashattention (S)' prefill row: Ops = 4*S^2*D, Memory = Q+O+K+V bytes,
    offload memory = K+V bytes.  heads=1 gives the 'head-wise' row (one of H_kv groups)."""
    D = shape.q_heads * shape.head_dim
    Dkv = shape.kv_heads * shape.head_dim
    frac = 1.0 if heads is None else heads / shape.kv_heads
    ops = 4.0 * S * S * D * frac
    mem = (2 * S * D + 2 * S * Dkv) * 2 * frac
    kv = 2 * S * Dkv * 2 * frac
    return {"ops": ops, "memory": mem, "kv_memory": kv}


def paper_decode(shape: Shape, S: int, heads: int | None = None) -> dict:
    """App. C decode row: Ops = 4*S*D, Memory = 2*S*D*2 bytes (full-D K+V, MHA convention)."""
    D = shape.q_heads * shape.head_dim
    frac = 1.0 if heads is None else heads / shape.kv_heads
    return {"ops": 4.0 * S * D * frac, "memory": 2.0 * S * D * 2 * frac}


# ---- measured peaks --------------------------------------------------------------------------
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}
# host link, measured on this pool's B200 box with 4 GiB pinned copies (tools/probe_box.sh ->
# profiles/host_link_r01.txt); per direction and both directions concurrently
HOST_LINK = {"h2d_gbs": 55.6, "d2h_gbs": 55.4, "bidir_gbs": 98.6, "source": "measured (profiles/host_link_r01.txt)"}


def load_peaks() -> dict:
    p = dict(FALLBACK)
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained"):
            if k in m:
                p[k] = float(m[k])
        p["source"] = "measured (MEASURED_PEAKS.json)"
    p.update({k: v for k, v in HOST_LINK.items() if k != "source"})
    p["host_link_source"] = HOST_LINK["source"]
    return p
