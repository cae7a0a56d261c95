"""bench.py -- HeadInfer head-wise offloaded attention on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload auto|8B-1M|8B-128K|tiny]

A "step" (ours): one pass of the hot path over one batch of synthetic input --
  prefill step = one 18944-token chunk (148 SMs x 256 rows / g) through all 32 layers (write-back D2H, history H2D through
                 the staging slots, causal attention over history + chunk, per layer call);
                 the timed chunks are the LAST K chunks of the 1M prefill (the most expensive ones),
                 the W warm-up chunks precede them; the history before them is placed in the host
                 store untimed (hi_write_host_kv, App. E P:L1010 "preparing decoding with large context").
  decode step  = one token through all 32 layers at context S (H2D of the whole history).
`value` = prefill tokens/s over the timed chunks (whole job, all ranks: each token is processed by
every rank for its heads, so scaling is strong); decode ms/token and host-link GB/s ride along.
Inputs are generated on the GPU by synth/ (seeded, bit-identical to the oracle's generator) and are
resident in HBM before the timed region (`value`); `e2e` re-runs the timed chunks through the public
API from pinned HOST buffers with the H2D of Q/K/V and the D2H of `out` inside the timed region.
Inputs per step (>= 6 GiB) exceed the 126 MB L2, so no extra flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1M-ctx Llama-3-8B-shape prefill tok/s, decode ms/tok; H2D GB/s vs link peak"
WORKLOADS = {
    # name: (layers, q_heads, kv_heads, d, context S, chunk)
    # chunk = 148 SMs x 256 rows (two 128-row Q tiles per CTA) / g = 18944 tokens for g = 4: every
    # prefill launch is exactly 2 full waves (16384 would leave a 73%-full second wave)
    "8B-1M": (32, 32, 8, 128, 1 << 20, 18944),
    "8B-128K": (32, 32, 8, 128, 131072, 18944),
    "tiny": (1, 4, 2, 64, 1024, 128),
    # configs[3] / configs[4] are 8-GPU head-sharded workloads; on one GPU they run as one rank's share
    # (--emulate-shard 0/8): 1 kv head per layer.  70B: g = 8, so 9472 tokens x 8 rows = 2 full waves.
    "8B-4M": (32, 32, 8, 128, 4 << 20, 18944),
    "70B-1M": (80, 64, 8, 128, 1 << 20, 9472),
}
SEED = 0x48454144
DIST = "U"  # throughput workload
# --model (NEXT-4): Llama-3-8B decoder-layer dims around the attention path (hidden, intermediate)
MODEL_DIMS = (4096, 14336)
MODEL_ROPE_THETA = 500000.0
MODEL_RMS_EPS = 1e-5


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
def mem_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def pick_workload(name: str, world: int, steps: int, warmup: int) -> str:
    if name != "auto":
        return name
    L, hq, hkv, d, S, c = WORKLOADS["8B-1M"]
    need = L * (hkv // world) * 4 * d * (S + steps + warmup) + L * (hq // world + 2 * hkv // world) * c * d * 2 * 2
    # the host store must fit with room to spare (a box driven out of memory is a strike)
    if mem_available_bytes() >= need * world + (24 << 30):
        return "8B-1M"
    log(f"bench: MemAvailable {mem_available_bytes()/2**30:.0f} GiB < need; falling back to 8B-128K")
    return "8B-128K"


def gen_layer_inputs(layer, pos0, n, hq_loc, hkv_loc, d, q_head0, kv_head0, torch, fill_):
    Q = fill_(torch.empty((n, hq_loc, d), dtype=torch.bfloat16, device="cuda"), SEED, 0, DIST, layer, q_head0, pos0)
    K = fill_(torch.empty((n, hkv_loc, d), dtype=torch.bfloat16, device="cuda"), SEED, 1, DIST, layer, kv_head0, pos0)
    V = fill_(torch.empty((n, hkv_loc, d), dtype=torch.bfloat16, device="cuda"), SEED, 2, DIST, layer, kv_head0, pos0)
    return Q, K, V


def fill_history(hi, L, hkv_loc, kv_head0, d, upto, torch, fill_, labels=None, duo=(0, 0)):
    """Untimed: place the K/V of positions [0, upto) in the host store (same bytes a prefill writes).
    Streaming heads (NEXT-3) keep only the sink rows and the last window rows: only those are written."""
    piece = 65536
    bk = torch.empty((piece, 1, d), dtype=torch.bfloat16, device="cuda")
    bv = torch.empty_like(bk)
    for l in range(L):
        for h in range(hkv_loc):
            ranges = [(0, upto)]
            if labels is not None and labels[l][kv_head0 + h]:
                ns = min(max(duo[0], 0), upto)
                ranges = [(0, ns), (max(ns, upto - duo[1]), upto)]
            for lo, end in ranges:
                for p0 in range(lo, end, piece):
                    n = min(piece, end - p0)
                    fill_(bk[:n], SEED, 1, DIST, l, kv_head0 + h, p0)
                    fill_(bv[:n], SEED, 2, DIST, l, kv_head0 + h, p0)
                    hi.write_host_kv(l, h, p0, bk[:n, 0], bv[:n, 0])


def run_ours(args, rank, world, local_rank, pg):
    import torch
    import torch.distributed as dist

    from paper_2502_12574_b200 import roofline as rf
    from paper_2502_12574_b200._lib import HI_FLAG_TIMING
    from paper_2502_12574_b200.headinfer import HeadInfer
    from paper_2502_12574_b200.parallel import gather_heads, shard
    from synth.cuda import fill_

    K, W = args.steps, args.warmup
    wl = pick_workload(args.workload, world, K, W)
    if world > 1:
        # every rank must agree on the workload
        t = torch.tensor([list(WORKLOADS).index(wl)], device="cpu" if args.ranks_share_gpu else "cuda")
        dist.broadcast(t, 0)
        wl = list(WORKLOADS)[int(t.item())]
    L, hq, hkv, d, S, c = WORKLOADS[wl]
    # head shard: this process's rank, or (--emulate-shard R/W) rank R of a W-GPU job run alone on this GPU
    hr, hw = (rank, world) if args.emulate_shard is None else args.emulate_shard
    sh = shard(hq, hkv, hr, hw)
    host_need = L * (hkv // hw) * 4 * d * (S + 2 * (K + W) + 8) * (world if args.emulate_shard is None else 1)
    if mem_available_bytes() < host_need + (24 << 30):   # a box driven out of memory is a strike
        raise SystemExit(f"workload {wl}: host store {host_need / 2**30:.0f} GiB does not fit in MemAvailable "
                         f"{mem_available_bytes() / 2**30:.0f} GiB with a 24 GiB margin")
    hq_loc, hkv_loc, q0h, kv0h = sh["q_local"], sh["kv_local"], sh["q"][0], sh["kv"][0]
    n_pre = W + K
    s0 = S - K * c - W * c                   # first warm-up chunk position
    if s0 < 0:
        raise SystemExit(f"workload {wl}: context {S} too short for {n_pre} chunks of {c}")
    max_ctx = S + 2 * n_pre + 8              # prefill to S, then decode steps (+ e2e re-runs)
    peaks = rf.load_peaks()
    shape = rf.Shape(L, hq, hkv, d)

    resident = args.resident_heads
    if resident < 0:  # as many (layer, kv head) pairs as fit next to this bench's inputs (NEXT-1)
        free_b, _ = torch.cuda.mem_get_info()
        inputs_b = (K + 2) * L * c * (hq_loc + 2 * hkv_loc) * d * 2 + L * c * hq_loc * d * 2
        if args.model:  # 32 layers of weights + the layer workspaces
            H, I = MODEL_DIMS
            inputs_b += L * (H * (hq + 2 * hkv) * d + H * hq * d + 3 * H * I) * 2 + c * (4 * H + 3 * I) * 2
        pair_b = 4 * d * max_ctx
        resident = int(max(0, min(L * hkv_loc, (free_b - inputs_b - (10 << 30)) // pair_b)))
    labels, duo = None, (args.duo_sink, args.duo_window)
    duo_opts = {}
    if args.duo > 0:  # NEXT-3: synthetic duo-attention labels, `args.duo` of each layer's kv heads streaming
        import synth
        labels = synth.streaming_labels(SEED, L, hkv, args.duo)
        duo_opts = dict(streaming_heads=labels.tolist(), duo_sink=args.duo_sink if args.duo_sink > 0 else -1,
                        duo_window=args.duo_window)
    t0 = time.time()
    hi = HeadInfer(L, hq, hkv, d, max_ctx, c, hr, hw, flags=HI_FLAG_TIMING, resident_kv_heads=resident,
                   head_group=args.head_group, **duo_opts)
    init_s = time.time() - t0
    t0 = time.time()
    fill_history(hi, L, hkv_loc, kv0h, d, s0, torch, fill_, labels, duo)
    fill_s = time.time() - t0
    log(f"[rank {rank}] {wl}: init {init_s:.1f}s (host store {hi.stats()['host_store_bytes']/2**30:.1f} GiB), "
        f"history fill {fill_s:.1f}s")
    for l in range(L):
        hi.set_seq_len(l, s0)

    stream = torch.cuda.current_stream()
    gathered = None

    def barrier():
        if world > 1:
            dist.barrier(group=pg)

    gathered0 = None

    # ---------------- the step: attention path only (default), or whole synthetic layers (--model, NEXT-4)
    model = None
    if args.model:
        from paper_2502_12574_b200.layer import HeadInferLayer
        from synth.cuda import fill_matrix_, gen_layer_weights_cuda
        if world != 1:
            raise SystemExit("--model runs at world 1 (the layer wrapper has no tensor parallelism)")
        H, I = MODEL_DIMS
        model = HeadInferLayer(hi, H, I, MODEL_ROPE_THETA, MODEL_RMS_EPS)
        weights = [gen_layer_weights_cuda(SEED, l, H, I, hq, hkv, d) for l in range(L)]
        torch.cuda.synchronize()

    def make_inputs(pos, n):
        """One step's inputs: per-layer (Q, K, V) for the attention path; x [n, H] for --model."""
        if model is not None:
            return fill_matrix_(torch.empty((n, MODEL_DIMS[0]), dtype=torch.bfloat16, device="cuda"), SEED,
                                synth_tensor_x, 0, row0=pos)
        return [gen_layer_inputs(l, pos, n, hq_loc, hkv_loc, d, q0h, kv0h, torch, fill_) for l in range(L)]

    def prefill_step(inputs, outs):
        nonlocal gathered, gathered0
        if model is not None:   # x flows through every layer in place; outs[0] keeps layer 0's input copy
            for l in range(L):
                model.prefill_chunk(l, weights[l], inputs)
            return
        for l in range(L):
            Q, Kt, Vt = inputs[l]
            hi.prefill_chunk(l, Q, Kt, Vt, outs[l])
            if world > 1:
                if l == 0:
                    gathered0 = gather_heads(outs[l], group=pg, out=gathered0)
                else:
                    gathered = gather_heads(outs[l], group=pg, out=gathered)

    synth_tensor_x = 3  # synth.TENSOR_X

    # ---------------- prefill: W warm-up chunks, then K timed chunks (all inputs resident) -------
    outs = [torch.empty((c, hq_loc, d), dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    for i in range(W):
        inputs = make_inputs(s0 + i * c, c)
        prefill_step(inputs, outs)
        del inputs
    timed_inputs = [make_inputs(s0 + (W + i) * c, c) for i in range(K)]
    hi.synchronize()
    st0 = hi.stats()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk_p:
        e0.record(stream)
        for i in range(K):
            prefill_step(timed_inputs[i], outs)
        hi.synchronize()  # drain the write-back stream too
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    pre_ms = e0.elapsed_time(e1)
    st1 = hi.stats()
    sample_out0 = outs[0].clone()     # layer 0 outputs of the last timed chunk (parity sample)
    last_chunk_pos = s0 + (W + K - 1) * c
    del timed_inputs

    # ---------------- decode: W warm-up tokens, then K timed tokens at context S ----------------
    dq = [make_inputs(S + i, 1) for i in range(W + K)]
    dout = [torch.empty((hq_loc, d), dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    gdec = None

    def decode_step(i):
        nonlocal gdec
        if model is not None:
            for l in range(L):
                model.decode(l, weights[l], dq[i][0])
            return
        for l in range(L):
            q, k, v = dq[i][l]
            hi.decode(l, q[0], k[0], v[0], dout[l])
            if world > 1:
                gdec = gather_heads(dout[l], group=pg, out=gdec)

    for i in range(W):
        decode_step(i)
    hi.synchronize()
    sd0 = hi.stats()
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(local_rank) as clk_d:
        e0.record(stream)
        for i in range(W, W + K):
            decode_step(i)
        hi.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    dec_ms = e0.elapsed_time(e1)
    sd1 = hi.stats()
    dec_sample = dout[0].clone()
    dec_pos = S + W + K - 1

    # ---------------- e2e: the timed prefill chunks again, inputs from pinned HOST memory --------
    e2e = None
    if not args.no_e2e:
        for l in range(L):
            hi.set_seq_len(l, s0 + W * c)
        if model is not None:   # x in, x out (the last layer's hidden states)
            shapes = [[(c, MODEL_DIMS[0])]]
            out_shape = (c, MODEL_DIMS[0])
        else:
            shapes = [[(c, hq_loc, d), (c, hkv_loc, d), (c, hkv_loc, d)] for _ in range(L)]
            out_shape = (c, hq_loc, d)
        host_in = [[torch.empty(sh, dtype=torch.bfloat16).pin_memory() for sh in per] for per in shapes]
        host_out = [torch.empty(out_shape, dtype=torch.bfloat16).pin_memory() for _ in shapes]
        dev_in = [[torch.empty(t.shape, dtype=t.dtype, device="cuda") for t in per] for per in host_in]
        e2e_ms = 0.0
        h2d_b = sum(t.numel() * 2 for per in host_in for t in per)
        d2h_b = sum(t.numel() * 2 for t in host_out)
        for i in range(K):
            step_in = make_inputs(s0 + (W + i) * c, c)   # untimed: this step's inputs into pinned host buffers
            step_in = [[step_in]] if model is not None else step_in
            for per_dev, per_host in zip(step_in, host_in):
                for t_dev, t_host in zip(per_dev, per_host):
                    t_host.copy_(t_dev)
            del step_in
            torch.cuda.synchronize()
            barrier()
            e0.record(stream)
            if model is not None:
                dev_in[0][0].copy_(host_in[0][0], non_blocking=True)
                for l in range(L):
                    model.prefill_chunk(l, weights[l], dev_in[0][0])
                host_out[0].copy_(dev_in[0][0], non_blocking=True)
            else:
                for l in range(L):
                    for t_dev, t_host in zip(dev_in[l], host_in[l]):
                        t_dev.copy_(t_host, non_blocking=True)
                    hi.prefill_chunk(l, *dev_in[l], outs[l])
                    if world > 1:
                        gathered = gather_heads(outs[l], group=pg, out=gathered)
                    host_out[l].copy_(outs[l], non_blocking=True)
            hi.synchronize()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            e2e_ms += e0.elapsed_time(e1)
        del host_in, host_out, dev_in
        e2e = {"ms": e2e_ms, "h2d": h2d_b, "d2h": d2h_b}

    # ---------------- max over ranks --------------------------------------------------------------
    times = torch.tensor([pre_ms, dec_ms, e2e["ms"] if e2e else 0.0], dtype=torch.float64,
                         device="cpu" if args.ranks_share_gpu else "cuda")
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX, group=pg)
    pre_ms, dec_ms, e2e_ms = times.tolist()

    # ---------------- report (rank 0) -------------------------------------------------------------
    if rank != 0:
        hi.close()
        return
    tok_s = K * c / (pre_ms / 1e3)
    dec_ms_tok = dec_ms / K
    h2d_dec = (sd1["h2d_bytes"] - sd0["h2d_bytes"]) / K
    h2d_gbs = h2d_dec / (dec_ms_tok / 1e3) / 1e9
    pf_flops = st1["prefill_attn_flops"] - st0["prefill_attn_flops"]
    pf_ms = st1["prefill_attn_ms"] - st0["prefill_attn_ms"]
    pf_launches = st1["prefill_attn_launches"] - st0["prefill_attn_launches"]
    achieved_tflops = pf_flops / (pf_ms / 1e3) / 1e12 if pf_ms > 0 else None
    peak_t = peaks["bf16_tflops_sustained"]
    dk_bytes = sd1["decode_attn_bytes"] - sd0["decode_attn_bytes"]
    dk_ms = sd1["decode_attn_ms"] - sd0["decode_attn_ms"]
    # step rooflines (measured peaks; sustained tensor peak inside a long step)
    pk = dict(peaks, bf16_tflops=peak_t)
    R = st1["resident_kv_heads"]
    dk = dict(streaming=st1["streaming_kv_heads"], n_sink=max(args.duo_sink, 0), win=args.duo_window)
    roof_p = rf.step_roofline_seconds(rf.prefill_step(shape, last_chunk_pos - c * (K - 1) // 2, c, hw, R, **dk), pk)
    t_roof_pre = sum(rf.step_roofline_seconds(rf.prefill_step(shape, s0 + (W + i) * c, c, hw, R, **dk), pk)["seconds"]
                     for i in range(K))
    dec_roofs = [rf.step_roofline_seconds(rf.decode_step(shape, S + i, hw, R, **dk), pk) for i in range(W, W + K)]
    t_roof_dec = sum(x["seconds"] for x in dec_roofs)
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "ncu_prefill_traffic.json")
    if os.path.exists(prof_path):
        with open(prof_path) as f:
            prof = json.load(f)
        traffic = prof.get("dram_bytes_per_launch")
    launches = (st1["kernel_launches"] - st0["kernel_launches"]) + (sd1["kernel_launches"] - sd0["kernel_launches"])
    # prefill copy engines (HI_FLAG_TIMING events on the copy streams): busy time, rate while busy, and how much
    # of the copy time the step hides (1 = every copy overlapped with attention, SURVEY.md §8(d) timing)
    pf_h2d_b, pf_d2h_b = st1["h2d_bytes"] - st0["h2d_bytes"], st1["d2h_bytes"] - st0["d2h_bytes"]
    pf_h2d_ms, pf_d2h_ms = st1["h2d_copy_ms"] - st0["h2d_copy_ms"], st1["d2h_copy_ms"] - st0["d2h_copy_ms"]
    prefill_copies = {
        "h2d_bytes_per_step": int(pf_h2d_b / K), "d2h_bytes_per_step": int(pf_d2h_b / K),
        "h2d_busy_ms_per_step": round(pf_h2d_ms / K, 3), "d2h_busy_ms_per_step": round(pf_d2h_ms / K, 3),
        "h2d_gbs_while_busy": round(pf_h2d_b / (pf_h2d_ms / 1e3) / 1e9, 2) if pf_h2d_ms > 0 else None,
        "d2h_gbs_while_busy": round(pf_d2h_b / (pf_d2h_ms / 1e3) / 1e9, 2) if pf_d2h_ms > 0 else None,
        "h2d_busy_frac_of_step": round(pf_h2d_ms / pre_ms, 4) if pre_ms else None,
        "attention_frac_of_step": round(pf_ms / pre_ms, 4) if pre_ms else None,
        "copy_hidden_frac": (round(max(0.0, min(1.0, (pf_ms + pf_h2d_ms - pre_ms) / pf_h2d_ms)), 4)
                             if pf_h2d_ms > 0 else None)}
    clk = clk_p.summary()

    res = {
        "metric": METRIC,
        "value": round(tok_s, 2),
        "unit": "tok/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(pre_ms / K, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded counter-hash generator, distribution U; Llama-3-8B attention shapes, "
                "no weights: attention-only path)",
        "config": {"workload": wl, "layers": L, "q_heads": hq, "kv_heads": hkv, "head_dim": d, "context": S,
                   "chunk": c, "head_group": st1["head_group"], "resident_kv_heads": R,
                   "duo": ({"streaming_frac": args.duo, "streaming_kv_heads": st1["streaming_kv_heads"],
                            "sink": max(args.duo_sink, 0), "window": args.duo_window,
                            "labels": "synthetic (synth.streaming_labels)"} if args.duo > 0 else None),
                   "parallelism": (f"head-shard{world}" if args.emulate_shard is None else
                                   f"rank {hr} of head-shard{hw}, run alone on 1 GPU (no all-gather)"),
                   "prefill_step": "1 chunk x all layers",
                   "timed_chunk_positions": [s0 + W * c, last_chunk_pos],
                   "decode_step": "1 token x all layers", "decode_context": [S + W, S + W + K - 1],
                   "l2": "inputs per step > L2 (>= 6 GiB), no flush needed"},
        "decode": {"ms_per_token": round(dec_ms_tok, 3), "h2d_gbs": round(h2d_gbs, 2),
                   "link_peak_gbs": peaks["h2d_gbs"], "link_frac": round(h2d_gbs / peaks["h2d_gbs"], 4),
                   "roofline_frac": round(t_roof_dec / (dec_ms / 1e3), 4), "roofline_bound": dec_roofs[-1]["bound"],
                   "h2d_bytes_per_token": int(h2d_dec),
                   "kernel": {"bound": "hbm", "achieved_gbs": round(dk_bytes / (dk_ms / 1e3) / 1e9, 1) if dk_ms else None,
                              "peak_gbs": peaks["hbm_gbs"],
                              "frac": round(dk_bytes / (dk_ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4) if dk_ms else None},
                   "clocks": clk_d.summary()},
        "prefill_copies": prefill_copies,
        "prefill_step_roofline": {"frac": round(t_roof_pre / (pre_ms / 1e3), 4), "bound": roof_p["bound"],
                                  "t_roof_s": round(t_roof_pre, 4), "t_meas_s": round(pre_ms / 1e3, 4)},
        "roofline": {"bound": "tensor", "kernel": "prefill attention (history + causal segments)",
                     "achieved": round(achieved_tflops, 2) if achieved_tflops else None,
                     "peak": peak_t, "unit": "TFLOP/s",
                     "frac": round(achieved_tflops / peak_t, 4) if achieved_tflops else None,
                     "traffic": traffic, "launches": pf_launches,
                     "flops_per_launch": pf_flops / max(pf_launches, 1),
                     "peak_source": peaks["source"] + " bf16_tflops_sustained"},
        "clocks": clk,
        "gpu_launches": launches,
        "residency": {"staging_bytes": st1["staging_bytes"], "staging_bound_bytes": st1["staging_bound_bytes"],
                      "one_head_bytes": 4 * d * max_ctx,
                      "head_group": st1["head_group"],
                      "host_store_bytes": st1["host_store_bytes"], "init_s": round(init_s, 2),
                      "resident_kv_heads": st1["resident_kv_heads"], "resident_bytes": st1["resident_bytes"]},
    }
    if e2e:
        res["e2e"] = {"value": round(K * c / (e2e_ms / 1e3), 2), "unit": "tok/s",
                      "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"]}
    if world > 1 and not args.no_cpu_baseline:
        res["parity_sample"] = sharded_parity(gathered0, last_chunk_pos, L, hq, hkv, d, world, torch, labels, duo)
    if model is not None:
        H, I = MODEL_DIMS
        gemm_tok = L * 2.0 * (H * (hq + 2 * hkv) * d + H * hq * d + 3 * H * I)  # QKV, O, gate+up, down
        t_gemm = K * c * gemm_tok / (peak_t * 1e12)
        res["config"]["path"] = "synthetic Llama-3-8B decoder layers (NEXT-4): RMSNorm, QKV/O/MLP GEMMs, RoPE, SwiGLU"
        res["data"] = ("synthetic (seeded counter-hash generator): hidden states in, random-init Llama-3-8B layer "
                       "weights (no trained weights, no embedding / LM head)")
        res["config"]["hidden"], res["config"]["intermediate"] = H, I
        res["model"] = {"prefill_tok_s": round(tok_s, 2), "decode_ms_per_token": round(dec_ms_tok, 3),
                        "gemm_flops_per_token": gemm_tok,
                        "attention_share_of_prefill": round(pf_ms / pre_ms, 4) if pre_ms else None,
                        "step_roofline_frac": round((t_roof_pre + t_gemm) / (pre_ms / 1e3), 4),
                        "parity": "tests/test_gpu_layer.py (layer oracle, incl. one 8B-shaped layer)",
                        "note": "history K/V below the timed chunks are synthetic (placed untimed), not produced "
                                "by running the layers; no embedding / LM head"}
        model.close()
    if world == 1 and not args.no_cpu_baseline and model is None:
        res["cpu_baseline"], res["parity_sample"] = cpu_baseline(hi, sample_out0, last_chunk_pos, dec_sample, dec_pos,
                                                                 L, hq, hkv, d, torch, labels=labels, duo=duo,
                                                                 kv0=kv0h, hkv_loc=hkv_loc)
    if args.emulate_shard is not None:
        res["shard_emulation"] = {
            "rank": hr, "world": hw, "kv_heads": list(sh["kv"]), "q_heads": list(sh["q"]),
            "note": "one rank's share of a head-sharded job, measured alone on one GPU: every rank does the same "
                    "work on its own heads (no K/V crosses GPUs), so value is the job's tok/s if the W ranks run "
                    "as fast as this one; the per-layer output all-gather and any host-link sharing between "
                    "ranks are not measured"}
    hi.close()
    print(json.dumps(res), flush=True)


# ---------------------------------------------------------------------------------------------
def _oracle_inputs_for_head(layer, kv_head, upto, d, torch):
    """K, V of (layer, kv head) positions [0, upto) from synth's GPU twin (bit-identical to
    synth.gen_block, pinned by tests) -> host numpy; the oracle never reads the library."""
    import numpy as np
    from synth.cuda import gen_block_cuda
    k = gen_block_cuda(SEED, 1, DIST, layer, kv_head, 1, 0, upto, d).cpu().view(torch.int16).numpy().view(np.uint16)
    v = gen_block_cuda(SEED, 2, DIST, layer, kv_head, 1, 0, upto, d).cpu().view(torch.int16).numpy().view(np.uint16)
    return k[:, 0], v[:, 0]


def _oracle_rows(oracle, q, last, k, v, streaming, duo):
    """The oracle for one head's rows: full causal (retrieval head) or sink + window (streaming head)."""
    if streaming:
        return oracle.attention_rows_duo(q, last, k, v, max(duo[0], 0), duo[1])
    return oracle.attention_rows(q, last, k, v)


def cpu_baseline(hi, sample_out0, chunk_pos, dec_sample, dec_pos, L, hq, hkv, d, torch, budget_s=15.0,
                 labels=None, duo=(0, 0), kv0=0, hkv_loc=None):
    """Time the fp64 oracle (as it stands) on this box's host cores on a bounded sample of the same
    workload: rows of layer 0's last timed prefill chunk; also check those rows against the GPU.
    With duo labels (NEXT-3) the sampled streaming heads use the duo oracle."""
    import numpy as np

    import oracle
    import synth
    oracle.build()
    g = hq // hkv
    c = sample_out0.shape[0]
    own = list(range(kv0, kv0 + (hkv if hkv_loc is None else hkv_loc)))  # global kv heads held in sample_out0
    heads = own[:2]                    # kv heads sampled (q heads of their groups)
    strm = {h: bool(labels is not None and labels[0][h]) for h in own}
    if labels is not None:             # one retrieval and one streaming head when both exist
        r_h = [h for h in own if not strm[h]][:1]
        s_h = [h for h in own if strm[h]][:1]
        heads = (r_h + s_h) or heads
    kv = {h: _oracle_inputs_for_head(0, h, dec_pos + 1, d, torch) for h in heads}
    q0 = own[0] * g                    # q heads of the owned kv heads only
    qpre = synth.gen_block(SEED, 0, DIST, 0, q0, len(own) * g, chunk_pos, c, d)
    # calibrate: one row per thread
    cores = oracle.num_threads()
    rng = np.random.default_rng(0)

    def rows_for(n_tok):
        toks = np.unique(np.concatenate([[0, c - 1], rng.integers(0, c, max(0, n_tok - 2))]))[:n_tok]
        return toks

    # calibrate on one call of `cores` rows (the oracle parallelises over the rows of a call)
    k0, v0 = kv[heads[0]]
    probe_t = rows_for(cores)
    t0 = time.time()
    _oracle_rows(oracle, qpre[probe_t, heads[0] * g - q0], chunk_pos + probe_t, k0, v0, strm[heads[0]], duo)
    rows_per_s = len(probe_t) / max(time.time() - t0, 1e-9)
    n_tok = int(max(2, min(c, budget_s * rows_per_s / (g * len(heads)))))
    toks = rows_for(n_tok)
    t0 = time.time()
    maxerr, sumerr, cnt, rows = 0.0, 0.0, 0, 0
    got = sample_out0.float().cpu().numpy()
    for h in heads:
        k, v = kv[h]
        for j in range(h * g, (h + 1) * g):
            ref = _oracle_rows(oracle, qpre[toks, j - q0], chunk_pos + toks, k, v, strm[h], duo)
            err = np.abs(got[toks, j - q0] - ref)
            maxerr = max(maxerr, float(err.max()))
            sumerr += float(err.sum())
            cnt += err.size
            rows += len(toks)
    el = time.time() - t0
    # decode row: the last timed decode token, sampled kv heads
    qd = synth.gen_block(SEED, 0, DIST, 0, q0, len(own) * g, dec_pos, 1, d)[0]
    dgot = dec_sample.float().cpu().numpy()
    dmax = 0.0
    for h in heads:
        k, v = kv[h]
        for j in range(h * g, (h + 1) * g):
            ref = _oracle_rows(oracle, qd[j - q0:j - q0 + 1], np.array([dec_pos]), k, v, strm[h], duo)[0]
            dmax = max(dmax, float(np.abs(dgot[j - q0] - ref).max()))
    rows_per_tok = L * hq
    cpu = {"value": round(rows / el / rows_per_tok, 6), "unit": "tok/s", "cores": cores, "kind": "oracle",
           "sample": f"{rows} (layer 0, q head, position) rows of the last timed prefill chunk at positions "
                     f"{chunk_pos}+t, q heads of kv heads {heads}, {el:.1f}s; tok/s = rows/s / "
                     f"({L} layers x {hq} q heads)"}
    parity = {"prefill_rows": rows, "prefill_max_abs": maxerr, "prefill_mean_abs": sumerr / max(cnt, 1),
              "decode_rows": len(heads) * g, "decode_max_abs": dmax, "tol_max_abs": 2e-2, "tol_mean_abs": 2e-3}
    return cpu, parity


def sharded_parity(gathered0, chunk_pos, L, hq, hkv, d, world, torch, labels=None, duo=(0, 0), n_tok=4):
    """Head-sharded run: rows of the all-gathered layer-0 output of the last timed chunk, one q head
    per rank, against the oracle (checks the shard arithmetic + the collective end to end)."""
    import numpy as np

    import oracle
    import synth
    from paper_2502_12574_b200.parallel import to_token_major
    oracle.build()
    full = to_token_major(gathered0).float().cpu().numpy()  # [c, hq, d]
    c = full.shape[0]
    g = hq // hkv
    toks = np.array([0, c // 3, 2 * c // 3, c - 1][:n_tok])
    maxerr = 0.0
    for r in range(world):
        j = r * (hq // world)          # first q head owned by rank r
        kv, v = _oracle_inputs_for_head(0, j // g, chunk_pos + c, d, torch)
        q = synth.gen_block(SEED, 0, DIST, 0, j, 1, chunk_pos, c, d)[toks, 0]
        ref = _oracle_rows(oracle, q, chunk_pos + toks, kv, v, bool(labels is not None and labels[0][j // g]), duo)
        maxerr = max(maxerr, float(np.abs(full[toks, j] - ref).max()))
    return {"gathered_rows": int(len(toks) * world), "max_abs": maxerr, "tol_max_abs": 2e-2}


# ---------------------------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle (as it stands) on this box's host cores, same metric/config.
    Each step is a bounded sample of the workload: a slice of the rows of one prefill chunk."""
    if rank != 0:
        return
    import numpy as np
    import torch

    import oracle
    import synth
    oracle.build()
    wl = args.workload if args.workload != "auto" else "8B-1M"
    L, hq, hkv, d, S, c = WORKLOADS[wl]
    g = hq // hkv
    pos = S - c
    # inputs from the numpy generator for one kv head of layer 0 (bounded: first 64K keys of
    # history are regenerated per call? no -- the whole prefix is needed; use a shorter prefix
    # at the same shapes is NOT the workload, so take the full prefix of one head)
    if torch.cuda.is_available():
        k, v = _oracle_inputs_for_head(0, 0, pos + c, d, torch)
    else:
        k = synth.gen_block(SEED, 1, DIST, 0, 0, 1, 0, pos + c, d)[:, 0]
        v = synth.gen_block(SEED, 2, DIST, 0, 0, 1, 0, pos + c, d)[:, 0]
    q = synth.gen_block(SEED, 0, DIST, 0, 0, g, pos, c, d)
    cores = oracle.num_threads()
    rows_per_step = max(cores, 16)
    rng = np.random.default_rng(1)

    def step():
        toks = rng.integers(0, c, rows_per_step)
        j = rng.integers(0, g)
        oracle.attention_rows(q[toks, j], pos + toks, k, v)

    for _ in range(args.warmup):
        step()
    t0 = time.time()
    for _ in range(args.steps):
        step()
    el = time.time() - t0
    val = args.steps * rows_per_step / el / (L * hq)
    res = {"impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "tok/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same generator and workload as the ours arm)",
           "config": {"workload": wl, "layers": L, "q_heads": hq, "kv_heads": hkv, "head_dim": d, "context": S,
                      "chunk": c, "parallelism": "host cores"},
           "cpu_baseline": {"value": round(val, 6), "unit": "tok/s", "cores": cores, "kind": "oracle",
                            "sample": f"per step {rows_per_step} (layer 0, q head, position) rows of the chunk at "
                                      f"{pos}; tok/s = rows/s / ({L} x {hq})"},
           "e2e": {"value": round(val, 6), "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["auto"] + list(WORKLOADS), default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--resident-heads", type=int, default=0,
                    help="NEXT-1: keep the first R (layer, kv head) pairs' KV in HBM (-1 = as many as fit)")
    ap.add_argument("--head-group", type=int, default=-1,
                    help="NEXT-2: kv heads per transfer/launch unit (-1 = auto: >= 8 waves per chunk launch)")
    ap.add_argument("--model", action="store_true",
                    help="NEXT-4: time whole synthetic Llama-3-8B decoder layers (RMSNorm, QKV/O/MLP GEMMs, RoPE, "
                         "SwiGLU) around the attention path instead of the attention path alone")
    ap.add_argument("--duo", type=float, default=0.0,
                    help="NEXT-3: fraction of each layer's kv heads that are duo-attention streaming heads "
                         "(synthetic labels; the paper's extension table uses 0.5)")
    ap.add_argument("--duo-sink", type=int, default=64, help="NEXT-3: attention-sink tokens of streaming heads")
    ap.add_argument("--duo-window", type=int, default=256, help="NEXT-3: recent-window tokens of streaming heads")
    ap.add_argument("--emulate-shard", type=lambda x: tuple(int(v) for v in x.split("/")), default=None,
                    metavar="R/W", help="run rank R's head shard of a W-GPU job alone on this GPU (configs[3]/[4] "
                                        "on one B200: e.g. --workload 70B-1M --emulate-shard 0/8)")
    ap.add_argument("--ranks-share-gpu", action="store_true",
                    help="validation only: every rank uses cuda:0 and the output gather goes through gloo")
    args = ap.parse_args()
    if args.warmup < 3:
        log("bench: warmup < 3 is not a valid measurement; using 3")
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if args.ranks_share_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    pg = None
    if world > 1:
        if args.ranks_share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        pg = dist.group.WORLD
    try:
        run_ours(args, rank, world, local_rank, pg)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
