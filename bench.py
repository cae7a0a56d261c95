"""bench.py -- HeadInfer head-wise offloaded attention on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload auto|8B-1M|8B-128K|tiny]

A "step" (ours): one pass of the hot path over one batch of synthetic input --
  prefill step = one 18944-token chunk (148 SMs x 256 rows / g) through all 32 layers (write-back D2H, history
                 H2D through the staging slots, causal attention over history + chunk, per layer call; at N > 1
                 the per-layer NCCL all-gather of the head-sharded outputs).  EVERY step (warm-up and timed) is
                 the SAME chunk, the last one of the 1M prefill (positions [S - c, S), history S - c): the layer
                 cursors are rewound before each step, and re-running a chunk rewrites identical host bytes.  So
                 `value` does not depend on --steps, and it is the most expensive chunk of the prefill
                 (conservative: the paper's 516 tok/s averages all chunks of a 1M prefill).  The history
                 below it is placed in the host store untimed (hi_write_host_kv, App. E P:L1010 "preparing
                 decoding with large context").
  decode step  = one token through all 32 layers at context S (H2D of the whole history), again the same
                 position every step.
`value` = prefill tokens/s (whole job: each token is processed by every rank for its own heads, so scaling is
strong); decode ms/token and host-link GB/s ride along.  Inputs are generated on the GPU by synth/ (seeded,
bit-identical to the oracle's generator) and are resident in HBM before the timed region (`value`); `e2e` re-runs
the timed chunk through the public API from pinned HOST buffers, with each layer's Q/K/V H2D (prefetched one
layer ahead on a side stream) and the D2H of its `out` inside the timed region.  Inputs per step (>= 6 GiB)
exceed the 126 MB L2, so no extra flush is needed.

Multi-GPU: `--gpus N` with N > 1 launched without torchrun re-executes itself under
`torch.distributed.run` (one rank per GPU, NCCL); under torchrun each rank runs on cuda:LOCAL_RANK with its own
context, head shard and NUMA-local host store.  NCCL init logging (NCCL_DEBUG=INFO, SUBSYS=INIT unless the caller
set them) goes to stderr: every rank's C-level stdout is redirected to stderr so that stdout carries exactly one
line, rank 0's JSON.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
    # several layers and kv heads per rank at W = 2: the sharded parity must check layer 0, not the last layer
    "small": (3, 16, 4, 128, 4096, 1024),
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
# parity bars (north_star; R10: relative L2 per (layer, q head) as well, since |o| ~ 1e-3 at 1M under U)
TOL_MAX_ABS, TOL_MEAN_ABS, TOL_REL_L2 = 2e-2, 2e-3, 1e-2

_JSON_FD = None   # the original stdout (fd), kept for the one JSON line


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def emit(res: dict):
    line = (json.dumps(res) + "\n").encode()
    if _JSON_FD is not None:
        os.write(_JSON_FD, line)
    else:
        sys.stdout.write(line.decode())
        sys.stdout.flush()


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
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": statistics.median(pw) if pw else None}


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


def host_store_bytes(wl: str, world: int) -> int:
    L, hq, hkv, d, S, c = WORKLOADS[wl]
    return L * hkv * 4 * d * (S + 16)   # all ranks together


def pick_workload(name: str, world: int) -> str:
    if name != "auto":
        return name
    # the host store (all ranks of this node) must fit with room to spare (a box driven out of memory is a strike)
    if mem_available_bytes() >= host_store_bytes("8B-1M", world) + (24 << 30) + world * (2 << 30):
        return "8B-1M"
    log(f"bench: MemAvailable {mem_available_bytes()/2**30:.0f} GiB too small for the 8B-1M host store; using 8B-128K")
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
    from paper_2502_12574_b200.hostlink import bind_process_to_gpu, measure_link
    from paper_2502_12574_b200.parallel import gather_heads, shard
    from synth.cuda import fill_

    K, W = args.steps, args.warmup
    dev = torch.device("cuda", local_rank)
    cpu_coll = args.ranks_share_gpu   # gloo validation mode: collectives on CPU tensors
    wl = pick_workload(args.workload, world)
    if world > 1:   # every rank must agree on the workload
        t = torch.tensor([list(WORKLOADS).index(wl)], device="cpu" if cpu_coll else dev)
        dist.broadcast(t, 0)
        wl = list(WORKLOADS)[int(t.item())]
    L, hq, hkv, d, S, c = WORKLOADS[wl]
    # head shard: this process's rank, or (--emulate-shard R/W) rank R of a W-GPU job run alone on this GPU
    hr, hw = (rank, world) if args.emulate_shard is None else args.emulate_shard
    sh = shard(hq, hkv, hr, hw)
    node_ranks = world if args.emulate_shard is None else 1
    host_need = host_store_bytes(wl, hw) // hw * node_ranks
    if mem_available_bytes() < host_need + (24 << 30):   # a box driven out of memory is a strike
        raise SystemExit(f"workload {wl}: host store {host_need / 2**30:.0f} GiB does not fit in MemAvailable "
                         f"{mem_available_bytes() / 2**30:.0f} GiB with a 24 GiB margin")
    hq_loc, hkv_loc, q0h, kv0h = sh["q_local"], sh["kv_local"], sh["q"][0], sh["kv"][0]
    p_last = S - c                            # the last chunk of the prefill: positions [S - c, S)
    if p_last < 0:
        raise SystemExit(f"workload {wl}: context {S} shorter than one chunk {c}")
    # the timed chunk: its history is the token-weighted MEAN history of a chunked prefill of S tokens, (S - c)/2;
    # a chunk's work (FLOPs s*c + c^2/2, history H2D 4d*s, write-back 4d*c) is linear in its history s, so
    # c / t(p_t) is the whole-prefill tok/s -- the paper's metric (516 tok/s averages a whole 1M prefill)
    p_t = p_last // 2
    max_ctx = S + 8                           # prefill to S, then decode at S (and S + 1 for parity)
    peaks = rf.load_peaks()
    shape = rf.Shape(L, hq, hkv, d)
    locality = bind_process_to_gpu(local_rank) if torch.cuda.is_available() else {}

    def barrier():
        if world > 1:
            dist.barrier(group=pg)

    # live host-link probe, every rank at once (the decode roofline's denominator under this W-concurrency)
    link = measure_link(local_rank, gib=0.5, reps=3, barrier=barrier if world > 1 else None)
    if world > 1:
        lt = torch.tensor([link["h2d_gbs"], link["d2h_gbs"], link["bidir_gbs"]], dtype=torch.float64,
                          device="cpu" if cpu_coll else dev)
        dist.all_reduce(lt, op=dist.ReduceOp.MIN, group=pg)
        link_min = dict(zip(("h2d_gbs", "d2h_gbs", "bidir_gbs"), lt.tolist()))
    else:
        link_min = {k: link[k] for k in ("h2d_gbs", "d2h_gbs", "bidir_gbs")}

    resident = args.resident_heads
    if resident < 0:  # as many (layer, kv head) pairs as fit next to this bench's inputs (NEXT-1)
        free_b, _ = torch.cuda.mem_get_info()
        inputs_b = 3 * L * c * (hq_loc + 2 * hkv_loc) * d * 2 + 2 * L * c * hq_loc * d * 2
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
                   head_group=args.head_group, device=local_rank, **duo_opts)
    init_s = time.time() - t0
    t0 = time.time()
    fill_history(hi, L, hkv_loc, kv0h, d, p_last, torch, fill_, labels, duo)
    fill_s = time.time() - t0
    log(f"[rank {rank}] {wl}: init {init_s:.1f}s (host store {hi.stats()['host_store_bytes']/2**30:.1f} GiB, "
        f"NUMA node {hi.stats()['numa_node']}), history fill {fill_s:.1f}s; link {link}")

    stream = torch.cuda.current_stream()

    wk = torch.empty((max(args.duo_window, 1), 1, d), dtype=torch.bfloat16, device="cuda") if labels is not None else None
    wv = torch.empty_like(wk) if wk is not None else None

    def refill_windows(pos, layers=None):
        """Duo streaming heads (NEXT-3) keep only their sink rows and a ring of the last `win` rows: a cursor moved
        back to `pos` must get the window below `pos` back (the same generator bytes a prefill wrote there)."""
        ns, win = max(args.duo_sink, 0), args.duo_window
        for l in (range(L) if layers is None else layers):
            for h in range(hkv_loc):
                if not labels[l][kv0h + h]:
                    continue
                lo = max(ns, pos - win)
                if pos > lo:
                    n = pos - lo
                    fill_(wk[:n], SEED, 1, DIST, l, kv0h + h, lo)
                    fill_(wv[:n], SEED, 2, DIST, l, kv0h + h, lo)
                    hi.write_host_kv(l, h, lo, wk[:n, 0], wv[:n, 0])

    def rewind(pos):
        for l in range(L):
            hi.set_seq_len(l, pos)
        if labels is not None:
            refill_windows(pos)

    # ---------------- the step: attention path only (default), or whole synthetic layers (--model, NEXT-4)
    model = None
    synth_tensor_x = 3  # synth.TENSOR_X
    if args.model:
        from paper_2502_12574_b200.layer import HeadInferLayer
        from synth.cuda import fill_matrix_, gen_layer_weights_cuda
        from paper_2502_12574_b200.layer import shard_layer_weights
        from paper_2502_12574_b200.parallel import tp_layer_step
        H, I = MODEL_DIMS
        model = HeadInferLayer(hi, H, I, MODEL_ROPE_THETA, MODEL_RMS_EPS)
        weights = []
        for l in range(L):   # full weights per layer, then this rank's tensor-parallel shard (world > 1)
            wfull = gen_layer_weights_cuda(SEED, l, H, I, hq, hkv, d)
            weights.append(wfull if hw == 1 else shard_layer_weights(wfull, hq, hkv, d, I, hr, hw))
            del wfull
        torch.cuda.synchronize()
        tp_bufs = {"y": torch.empty((c, H), dtype=torch.float32, device="cuda"),
                   "z": torch.empty((c, H), dtype=torch.float32, device="cuda")} if world > 1 else None

    def model_layer(l, x, decode=False):
        if world == 1:
            return model.decode(l, weights[l], x) if decode else model.prefill_chunk(l, weights[l], x)
        n = 1 if decode else x.shape[0]
        return tp_layer_step(model, l, weights[l], x, group=pg, decode=decode,
                             bufs={k: v[:n] for k, v in tp_bufs.items()})

    def make_inputs(pos, n):
        """One step's inputs: per-layer (Q, K, V) for the attention path; x [n, H] for --model."""
        if model is not None:
            return fill_matrix_(torch.empty((n, MODEL_DIMS[0]), dtype=torch.bfloat16, device="cuda"), SEED,
                                synth_tensor_x, 0, row0=pos)
        return [gen_layer_inputs(l, pos, n, hq_loc, hkv_loc, d, q0h, kv0h, torch, fill_) for l in range(L)]

    outs = [torch.empty((c, hq_loc, d), dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    gathered = torch.empty((world, c, hq_loc, d), dtype=torch.bfloat16, device="cuda") if world > 1 else None
    gathered0 = torch.empty_like(gathered) if world > 1 else None
    x_work = None

    def prefill_step(inputs):
        nonlocal x_work
        if model is not None:   # x flows through every layer in place: start every step from the same x
            x_work.copy_(inputs)
            for l in range(L):
                model_layer(l, x_work)
            return
        for l in range(L):
            Q, Kt, Vt = inputs[l]
            hi.prefill_chunk(l, Q, Kt, Vt, outs[l])
            if world > 1:   # Alg. 1 l.15 "Concatenate" across the head shards, on the critical path
                gather_heads(outs[l], group=pg, out=gathered0 if l == 0 else gathered)

    # ---------------- prefill: W warm-up steps, then K timed steps, all at the last chunk [S - c, S) ------
    step_in = make_inputs(p_t, c)
    if model is not None:
        x_work = torch.empty_like(step_in)
    for i in range(W):
        rewind(p_t)
        prefill_step(step_in)
    hi.synchronize()
    st0 = hi.stats()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ms = []
    with ClockSampler(local_rank) as clk_p:
        for i in range(K):
            rewind(p_t)      # cursor reset (+ duo windows put back): between the timed steps, not in them
            es = torch.cuda.Event(enable_timing=True)
            es.record(stream)
            prefill_step(step_in)
            hi.synchronize()  # the step ends when its last write-back has drained
            ee = torch.cuda.Event(enable_timing=True)
            ee.record(stream)
            step_ms.append((es, ee))
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ms]
    pre_ms = sum(step_ms)
    st1 = hi.stats()
    sample_outs = {("mid", 0): outs[0].clone(), ("mid", L - 1): outs[L - 1].clone()} if model is None else {}
    gathered_mid = gathered0.clone() if gathered0 is not None else None   # the last-chunk step below re-gathers

    # ---------------- the last chunk of the prefill (the most expensive one), one step, reported beside ------
    last_in = make_inputs(p_last, c)
    rewind(p_last)
    torch.cuda.synchronize()
    barrier()
    sl0 = hi.stats()
    e0.record(stream)
    prefill_step(last_in)
    hi.synchronize()
    e1.record(stream)
    torch.cuda.synchronize()
    last_ms = e0.elapsed_time(e1)
    sl1 = hi.stats()
    del last_in
    if model is None:
        sample_outs[("last", 0)] = outs[0].clone()
        sample_outs[("last", L - 1)] = outs[L - 1].clone()

    # ---------------- decode: W warm-up tokens, then K timed tokens, all at context S -------------------
    dq = make_inputs(S, 1)
    dout = [torch.empty((hq_loc, d), dtype=torch.bfloat16, device="cuda") for _ in range(L)]
    gdec = torch.empty((world, hq_loc, d), dtype=torch.bfloat16, device="cuda") if world > 1 else None

    def decode_step():
        if model is not None:
            xd = dq[0].clone()
            for l in range(L):
                model_layer(l, xd, decode=True)
            return
        for l in range(L):
            q, k, v = dq[l]
            hi.decode(l, q[0], k[0], v[0], dout[l])
            if world > 1:
                gather_heads(dout[l], group=pg, out=gdec)

    for i in range(W):
        rewind(S)
        decode_step()
    hi.synchronize()
    sd0 = hi.stats()
    torch.cuda.synchronize()
    barrier()
    dec_ms = 0.0
    with ClockSampler(local_rank) as clk_d:
        for i in range(K):
            rewind(S)
            e0.record(stream)
            decode_step()
            hi.synchronize()
            e1.record(stream)
            torch.cuda.synchronize()
            dec_ms += e0.elapsed_time(e1)
    barrier()
    sd1 = hi.stats()
    dec_sample = dout[0].clone() if model is None else None
    if gdec is not None:   # the parity check is on layer 0: gather its decode output again (gdec holds the last layer's)
        gather_heads(dout[0], group=pg, out=gdec)
    gdec_sample = gdec.clone() if gdec is not None else None

    # ---------------- e2e: the timed chunk again, inputs from pinned HOST memory --------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(hi, model_layer if model is not None else None, None, step_in, outs, L, c, K, W, p_t, rewind,
                      world, pg, gathered, barrier, stream, torch, ref_outs=sample_outs)
    del step_in

    # ---------------- max over ranks --------------------------------------------------------------
    times = torch.tensor([pre_ms, dec_ms, e2e["ms"] if e2e else 0.0], dtype=torch.float64,
                         device="cpu" if cpu_coll else dev)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX, group=pg)
    pre_ms, dec_ms, e2e_ms = times.tolist()

    # ---------------- parity (and, at N = 1, the cpu baseline) on sampled rows ------------------------------
    parity, cpu = None, None
    if not args.no_cpu_baseline and model is None:
        if world == 1:
            parity, cpu = full_size_parity(hi, sample_outs, dec_sample, p_t, p_last, S, L, hq, hkv, d, c, torch,
                                           labels=labels, duo=duo, kv0=kv0h, hkv_loc=hkv_loc, q0=q0h,
                                           restore=(lambda pos: refill_windows(pos, [0])) if labels is not None else None)
        else:
            parity = sharded_parity(gathered_mid, gdec_sample, p_t, S, L, hq, hkv, d, world, rank, pg, torch,
                                    labels, duo)

    # ---------------- report (rank 0) -------------------------------------------------------------
    if rank != 0:
        hi.close()
        return None
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
    # step rooflines: measured peaks; sustained tensor peak inside a long step; host link measured live in this run
    # under the same W-concurrency (min over ranks)
    pk = dict(peaks, bf16_tflops=peak_t, **link_min)
    R = st1["resident_kv_heads"]
    dk = dict(streaming=st1["streaming_kv_heads"], n_sink=max(args.duo_sink, 0), win=args.duo_window)
    roof_p = rf.step_roofline_seconds(rf.prefill_step(shape, p_t, c, hw, R, **dk), pk)
    roof_last = rf.step_roofline_seconds(rf.prefill_step(shape, p_last, c, hw, R, **dk), pk)
    t_roof_pre = K * roof_p["seconds"]
    roof_d = rf.step_roofline_seconds(rf.decode_step(shape, S, hw, R, **dk), pk)
    t_roof_dec = K * roof_d["seconds"]
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
    rank_pre_ms = pre_ms   # max over ranks (the copy statistics are rank 0's)
    prefill_copies = {
        "h2d_bytes_per_step": int(pf_h2d_b / K), "d2h_bytes_per_step": int(pf_d2h_b / K),
        "h2d_busy_ms_per_step": round(pf_h2d_ms / K, 3), "d2h_busy_ms_per_step": round(pf_d2h_ms / K, 3),
        "h2d_gbs_while_busy": round(pf_h2d_b / (pf_h2d_ms / 1e3) / 1e9, 2) if pf_h2d_ms > 0 else None,
        "d2h_gbs_while_busy": round(pf_d2h_b / (pf_d2h_ms / 1e3) / 1e9, 2) if pf_d2h_ms > 0 else None,
        "h2d_busy_frac_of_step": round(pf_h2d_ms / rank_pre_ms, 4) if rank_pre_ms else None,
        "attention_frac_of_step": round(pf_ms / rank_pre_ms, 4) if rank_pre_ms else None,
        "copy_hidden_frac": (round(max(0.0, min(1.0, (pf_ms + pf_h2d_ms - rank_pre_ms) / pf_h2d_ms)), 4)
                             if pf_h2d_ms > 0 else None)}
    clk = clk_p.summary()
    per_step = sorted(step_ms)

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
                   "parallelism": (f"head-shard{world}" + (" (ranks share cuda:0, gloo)" if cpu_coll else "")
                                   if args.emulate_shard is None else
                                   f"rank {hr} of head-shard{hw}, run alone on 1 GPU (no all-gather)"),
                   "prefill_step": "1 chunk x all layers (+ per-layer all-gather at N > 1)",
                   "timed_chunk": [p_t, p_t + c], "timed_chunk_note": "every warm-up and timed step re-runs the chunk "
                   "whose history is the token-weighted mean history of the whole S-token chunked prefill, (S - c)/2 "
                   "(cursor rewound): per-chunk work is linear in the history, so value = the whole-prefill tok/s, "
                   "independent of --steps; the last (most expensive) chunk is in last_chunk",
                   "decode_step": "1 token x all layers", "decode_context": S,
                   "l2": "inputs per step > L2 (>= 6 GiB), no flush needed"},
        "prefill_step_ms": {"min": round(per_step[0], 3), "median": round(per_step[len(per_step) // 2], 3),
                            "max": round(per_step[-1], 3), "rank": 0},
        "last_chunk": {"positions": [p_last, S], "tok_s": round(c / (last_ms / 1e3), 2), "ms": round(last_ms, 3),
                       "kernel_tflops": round((sl1["prefill_attn_flops"] - sl0["prefill_attn_flops"]) /
                                              max(sl1["prefill_attn_ms"] - sl0["prefill_attn_ms"], 1e-9) / 1e9, 1),
                       "step_roofline_frac": round(roof_last["seconds"] / (last_ms / 1e3), 4),
                       "note": "one step of the most expensive chunk (history S - c), rank 0, after the timed steps"},
        "decode": {"ms_per_token": round(dec_ms_tok, 3), "h2d_gbs": round(h2d_gbs, 2),
                   "link_peak_gbs": round(link_min["h2d_gbs"], 2), "link_frac": round(h2d_gbs / link_min["h2d_gbs"], 4),
                   "link_peak_source": f"measured live in this run, {world} rank(s) copying concurrently, min over ranks",
                   "roofline_frac": round(t_roof_dec / (dec_ms / 1e3), 4), "roofline_bound": roof_d["bound"],
                   "h2d_bytes_per_token": int(h2d_dec),
                   "kernel": {"bound": "hbm", "achieved_gbs": round(dk_bytes / (dk_ms / 1e3) / 1e9, 1) if dk_ms else None,
                              "peak_gbs": peaks["hbm_gbs"],
                              "frac": round(dk_bytes / (dk_ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4) if dk_ms else None},
                   "clocks": clk_d.summary()},
        "host_link": {"rank0": link, "min_over_ranks": link_min, "committed_1gpu": {k: v for k, v in rf.HOST_LINK.items()},
                      "locality_rank0": {k: v for k, v in locality.items() if k != "affinity"}},
        "prefill_copies": prefill_copies,
        "prefill_step_roofline": {"frac": round(t_roof_pre / (pre_ms / 1e3), 4), "bound": roof_p["bound"],
                                  "t_roof_s": round(t_roof_pre, 4), "t_meas_s": round(pre_ms / 1e3, 4)},
        "roofline": {"bound": "tensor", "kernel": "prefill attention (history + causal segments)",
                     "achieved": round(achieved_tflops, 2) if achieved_tflops else None,
                     "peak": peak_t, "unit": "TFLOP/s",
                     "frac": round(achieved_tflops / peak_t, 4) if achieved_tflops else None,
                     "traffic": traffic, "traffic_source": "committed ncu --set full capture of the dominant launch "
                                                           "(profiles/ncu_prefill_traffic.json), not this run",
                     "launches": pf_launches,
                     "flops_per_launch": pf_flops / max(pf_launches, 1),
                     "peak_source": peaks["source"] + " bf16_tflops_sustained"},
        "clocks": clk,
        "gpu_launches": launches,
        "residency": {"staging_bytes": st1["staging_bytes"], "staging_bound_bytes": st1["staging_bound_bytes"],
                      "one_head_bytes": 4 * d * max_ctx,
                      "head_group": st1["head_group"], "numa_node": st1["numa_node"],
                      "host_store_bytes": st1["host_store_bytes"], "init_s": round(init_s, 2),
                      "resident_kv_heads": st1["resident_kv_heads"], "resident_bytes": st1["resident_bytes"]},
    }
    if world > 1:
        res["nccl"] = {"backend": dist.get_backend(pg), "comm_nranks": dist.get_world_size(pg),
                       "collective": "all_gather_into_tensor of each layer call's out (prefill and decode)",
                       "init_log": "NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT on stderr"}
    if e2e:
        res["e2e"] = {"value": round(K * c / (e2e_ms / 1e3), 2), "unit": "tok/s",
                      "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                      "bit_identical_to_resident_run": e2e.get("bit_identical_to_resident_run"),
                      "overlap": "layer l+1's Q/K/V H2D on a side stream under layer l's attention; out D2H on "
                                 "another side stream"}
    if parity is not None:
        res["parity_sample"] = parity
    if cpu is not None:
        res["cpu_baseline"] = cpu
    if model is not None:
        H, I = MODEL_DIMS
        gemm_tok = L * 2.0 * (H * (hq + 2 * hkv) * d + H * hq * d + 3 * H * I)  # QKV, O, gate+up, down
        t_gemm = K * c * gemm_tok / hw / (peak_t * 1e12)   # each rank runs 1/W of the projections (tensor parallel)
        res["config"]["path"] = ("synthetic Llama-3-8B decoder layers (NEXT-4): RMSNorm, QKV/O/MLP GEMMs, RoPE, SwiGLU"
                                 + (f"; tensor parallel over {world} ranks (2 all-reduces per layer)" if world > 1 else ""))
        res["data"] = ("synthetic (seeded counter-hash generator): hidden states in, random-init Llama-3-8B layer "
                       "weights (no trained weights, no embedding / LM head)")
        res["config"]["hidden"], res["config"]["intermediate"] = H, I
        res["model"] = {"prefill_tok_s": round(tok_s, 2), "decode_ms_per_token": round(dec_ms_tok, 3),
                        "gemm_flops_per_token": gemm_tok,
                        "attention_share_of_prefill": round(pf_ms / pre_ms, 4) if pre_ms else None,
                        "step_roofline_frac": round((t_roof_pre + t_gemm) / (pre_ms / 1e3), 4),
                        "parity": "tests/test_gpu_layer.py (layer oracle, incl. one 8B-shaped layer)",
                        "note": "history K/V below the timed chunk are synthetic (placed untimed), not produced "
                                "by running the layers; no embedding / LM head"}
        model.close()
    if args.emulate_shard is not None:
        res["shard_emulation"] = {
            "rank": hr, "world": hw, "kv_heads": list(sh["kv"]), "q_heads": list(sh["q"]),
            "note": "one rank's share of a head-sharded job, measured alone on one GPU: every rank does the same "
                    "work on its own heads (no K/V crosses GPUs), so value is the job's tok/s if the W ranks run "
                    "as fast as this one; the per-layer output all-gather and any host-link sharing between "
                    "ranks are not measured"}
    hi.close()
    return res


def run_e2e(hi, model, weights, step_in, outs, L, c, K, W, p_last, rewind, world, pg, gathered, barrier, stream, torch,
            ref_outs=None):
    """The timed chunk through the public API from pinned HOST buffers: per step, every layer's Q/K/V go host ->
    device (double-buffered, layer l+1's copy on a side stream under layer l's attention) and every layer's `out`
    device -> host (side stream); both inside the timed region."""
    from paper_2502_12574_b200.parallel import gather_heads
    if model is not None:   # x in, x out (the last layer's hidden states)
        host_x = step_in.cpu().pin_memory()
        host_out = torch.empty_like(host_x).pin_memory()
        dev_x = torch.empty_like(step_in)
        e2e_ms = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(W + K):
            rewind(p_last)
            torch.cuda.synchronize()
            barrier()
            e0.record(stream)
            dev_x.copy_(host_x, non_blocking=True)
            for l in range(L):
                model(l, dev_x)   # model_layer: the single-rank layer, or the tensor-parallel one
            host_out.copy_(dev_x, non_blocking=True)
            hi.synchronize()
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= W:
                e2e_ms += e0.elapsed_time(e1)
        return {"ms": e2e_ms, "h2d": host_x.numel() * 2, "d2h": host_out.numel() * 2 * world}
    host_in = [[t.cpu().pin_memory() for t in per] for per in step_in]
    host_out = [torch.empty(outs[0].shape, dtype=torch.bfloat16).pin_memory() for _ in range(L)]
    dev_in = [[torch.empty_like(t) for t in step_in[0]] for _ in range(2)]
    dev_out = [torch.empty_like(outs[0]) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_ready = [torch.cuda.Event() for _ in range(2)]
    ev_in_free = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out_free = [torch.cuda.Event() for _ in range(2)]
    h2d_b = sum(t.numel() * 2 for per in host_in for t in per)
    d2h_b = sum(t.numel() * 2 for t in host_out) * world

    def issue_in(l):
        b = l % 2
        s_in.wait_event(ev_in_free[b])           # layer l-2's attention has read this buffer
        with torch.cuda.stream(s_in):
            for t_dev, t_host in zip(dev_in[b], host_in[l]):
                t_dev.copy_(t_host, non_blocking=True)
        ev_ready[b].record(s_in)

    for ev in ev_in_free + ev_out_free:
        ev.record(stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_ms = 0.0
    for i in range(W + K):
        rewind(p_last)
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        s_in.wait_stream(stream)
        issue_in(0)
        for l in range(L):
            b = l % 2
            if l + 1 < L:
                issue_in(l + 1)
            stream.wait_event(ev_ready[b])
            stream.wait_event(ev_out_free[b])    # layer l-2's out has reached the host
            hi.prefill_chunk(l, *dev_in[b], dev_out[b])
            ev_in_free[b].record(stream)
            if world > 1:
                gather_heads(dev_out[b], group=pg, out=gathered)
            ev_done[b].record(stream)
            s_out.wait_event(ev_done[b])
            with torch.cuda.stream(s_out):
                host_out[l].copy_(dev_out[b], non_blocking=True)
            ev_out_free[b].record(s_out)
        stream.wait_stream(s_out)
        hi.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= W:
            e2e_ms += e0.elapsed_time(e1)
    # the e2e outputs are the same chunk as the timed one: they must equal the resident-input outputs bit for bit
    same = all(torch.equal(host_out[l], ref_outs[("mid", l)].cpu()) for l in (0, L - 1))
    if not same:
        log("bench: WARNING e2e outputs differ from the resident-input run")
    return {"ms": e2e_ms, "h2d": h2d_b, "d2h": d2h_b, "bit_identical_to_resident_run": same}


# ---------------------------------------------------------------------------------------------
def _oracle_kv(layer, kv_head, upto, d, torch):
    """K, V of (layer, kv head) positions [0, upto) from synth's GPU twin (bit-identical to synth.gen_block,
    pinned by tests) -> host numpy; the oracle never reads the library."""
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


class ParityAcc:
    """max-abs / mean-abs over everything, relative L2 per (layer, q head) (reading R10)."""

    def __init__(self):
        import numpy as np
        self.np = np
        self.maxerr, self.sumerr, self.cnt, self.rows = 0.0, 0.0, 0, 0
        self.sq = {}   # (layer, q head) -> [sum (o - ref)^2, sum ref^2]

    def add(self, layer, qhead, got, ref):
        np = self.np
        err = np.abs(got - ref)
        self.maxerr = max(self.maxerr, float(err.max()))
        self.sumerr += float(err.sum())
        self.cnt += err.size
        self.rows += got.shape[0]
        a = self.sq.setdefault((layer, qhead), [0.0, 0.0])
        a[0] += float(((got - ref) ** 2).sum())
        a[1] += float((ref ** 2).sum())

    def result(self, prefix=""):
        rel = {k: (v[0] ** 0.5) / max(v[1] ** 0.5, 1e-300) for k, v in self.sq.items()}
        worst = max(rel, key=rel.get) if rel else None
        return {f"{prefix}rows": self.rows, f"{prefix}max_abs": self.maxerr,
                f"{prefix}mean_abs": self.sumerr / max(self.cnt, 1),
                f"{prefix}rel_l2_max": rel[worst] if worst else None,
                f"{prefix}rel_l2_worst_layer_qhead": list(worst) if worst else None,
                f"{prefix}qheads_checked": len({k[1] for k in rel}),
                f"{prefix}ok": bool(self.maxerr <= TOL_MAX_ABS and self.sumerr / max(self.cnt, 1) <= TOL_MEAN_ABS
                                    and (not rel or rel[worst] <= TOL_REL_L2))}


def full_size_parity(hi, sample_outs, dec_sample, p_t, p_last, S, L, hq, hkv, d, c, torch, labels=None, duo=(0, 0),
                     kv0=0, hkv_loc=None, q0=0, restore=None):
    """Sampled full-size parity + the cpu baseline (SURVEY.md §8(d) "Timing procedure"), at N = 1:
      * GPU outputs of layer 0 at the first, middle and last chunk (the last = the timed one; the first and middle
        are re-run untimed through the same API) and of layer L-1 at the last chunk;
      * >= 4096 (layer, q head, position) rows covering EVERY q head, the first and last row of each of those
        chunks plus random rows, checked against the fp64 oracle (max-abs, mean-abs, rel-L2 per (layer, q head));
      * the decode token at S (timed run) and at S + 1 (one more decode of layer 0), every q head of layer 0:
        the full-oracle decode of one layer for 2 steps;
      * the oracle's time on these rows gives key-visits/s on this box's cores, the baseline's tok/s on the
        timed chunk, and an EXTRAPOLATED full 1M-prefill oracle time."""
    import numpy as np

    import oracle
    import synth
    from synth.cuda import fill_
    oracle.build()
    g = hq // hkv
    hkv_loc = hkv if hkv_loc is None else hkv_loc
    hq_loc = hkv_loc * g
    own = list(range(kv0, kv0 + hkv_loc))
    strm = {(l, h): bool(labels is not None and labels[l][h]) for l in (0, L - 1) for h in own}
    cores = oracle.num_threads()
    # GPU: the timed (mean-history) chunk and the last chunk are in sample_outs; layer 0 at the first chunk is
    # re-run untimed through the same API (it rewrites identical host rows), then one more decode at S + 1
    chunk_out = dict(sample_outs)
    hi.set_seq_len(0, 0)
    Q, Kt, Vt = gen_layer_inputs(0, 0, c, hq_loc, hkv_loc, d, q0, kv0, torch, fill_)
    chunk_out[("first", 0)] = hi.prefill_chunk(0, Q, Kt, Vt).clone()
    hi.set_seq_len(0, S + 1)   # rows [0, S] hold the prefill and the decode token at S
    if restore is not None:    # duo streaming heads: their window below S + 1 (the e2e leg re-ran an earlier chunk)
        restore(S + 1)
    qd1 = [fill_(torch.empty((1, n, d), dtype=torch.bfloat16, device="cuda"), SEED, t, DIST, 0, h0, S + 1)[0]
           for t, n, h0 in ((0, hq_loc, q0), (1, hkv_loc, kv0), (2, hkv_loc, kv0))]
    dec_next = hi.decode(0, *qd1).clone()
    hi.synchronize()
    chunk_pos = {"first": 0, "mid": p_t, "last": p_last}
    rng = np.random.default_rng(0)
    # row plan per q head: first/last row of every sampled chunk + random rows; the first chunk is cheap, so it
    # carries most rows; >= 4096 rows in total over the sampled chunks
    per_head = max(1, -(-4096 // hq_loc))
    plan = {}   # (layer, name) -> token indices within the chunk
    names = [n for n in ("first", "mid", "last") if (n, 0) in chunk_out]
    n_last = max(2, min(24, per_head // 4))
    n_mid = max(2, min(24, per_head // 4)) if "mid" in names else 0
    n_first = per_head - n_last - n_mid
    for name, n in (("first", n_first), ("mid", n_mid), ("last", n_last)):
        if name in names:
            plan[(0, name)] = np.unique(np.concatenate([[0, c - 1], rng.integers(1, c - 1, max(0, n - 2))]))
    if L > 1:
        plan[(L - 1, "last")] = np.array([0, c // 2, c - 1])
        plan[(L - 1, "mid")] = np.array([0, c - 1])
    kvcache = {}

    def kv_of(layer, h):
        if (layer, h) not in kvcache:
            kvcache[(layer, h)] = _oracle_kv(layer, h, S + 2, d, torch)
        return kvcache[(layer, h)]

    acc = ParityAcc()
    visits, t_oracle = 0.0, 0.0
    for (layer, name), toks in plan.items():
        pos0 = chunk_pos[name]
        qblk = synth.gen_block(SEED, 0, DIST, layer, q0, hq_loc, pos0, c, d)
        got = chunk_out[(name, layer)].float().cpu().numpy()
        for h in own:
            k, v = kv_of(layer, h)
            js = list(range(h * g - q0, (h + 1) * g - q0))            # local q heads of kv head h
            qrows = qblk[toks][:, js].transpose(1, 0, 2).reshape(-1, d)  # all g heads' rows in one oracle call
            last = np.tile(pos0 + toks, g)
            t0 = time.time()
            ref = _oracle_rows(oracle, qrows, last, k, v, strm.get((layer, h), False), duo).reshape(g, len(toks), d)
            t_oracle += time.time() - t0
            visits += float((last + 1).sum())
            for jj, jl in enumerate(js):
                acc.add(layer, q0 + jl, got[toks, jl], ref[jj])
    # decode: every q head of layer 0 at S (timed decode) and S + 1
    dacc = ParityAcc()
    t_dec = 0.0
    for pos, out in ((S, dec_sample), (S + 1, dec_next)):
        qd = synth.gen_block(SEED, 0, DIST, 0, q0, hq_loc, pos, 1, d)[0]
        got = out.float().cpu().numpy()
        for h in own:
            k, v = kv_of(0, h)
            t0 = time.time()
            ref = _oracle_rows(oracle, qd[(h - kv0) * g:(h - kv0 + 1) * g], np.full(g, pos), k, v,
                               strm.get((0, h), False), duo)
            t_dec += time.time() - t0
            for jj in range(g):
                dacc.add(0, h * g + jj, got[(h - kv0) * g + jj][None], ref[jj][None])
    parity = {**acc.result("prefill_"), **dacc.result("decode_"),
              "chunks": {n: [chunk_pos[n], chunk_pos[n] + c] for n in names}, "layers": sorted({k[0] for k in plan}),
              "tol_max_abs": TOL_MAX_ABS, "tol_mean_abs": TOL_MEAN_ABS, "tol_rel_l2": TOL_REL_L2}
    parity["ok"] = parity["prefill_ok"] and parity["decode_ok"]
    if not parity["ok"]:
        log(f"bench: PARITY FAILURE {parity}")
    # cpu baseline: key visits per second of the fp64 oracle on this box's cores (work per row = keys visited)
    kv_rate = visits / max(t_oracle, 1e-9)
    visits_timed_tok = L * hq * (p_t + (c + 1) / 2.0)           # key visits per token of the timed chunk
    full_visits = L * hq * S * (S + 1) / 2.0                     # the whole causal prefill of S tokens
    cpu = {"value": round(kv_rate / visits_timed_tok, 6), "unit": "tok/s", "cores": cores, "kind": "oracle",
           "sample": f"{acc.rows} (layer, q head, position) prefill rows over every q head of layers "
                     f"{sorted({k[0] for k in plan})}, first/last + random rows of chunks {names} "
                     f"({t_oracle:.1f} s), + {dacc.rows} decode rows (layer 0, positions {S}, {S + 1}; {t_dec:.1f} s)",
           "rows_per_s": round(acc.rows / max(t_oracle, 1e-9), 2), "key_visits_per_s": round(kv_rate, 1),
           "value_definition": "key_visits_per_s / key visits per token of the timed chunk (L x Hq x (s + (c+1)/2))",
           "decode_full_oracle_s_per_layer_token": float(f"{t_dec / 2:.4g}"),
           "decode_full_oracle_s_per_token_extrapolated": float(f"{t_dec / 2 * L:.4g}"),
           "extrapolated_full_prefill_oracle_s": float(f"{full_visits / kv_rate:.4g}"),
           "extrapolated_note": "EXTRAPOLATED, not run: L x Hq x S(S+1)/2 key visits at the measured rate"}
    return parity, cpu


def sharded_parity(gathered0, gdec, p_last, S, L, hq, hkv, d, world, rank, pg, torch, labels=None, duo=(0, 0),
                   n_tok=6):
    """Head-sharded run: rows of the all-gathered layer-0 output of the timed chunk for EVERY q head (so every
    rank's shard and the collective are checked end to end), and the gathered decode output at S, against the
    oracle.  The rows are split over the ranks (each rank checks the q heads of its own kv heads against the
    GATHERED tensor, then the results are reduced)."""
    import numpy as np

    import oracle
    import synth
    import torch.distributed as dist
    from paper_2502_12574_b200.parallel import to_token_major
    oracle.build()
    c = gathered0.shape[1]
    full = to_token_major(gathered0).float().cpu().numpy()       # [c, hq, d]
    dfull = to_token_major(gdec).float().cpu().numpy()           # [hq, d]
    g = hq // hkv
    toks = np.array([0, 1, c // 3, c // 2, 2 * c // 3, c - 1][:n_tok])
    qblk = synth.gen_block(SEED, 0, DIST, 0, 0, hq, p_last, c, d)
    qd = synth.gen_block(SEED, 0, DIST, 0, 0, hq, S, 1, d)[0]
    acc, dacc = ParityAcc(), ParityAcc()
    for h in range(rank * hkv // world, (rank + 1) * hkv // world):
        k, v = _oracle_kv(0, h, S + 1, d, torch)
        st = bool(labels is not None and labels[0][h])
        for j in range(h * g, (h + 1) * g):
            acc.add(0, j, full[toks, j], _oracle_rows(oracle, qblk[toks, j], p_last + toks, k, v, st, duo))
            dacc.add(0, j, dfull[j][None], _oracle_rows(oracle, qd[j][None], np.array([S]), k, v, st, duo))
    pr, dr = acc.result("prefill_"), dacc.result("decode_")
    on = "cpu" if dist.get_backend(pg) == "gloo" else "cuda"
    vals = torch.tensor([pr["prefill_max_abs"], pr["prefill_rel_l2_max"] or 0.0, dr["decode_max_abs"],
                         dr["decode_rel_l2_max"] or 0.0, float(not (pr["prefill_ok"] and dr["decode_ok"]))],
                        dtype=torch.float64, device=on)
    rows = torch.tensor([pr["prefill_rows"], dr["decode_rows"]], dtype=torch.float64, device=on)
    dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=pg)
    dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=pg)
    vals, rows = vals.cpu(), rows.cpu()
    v = vals.tolist()
    return {"gathered_prefill_rows": int(rows[0]), "qheads_checked": hq, "prefill_max_abs": v[0],
            "prefill_rel_l2_max": v[1], "gathered_decode_rows": int(rows[1]), "decode_max_abs": v[2],
            "decode_rel_l2_max": v[3], "ok": v[4] == 0.0, "chunk": [p_last, p_last + c], "layer": 0,
            "tol_max_abs": TOL_MAX_ABS, "tol_rel_l2": TOL_REL_L2}


# ---------------------------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle (as it stands) on this box's host cores, same metric/config.
    Each step is a bounded sample of the workload: rows of the ours arm's timed chunk (the mean-history chunk at
    (S - c)/2, whose per-token work is the whole prefill's average)."""
    if rank != 0:
        return None
    import numpy as np
    import torch

    import oracle
    import synth
    oracle.build()
    wl = args.workload if args.workload != "auto" else "8B-1M"
    L, hq, hkv, d, S, c = WORKLOADS[wl]
    g = hq // hkv
    pos = (S - c) // 2   # the ours arm's timed chunk (p_t in run())
    if torch.cuda.is_available():
        k, v = _oracle_kv(0, 0, pos + c, d, torch)
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
    return {"impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same generator and workload as the ours arm)",
            "config": {"workload": wl, "layers": L, "q_heads": hq, "kv_heads": hkv, "head_dim": d, "context": S,
                       "chunk": c, "timed_chunk": [pos, pos + c], "parallelism": "host cores"},
            "cpu_baseline": {"value": round(val, 6), "unit": "tok/s", "cores": cores, "kind": "oracle",
                             "sample": f"per step {rows_per_step} (layer 0, q head, position) rows of the chunk at "
                                       f"{pos}; tok/s = rows/s / ({L} x {hq})"},
            "e2e": {"value": round(val, 6), "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) without torchrun: re-execute this script as N ranks (one per GPU) on this node."""
    n = args.gpus
    if not args.ranks_share_gpu:
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < n:
            raise SystemExit(f"--gpus {n}: only {have} GPU(s) visible (use --ranks-share-gpu for a 1-GPU validation)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    log("bench: launching " + " ".join(cmd[2:]))
    return subprocess.call(cmd, cwd=ROOT)


def main():
    global _JSON_FD
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
                    help="validation only: every rank uses cuda:0 and the collectives go through gloo")
    args = ap.parse_args()
    if args.warmup < 3:
        log("bench: warmup < 3 is not a valid measurement; using 3")
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        log(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}: running {world} ranks")
    if args.impl == "reference":   # rank 0 alone runs the oracle (the other ranks of a torchrun launch exit 0)
        res = run_reference(args, rank, max(world, args.gpus))
        if res is not None:
            emit(res)
        return
    # stdout carries exactly one line (rank 0's JSON): C-level stdout (NCCL's INFO log) goes to stderr
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
    res = None
    try:
        res = run_ours(args, rank, world, local_rank, pg)
        if world > 1:
            dist.barrier(group=pg)
    finally:
        if world > 1:
            dist.destroy_process_group()
    if res is not None:
        emit(res)


if __name__ == "__main__":
    main()
