"""Concurrent host-link probe (host-link bandwidth "alone and with all 8 GPUs concurrent"; §8(e)
scaling caveat).  One process per GPU, each pinned to its GPU's local CPUs (its pinned buffers are first-
touched on that NUMA node); H2D, D2H and both directions are timed with CUDA events, first on GPU 0 alone,
then on all N GPUs in lock-step (a barrier before every timed copy).

    python tools/probe_link.py [--gpus N] [--gib 1] [--reps 3]   ->  one JSON line (stdout)

The per-GPU concurrent H2D figure is the decode roofline's host-link denominator at that N (bench.py measures
the same thing live inside each run; this tool is the stand-alone version for profiles/).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, n, gib, reps, barrier, q):
    from paper_2502_12574_b200.hostlink import bind_process_to_gpu, measure_link
    torch.cuda.set_device(rank)
    loc = bind_process_to_gpu(rank)
    alone = None
    if rank == 0:
        alone = measure_link(0, gib, reps)
    barrier.wait()
    conc = measure_link(rank, gib, reps, barrier=barrier.wait)
    q.put((rank, {"locality": {k: v for k, v in loc.items() if k != "affinity"},
                  "affinity_cpus": len(loc["affinity"]), "alone": alone, "concurrent": conc}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count() if torch.cuda.is_available() else 1)
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = min(a.gpus, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(n), ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, n, a.gib, a.reps, barrier, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(n))
    for p in procs:
        p.join()
    conc = [res[r]["concurrent"] for r in range(n)]
    out = {"n_gpus": n, "gib": a.gib, "reps": a.reps,
           "alone_gpu0": res[0]["alone"],
           "concurrent_per_gpu": {str(r): res[r]["concurrent"] for r in range(n)},
           "concurrent_min_per_gpu": {k: min(c[k] for c in conc) for k in ("h2d_gbs", "d2h_gbs", "bidir_gbs")},
           "concurrent_aggregate": {k: round(sum(c[k] for c in conc), 2) for k in ("h2d_gbs", "d2h_gbs", "bidir_gbs")},
           "locality": {str(r): res[r]["locality"] for r in range(n)}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
