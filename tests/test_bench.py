"""bench.py's JSON contract, run as the driver runs it (a subprocess printing one JSON line).

CPU: the reference arm (`--impl reference`, the fp64 oracle on host cores) on the tiny workload.
GPU: the tiny workload through the product path, at N=1 and as one rank's share of a head-sharded
job (`--emulate-shard 1/2`: kv head 1 and its q heads only), checking the keys the driver reads
and the sampled parity against the oracle."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    res = run_bench("--impl", "reference", "--workload", "tiny", "--steps", "2", "--warmup", "3")
    assert res["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in res, k
    assert res["value"] > 0 and res["steps"] == 2
    assert res["cpu_baseline"]["kind"] == "oracle" and res["cpu_baseline"]["cores"] >= 1
    assert res["e2e"]["h2d_bytes_per_step"] == 0 and res["e2e"]["d2h_bytes_per_step"] == 0
    assert res["config"]["workload"] == "tiny"


def _check_ours(res):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches", "decode", "parity_sample"):
        assert k in res, k
    assert res["value"] > 0 and res["gpu_launches"] > 0
    rl = res["roofline"]
    assert rl["bound"] == "tensor" and rl["unit"] == "TFLOP/s" and rl["achieved"] > 0
    assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    ps = res["parity_sample"]
    assert ps["prefill_rows"] > 0 and ps["prefill_max_abs"] <= 2e-2 and ps["prefill_mean_abs"] <= 2e-3
    assert ps["prefill_rel_l2_max"] <= 1e-2 and ps["decode_rel_l2_max"] <= 1e-2
    assert ps["decode_max_abs"] <= 2e-2 and ps["ok"]
    # every q head of the shard is checked, at the first, middle and last chunk, and 2 decode steps
    assert ps["prefill_qheads_checked"] == res["config"]["q_heads"] // res.get("shard_emulation", {}).get("world", 1)
    assert set(ps["chunks"]) == {"first", "mid", "last"} and ps["decode_rows"] == 2 * ps["decode_qheads_checked"]
    cb = res["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["extrapolated_full_prefill_oracle_s"] > 0 and "EXTRAPOLATED" in cb["extrapolated_note"]
    assert res["e2e"]["h2d_bytes_per_step"] > 0 and res["e2e"]["d2h_bytes_per_step"] > 0
    S, c = res["config"]["context"], res["config"]["chunk"]
    assert res["config"]["timed_chunk"] == [(S - c) // 2, (S - c) // 2 + c]   # the mean-history chunk
    assert res["last_chunk"]["positions"] == [S - c, S] and res["last_chunk"]["tok_s"] > 0
    assert res["e2e"]["bit_identical_to_resident_run"]
    assert res["host_link"]["min_over_ranks"]["h2d_gbs"] > 0


@pytest.mark.gpu
def test_bench_tiny_contract():
    res = run_bench("--workload", "tiny", "--steps", "2", "--warmup", "3")
    _check_ours(res)
    assert res["config"]["workload"] == "tiny" and res["n_gpus"] == 1
    assert "shard_emulation" not in res


@pytest.mark.gpu
def test_bench_emulated_shard():
    """Rank 1 of a 2-way head shard run alone: kv head 1 (global) and q heads 2, 3 of the tiny config; the
    sampled rows are checked against the oracle at their GLOBAL head indices."""
    res = run_bench("--workload", "tiny", "--steps", "2", "--warmup", "3", "--emulate-shard", "1/2")
    _check_ours(res)
    em = res["shard_emulation"]
    assert em["rank"] == 1 and em["world"] == 2 and em["kv_heads"] == [1, 2] and em["q_heads"] == [2, 4]
    assert "rank 1 of head-shard2" in res["config"]["parallelism"]
    assert res["residency"]["host_store_bytes"] >= 1 * 1 * 2 * 1024 * 64 * 2   # 1 layer x 1 kv head (K+V)


@pytest.mark.gpu
def test_bench_value_independent_of_steps():
    """Every step re-runs the same chunk, so the step time does not depend on --steps (the headline
    drifted with --steps when the timed chunks were the last K ones)."""
    a = run_bench("--workload", "8B-128K", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline")
    b = run_bench("--workload", "8B-128K", "--steps", "6", "--warmup", "3", "--no-e2e", "--no-cpu-baseline")
    assert a["config"]["timed_chunk"] == b["config"]["timed_chunk"]
    assert abs(a["value"] / b["value"] - 1) < 0.05, (a["value"], b["value"])


@pytest.mark.gpu
def test_bench_two_ranks_self_launch():
    """`--gpus 2` without torchrun re-launches itself as 2 ranks (torch.distributed.run); with one GPU the ranks
    share cuda:0 and gather through gloo (--ranks-share-gpu).  Rank 0 prints the one JSON line: n_gpus 2, every
    q head of the gathered output checked against the oracle."""
    res = run_bench("--workload", "tiny", "--steps", "2", "--warmup", "3", "--gpus", "2", "--ranks-share-gpu",
                    timeout=900)
    assert res["n_gpus"] == 2 and res["nccl"]["comm_nranks"] == 2
    assert "head-shard2" in res["config"]["parallelism"]
    ps = res["parity_sample"]
    assert ps["ok"] and ps["qheads_checked"] == 4 and ps["gathered_prefill_rows"] > 0 and ps["gathered_decode_rows"] == 4
    assert res["value"] > 0 and res["e2e"]["value"] > 0


@pytest.mark.gpu
def test_bench_two_ranks_multi_layer():
    """Same launch on a 3-layer workload with 2 kv heads per rank: the gathered prefill AND decode rows of layer 0
    must match the oracle (the decode gather buffer is overwritten by every layer, so the check re-gathers layer 0;
    round 2 found it comparing the last layer's output against layer 0's oracle at 8B-128K)."""
    res = run_bench("--workload", "small", "--steps", "2", "--warmup", "3", "--gpus", "2", "--ranks-share-gpu",
                    timeout=900)
    assert res["n_gpus"] == 2
    ps = res["parity_sample"]
    assert ps["ok"], ps
    assert ps["qheads_checked"] == 16 and ps["gathered_decode_rows"] == 16
    assert ps["decode_rel_l2_max"] <= ps["tol_rel_l2"]
