"""Host-side logic of the multi-GPU launch (CPU): sysfs cpulist parsing for the per-rank NUMA/CPU binding, and
bench.py's --gpus N self-launch command line and workload sizing."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parse_cpulist():
    from paper_2502_12574_b200.hostlink import parse_cpulist
    assert parse_cpulist("0-3,8,10-11") == [0, 1, 2, 3, 8, 10, 11]
    assert parse_cpulist("5") == [5]
    assert parse_cpulist("") == []
    assert parse_cpulist("0-15\n".strip()) == list(range(16))


def test_bind_process_keeps_affinity_without_sysfs(monkeypatch):
    from paper_2502_12574_b200 import hostlink
    monkeypatch.setattr(hostlink, "gpu_locality", lambda dev: {"pci": None, "numa_node": -1, "local_cpus": []})
    before = sorted(os.sched_getaffinity(0))
    loc = hostlink.bind_process_to_gpu(0)
    assert loc["affinity"] == before == sorted(os.sched_getaffinity(0))


def test_bench_host_store_sizing_and_workload_choice(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    # 8B-1M: 32 layers x 8 kv heads x 4*128 B per token x (2^20 + 16) tokens = 128 GiB for the whole job
    assert bench.host_store_bytes("8B-1M", 8) == 32 * 8 * 512 * ((1 << 20) + 16)
    monkeypatch.setattr(bench, "mem_available_bytes", lambda: 1 << 40)
    assert bench.pick_workload("auto", 8) == "8B-1M"
    monkeypatch.setattr(bench, "mem_available_bytes", lambda: 100 << 30)
    assert bench.pick_workload("auto", 1) == "8B-128K"
    assert bench.pick_workload("tiny", 1) == "tiny"


def test_bench_relaunch_command(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, cwd=None: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--ranks-share-gpu", "--steps", "2"])

    class A:
        gpus, ranks_share_gpu = 4, True
    bench.relaunch_under_torchrun(A())
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-5:] == ["--gpus", "4", "--ranks-share-gpu", "--steps", "2"]
