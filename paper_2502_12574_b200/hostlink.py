"""Host-link placement and measurement (SURVEY.md §5 "host-link measurement alone and with all GPUs
concurrent"; §8(e) scaling caveat: the decode roofline per GPU is the CONCURRENT per-GPU H2D bandwidth).

Not on the hot path: the library streams K/V with its own copy engine (hi_runtime.cu); this module only
  * finds a GPU's PCI address, NUMA node and local CPUs (sysfs), and pins the calling process to them, so
    pinned buffers it first-touches and the host thread that enqueues work sit next to the GPU (the host KV
    store itself is mbind-ed by hi_init, numa_policy 0);
  * times pinned H2D / D2H / both-directions copies with CUDA events, optionally in lock-step with other
    ranks (a barrier callback), which is how bench.py and tools/probe_link.py measure the per-GPU link
    bandwidth under the same W-concurrency as the run.
"""
from __future__ import annotations

import os

import torch


def pci_bus_id(device: int) -> str | None:
    """'0000:40:00.0'-style PCI address of a CUDA device (lower case), or None."""
    props = torch.cuda.get_device_properties(device)
    dom = getattr(props, "pci_domain_id", None)
    bus = getattr(props, "pci_bus_id", None)
    dev = getattr(props, "pci_device_id", None)
    if bus is not None and dev is not None:
        return f"{dom or 0:04x}:{bus:02x}:{dev:02x}.0"
    try:
        import pynvml  # nvidia_ml_py; CUDA and NVML orders agree under CUDA_DEVICE_ORDER=PCI_BUS_ID only
        pynvml.nvmlInit()
        uuid = str(getattr(props, "uuid", ""))
        for i in range(pynvml.nvmlDeviceGetCount()):
            h = pynvml.nvmlDeviceGetHandleByIndex(i)
            u = pynvml.nvmlDeviceGetUUID(h)
            u = u.decode() if isinstance(u, bytes) else u
            if uuid and uuid in u:
                b = pynvml.nvmlDeviceGetPciInfo(h).busId
                b = b.decode() if isinstance(b, bytes) else b
                return b.lower()[-12:]
    except Exception:  # noqa: BLE001
        pass
    return None


def _sysfs(bdf: str | None, leaf: str) -> str | None:
    if not bdf:
        return None
    try:
        with open(f"/sys/bus/pci/devices/{bdf}/{leaf}") as f:
            return f.read().strip()
    except OSError:
        return None


def parse_cpulist(s: str) -> list[int]:
    out: list[int] = []
    for part in s.split(","):
        part = part.strip()
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_locality(device: int) -> dict:
    """{'pci': bdf, 'numa_node': n (-1 unknown), 'local_cpus': [...]} from sysfs."""
    bdf = pci_bus_id(device)
    node = _sysfs(bdf, "numa_node")
    cpus = _sysfs(bdf, "local_cpulist")
    return {"pci": bdf, "numa_node": int(node) if node not in (None, "") else -1,
            "local_cpus": parse_cpulist(cpus) if cpus else []}


def bind_process_to_gpu(device: int) -> dict:
    """Restrict this process to the GPU's local CPUs (when sysfs knows them and they intersect the current
    affinity).  Returns gpu_locality() plus the affinity actually set."""
    loc = gpu_locality(device)
    cur = sorted(os.sched_getaffinity(0))
    want = sorted(set(loc["local_cpus"]) & set(cur))
    if want and want != cur:
        try:
            os.sched_setaffinity(0, want)
        except OSError:
            want = cur
    loc["affinity"] = sorted(os.sched_getaffinity(0))
    return loc


def measure_link(device: int, gib: float = 1.0, reps: int = 3, barrier=None) -> dict:
    """Pinned-host <-> device copy bandwidth of `device` in GB/s (1e9 B/s): H2D alone, D2H alone, and both
    directions at once (two streams).  `barrier()` (if given) is called before each phase so that several
    ranks copy at the same time (the concurrent figure).  Best of `reps` timed copies of `gib` GiB each."""
    n = int(gib * (1 << 30))
    with torch.cuda.device(device):
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h.fill_(1)
        h2.fill_(2)
        d = torch.empty(n, dtype=torch.uint8, device=device)
        d2 = torch.empty(n, dtype=torch.uint8, device=device)
        s1, s2 = torch.cuda.Stream(device), torch.cuda.Stream(device)

        def timed(fn_list):
            best = float("inf")
            for _ in range(reps + 1):      # first round is a warm-up
                torch.cuda.synchronize(device)
                if barrier:
                    barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                cur = torch.cuda.current_stream(device)
                e0.record(cur)
                for st, fn in fn_list:
                    st.wait_stream(cur)
                    with torch.cuda.stream(st):
                        fn()
                for st, _ in fn_list:
                    cur.wait_stream(st)
                e1.record(cur)
                torch.cuda.synchronize(device)
                best = min(best, e0.elapsed_time(e1))
            return best

        t_h2d = timed([(s1, lambda: d.copy_(h, non_blocking=True))])
        t_d2h = timed([(s1, lambda: h.copy_(d, non_blocking=True))])
        t_bi = timed([(s1, lambda: d.copy_(h, non_blocking=True)), (s2, lambda: h2.copy_(d2, non_blocking=True))])
        del h, h2, d, d2
    return {"h2d_gbs": round(n / t_h2d / 1e6, 2), "d2h_gbs": round(n / t_d2h / 1e6, 2),
            "bidir_gbs": round(2 * n / t_bi / 1e6, 2), "bytes": n, "reps": reps}
