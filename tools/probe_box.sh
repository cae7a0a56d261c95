#!/bin/bash
# One-off probe of the GPU box: host RAM, NUMA, PCIe, pinned-copy bandwidth.
set -x
nvidia-smi
nvidia-smi topo -m
free -g
lscpu | head -30
numactl -H 2>/dev/null || ls /sys/devices/system/node/
ulimit -l
cat /proc/meminfo | grep -i huge
cat /sys/kernel/mm/transparent_hugepage/enabled
nproc
python - <<'PY'
import torch, time, os
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
bdf = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0),'pci_bus_id') else None
print("bdf", bdf)
for gib in [1, 4]:
    n = gib << 30
    t0=time.time(); h = torch.empty(n, dtype=torch.uint8, pin_memory=True); t1=time.time()
    print(f"pin {gib} GiB: {t1-t0:.2f}s")
    d = torch.empty(n, dtype=torch.uint8, device='cuda')
    s = torch.cuda.Stream()
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); 
        for _ in range(3): fn()
        e1.record(); torch.cuda.synchronize()
        print(f"{name} {gib} GiB: {3*n/e0.elapsed_time(e1)/1e6:.1f} GB/s")
    # bidirectional
    d2 = torch.empty(n, dtype=torch.uint8, device='cuda'); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    print(f"bidir {gib} GiB each: {2*n/e0.elapsed_time(e1)/1e6:.1f} GB/s total")
    del h, d, d2, h2
PY
