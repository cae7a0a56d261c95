"""Decode-only probe: L layers of an 8B-shape context at s tokens, all pairs resident (NEXT-1) or
offloaded; times decode steps (for ncu captures of the decode kernels)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_12574_b200.headinfer import HeadInfer
from synth.cuda import fill_

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
R = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = HeadInfer(L, 32, 8, 128, S + 16, 18944, resident_kv_heads=R)
piece = 65536
bk = torch.empty((piece, 1, 128), dtype=torch.bfloat16, device="cuda"); bv = torch.empty_like(bk)
for l in range(L):
    for h in range(8):
        for p0 in range(0, S, piece):
            n = min(piece, S - p0)
            fill_(bk[:n], 1, 1, "U", l, h, p0); fill_(bv[:n], 1, 2, "U", l, h, p0)
            hi.write_host_kv(l, h, p0, bk[:n, 0], bv[:n, 0])
for l in range(L):
    hi.set_seq_len(l, S)
q = fill_(torch.empty((1, 32, 128), dtype=torch.bfloat16, device="cuda"), 1, 0, "U", 0, 0, S)[0]
k = fill_(torch.empty((1, 8, 128), dtype=torch.bfloat16, device="cuda"), 1, 1, "U", 0, 0, S)[0]
v = fill_(torch.empty((1, 8, 128), dtype=torch.bfloat16, device="cuda"), 1, 2, "U", 0, 0, S)[0]
o = torch.empty_like(q)
for it in range(4):
    for l in range(L):
        hi.set_seq_len(l, S)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for l in range(L):
        hi.decode(l, q, k, v, o)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"decode s={S} L={L} R={R}: {ms:.2f} ms  KV {L*8*S*512/ms/1e6:.1f} GB/s", flush=True)
