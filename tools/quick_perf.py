"""Quick timing probe (not the bench): 8B shape, one prefill chunk + one decode step."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_12574_b200.headinfer import HeadInfer
from synth.cuda import fill_

ctxlen = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
c = int(sys.argv[3]) if len(sys.argv) > 3 else 18944
t0 = time.time()
from paper_2502_12574_b200._lib import HI_FLAG_TIMING
hi = HeadInfer(L, 32, 8, 128, ctxlen + 128, c, flags=HI_FLAG_TIMING | int(os.environ.get("HI_QP_FLAGS", "0"), 0),
               head_group=int(os.environ.get("HI_QP_GROUP", "1")))
print(f"init {time.time()-t0:.1f}s stats={hi.stats()}", flush=True)
t0 = time.time()
buf_k = torch.empty((c, 1, 128), dtype=torch.bfloat16, device="cuda"); buf_v = torch.empty_like(buf_k)
for l in range(L):
    for h in range(8):
        for p0 in range(0, ctxlen, c):
            n = min(c, ctxlen - p0)
            fill_(buf_k[:n], 1, 1, "U", l, h, p0); fill_(buf_v[:n], 1, 2, "U", l, h, p0)
            hi.write_host_kv(l, h, p0, buf_k[:n, 0], buf_v[:n, 0])
print(f"fill {time.time()-t0:.1f}s", flush=True)
s = ctxlen - c
Q = fill_(torch.empty((c, 32, 128), dtype=torch.bfloat16, device="cuda"), 1, 0, "U", 0, 0, s)
K = fill_(torch.empty((c, 8, 128), dtype=torch.bfloat16, device="cuda"), 1, 1, "U", 0, 0, s)
V = fill_(torch.empty((c, 8, 128), dtype=torch.bfloat16, device="cuda"), 1, 2, "U", 0, 0, s)
out = torch.empty_like(Q)
for it in range(3):
    for l in range(L): hi.set_seq_len(l, s)
    torch.cuda.synchronize()
    st0 = hi.stats()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for l in range(L): hi.prefill_chunk(l, Q, K, V, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st1 = hi.stats()
    fl = L * 4 * 128 * 32 * (s * c + c * (c + 1) / 2)
    kms = st1["prefill_attn_ms"] - st0["prefill_attn_ms"]
    kfl = st1["prefill_attn_flops"] - st0["prefill_attn_flops"]
    print(f"prefill chunk s={s} L={L}: {ms:.1f} ms  {fl/ms/1e9:.1f} TFLOP/s  kernel {kms:.1f} ms {kfl/max(kms,1e-9)/1e9:.1f} TFLOP/s", flush=True)
q = Q[0].contiguous(); k = K[0].contiguous(); v = V[0].contiguous(); o = torch.empty_like(q)
for it in range(3):
    for l in range(L): hi.set_seq_len(l, ctxlen - 1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for l in range(L): hi.decode(l, q, k, v, o)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    by = L * 8 * (ctxlen - 1) * 512
    print(f"decode s={ctxlen-1} L={L}: {ms:.1f} ms  H2D {by/ms/1e6:.1f} GB/s", flush=True)
print(hi.stats())
