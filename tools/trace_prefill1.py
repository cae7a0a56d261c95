"""Timeline trace of the one-tile prefill kernel (k_prefill_tc1.cu, variant build with -DHI_TRACE):
one history-block launch, CTA (0,0), per-KV-tile clock64() stamps of the softmax warps 0 (key half 0)
and 4 (key half 1) and of the MMA issuer."""
import ctypes, os, sys
os.environ.setdefault("HI_LIB_VARIANT", "trace")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_12574_b200 import _lib
from paper_2502_12574_b200.headinfer import HeadInfer
from synth.cuda import fill_

S, c = 65536, 18944
hi = HeadInfer(1, 32, 8, 128, S + c, c, n_slots=2, slot_tokens=S, flags=0x40)
for h in range(8):
    bk = torch.empty((S, 1, 128), dtype=torch.bfloat16, device="cuda"); bv = torch.empty_like(bk)
    fill_(bk, 1, 1, "U", 0, h, 0); fill_(bv, 1, 2, "U", 0, h, 0)
    hi.write_host_kv(0, h, 0, bk[:, 0], bv[:, 0])
hi.set_seq_len(0, S)
Q = fill_(torch.empty((c, 32, 128), dtype=torch.bfloat16, device="cuda"), 1, 0, "U", 0, 0, S)
K = fill_(torch.empty((c, 8, 128), dtype=torch.bfloat16, device="cuda"), 1, 1, "U", 0, 0, S)
V = fill_(torch.empty((c, 8, 128), dtype=torch.bfloat16, device="cuda"), 1, 2, "U", 0, 0, S)
hi.prefill_chunk(0, Q, K, V)
torch.cuda.synchronize()
lib = _lib.load()
buf = np.zeros((16, 512), dtype=np.uint64)
assert lib.hi_debug_prefill_trace1(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes)) == 0
names = {0: "h0.s_rdy", 1: "h0.max", 2: "h0.exp", 3: "h0.pvwait", 4: "P.Kissue",
         5: "h1.s_rdy", 6: "h1.max", 7: "h1.exp", 8: "h1.pvwait", 9: "h1.arrive",
         10: "M.p_seen", 11: "M.v_seen", 12: "M.pv_iss", 13: "M.it_end", 14: "M.k(j)rdy", 15: "M.S(j)iss"}
order = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15]
t0 = int(buf[0, 100])
print("j   " + " ".join(f"{names[k]:>10s}" for k in order))
for j in range(100, 112):
    print(f"{j:3d} " + " ".join(f"{int(buf[k, j]) - t0:10d}" for k in order))
per = (int(buf[0, 400]) - int(buf[0, 100])) / 300
print(f"period per KV tile (one 128-row Q tile): {per:.0f} cycles; ideal TC time 1024")
