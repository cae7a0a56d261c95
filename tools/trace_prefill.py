"""Timeline trace of the prefill kernel (variant build with -DHI_TRACE): one history-block launch,
CTA 0, per-KV-tile clock64() stamps of the softmax (tiles 0/1) and the MMA issuer."""
import ctypes, os, sys
os.environ.setdefault("HI_LIB_VARIANT", "trace")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2502_12574_b200 import _lib
from paper_2502_12574_b200.headinfer import HeadInfer
from synth.cuda import fill_

S, c = 65536, 18944
hi = HeadInfer(1, 32, 8, 128, S + c, c, n_slots=2, slot_tokens=S)
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
assert lib.hi_debug_prefill_trace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes)) == 0
# the LAST launch (head 7's history block, 512 KV tiles) left its stamps
names = {10: "A.wait_done", 0: "A.ld_done", 1: "A.max", 2: "A.exp", 3: "A.st_done", 4: "A.arrived",
         11: "B.wait_done", 5: "B.ld_done", 6: "B.max", 7: "B.exp", 8: "B.st_done", 9: "B.arrived",
         12: "M.pA", 13: "M.issA", 14: "M.pB", 15: "M.issB"}
t0 = int(buf[10, 100])
print("j   " + " ".join(f"{names[k]:>11s}" for k in [10, 0, 1, 2, 3, 4, 12, 13, 11, 5, 6, 7, 8, 9, 14, 15]))
for j in range(100, 112):
    row = [int(buf[k, j]) - t0 for k in [10, 0, 1, 2, 3, 4, 12, 13, 11, 5, 6, 7, 8, 9, 14, 15]]
    print(f"{j:3d} " + " ".join(f"{v:11d}" for v in row))
per = (int(buf[10, 400]) - int(buf[10, 100])) / 300
print(f"period per KV tile (both Q tiles): {per:.0f} cycles; ideal TC time 2048")
