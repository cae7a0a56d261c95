"""Sticky CUDA failure (SURVEY.md §8(b) "Errors": a CUDA error makes the ctx sticky-failed -- every later call
returns HI_ECUDA until hi_free; SPEC.md negative-control idea).  The errors are real CUDA errors,
injected through test-only flags: HI_FLAG_FAULT_LAUNCH (an invalid launch configuration, synchronous, the
CUDA context survives) in process, HI_FLAG_FAULT_TRAP (a device-side `trap`, asynchronous, the process's
CUDA context is lost) in a subprocess."""
import ctypes
import os
import subprocess
import sys

import pytest
import torch

from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# shared by the in-process test and the subprocess script: every ABI call on a failed context returns HI_ECUDA
PROBE = r'''
import ctypes, torch
from paper_2502_12574_b200 import _lib
from paper_2502_12574_b200.headinfer import hi_init
lib = _lib.load()

def calls_after_failure(h, ptr, n=64, d=64):
    """ptr: a device buffer allocated BEFORE the failure (nothing may touch CUDA after a device fault)."""
    st = {}
    args = [ptr] * 4
    st["prefill"] = lib.hi_prefill_chunk(h, 0, *args, n, None)
    st["decode"] = lib.hi_decode(h, 0, *args, None)
    st["synchronize"] = lib.hi_synchronize(h)
    buf = (ctypes.c_uint16 * (n * d))()
    st["read_host_kv"] = lib.hi_read_host_kv(h, 0, 0, 0, 1, buf, buf)
    st["write_host_kv"] = lib.hi_write_host_kv(h, 0, 0, 0, 1, buf, buf, 0)
    st["set_seq_len"] = lib.hi_set_seq_len(h, 0, 0)
    s = _lib.hi_stats()
    st["get_stats"] = lib.hi_get_stats(h, ctypes.byref(s))
    return st
'''


def _ctx(flags):
    from paper_2502_12574_b200.headinfer import hi_init
    return hi_init(1, 4, 2, 64, 4096, 256, flags=flags)


def _inputs(n=64):
    Q = torch.randn((n, 4, 64), device="cuda").bfloat16()
    K = torch.randn((n, 2, 64), device="cuda").bfloat16()
    return Q, K, K.clone(), torch.empty_like(Q)


def test_sticky_after_launch_error():
    from paper_2502_12574_b200 import _lib
    from paper_2502_12574_b200._lib import HI_ECUDA, HI_FLAG_FAULT_LAUNCH, HI_OK
    lib = _lib.load()
    ns = {}
    exec(PROBE, ns)
    h = _ctx(HI_FLAG_FAULT_LAUNCH)
    Q, K, V, out = _inputs()
    cs = torch.cuda.current_stream().cuda_stream
    assert lib.hi_prefill_chunk(h, 0, Q.data_ptr(), K.data_ptr(), V.data_ptr(), out.data_ptr(), 64, cs) == HI_OK
    assert lib.hi_prefill_chunk(h, 0, Q.data_ptr(), K.data_ptr(), V.data_ptr(), out.data_ptr(), 64, cs) == HI_ECUDA
    assert b"cudaErrorInvalidConfiguration" in lib.hi_last_error(h)
    st = ns["calls_after_failure"](h, Q.data_ptr())
    assert all(v == HI_ECUDA for v in st.values()), st
    assert lib.hi_seq_len(h, 0) == 64          # the failed call did not advance the cursor
    assert lib.hi_free(h) == HI_OK
    # the failure is per context: the CUDA context survived, a fresh context works
    h2 = _ctx(0)
    for _ in range(3):
        assert lib.hi_prefill_chunk(h2, 0, Q.data_ptr(), K.data_ptr(), V.data_ptr(), out.data_ptr(), 64, cs) == HI_OK
    assert lib.hi_synchronize(h2) == HI_OK
    assert torch.isfinite(out.float()).all()
    assert lib.hi_free(h2) == HI_OK


def test_sticky_after_device_trap_subprocess():
    script = PROBE + r'''
from paper_2502_12574_b200._lib import HI_ECUDA, HI_OK, HI_FLAG_FAULT_TRAP
torch.cuda.init()
h = hi_init(1, 4, 2, 64, 4096, 256, flags=HI_FLAG_FAULT_TRAP)
Q = torch.randn((64, 4, 64), device="cuda").bfloat16(); K = torch.randn((64, 2, 64), device="cuda").bfloat16()
out = torch.empty_like(Q)
cs = torch.cuda.current_stream().cuda_stream
assert lib.hi_prefill_chunk(h, 0, Q.data_ptr(), K.data_ptr(), K.data_ptr(), out.data_ptr(), 64, cs) == HI_OK
r = lib.hi_prefill_chunk(h, 0, Q.data_ptr(), K.data_ptr(), K.data_ptr(), out.data_ptr(), 64, cs)  # enqueues the trap
assert r in (HI_OK, HI_ECUDA), r
assert lib.hi_synchronize(h) == HI_ECUDA       # the asynchronous fault surfaces here at the latest
msg = lib.hi_last_error(h)
assert b"cudaError" in msg, msg
st = calls_after_failure(h, Q.data_ptr())
assert all(v == HI_ECUDA for v in st.values()), st
assert lib.hi_free(h) == HI_OK
print("STICKY_OK", msg.decode())
'''
    r = subprocess.run([sys.executable, "-c", script], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    assert r.returncode == 0 and "STICKY_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
