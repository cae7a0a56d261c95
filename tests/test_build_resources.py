"""Build-time resource checks of the product kernels (no GPU needed): the sm_100a cubins in
libheadinfer.so must keep their hot loops in registers -- no stack frame / local memory for the
product prefill and decode kernels (a runtime-indexed register array silently turns into local memory
and costs ~7x; seen once during development), and every kernel is compiled for sm_100a."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2502_12574_b200", "libheadinfer.so")
PRODUCT = ("prefill_tc_kernel", "decode_partial_kernel", "decode_combine_kernel", "pack_kv_kernel", "gemm_tc2_kernel",
           "gemv_kernel")


def _res_usage():
    if not os.path.exists(LIB):
        from paper_2502_12574_b200 import build
        build.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-res-usage", LIB], capture_output=True, text=True).stdout
    res = {}
    fn = None
    for line in out.splitlines():
        m = re.search(r"Function ([^:\s]+)", line)
        if m:
            fn = m.group(1)
            continue
        if fn and "REG:" in line:
            res[fn] = {k: int(v) for k, v in re.findall(r"(REG|STACK|LOCAL|SHARED):(\d+)", line)}
            fn = None
    return res, out


def test_product_kernels_have_no_local_memory():
    res, _ = _res_usage()
    seen = set()
    for fn, r in res.items():
        for name in PRODUCT:
            if name in fn:
                seen.add(name)
                assert r.get("STACK", 0) == 0 and r.get("LOCAL", 0) == 0, (fn, r)
    assert seen == set(PRODUCT), seen


def test_cubins_are_sm_100a():
    _, out = _res_usage()
    archs = set(re.findall(r"arch = (sm_\w+)", out))
    assert archs == {"sm_100a"}, archs
