"""C-ABI contract checks that need no GPU: the library loads, exports every symbol
include/headinfer.h declares, and fails loudly (HI_ECUDA, no CPU fallback) without a device."""
import ctypes
import os
import re

import pytest

from conftest import cuda_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    syms = set()
    for hdr in ("headinfer.h", "hilayer.h"):
        src = open(os.path.join(ROOT, "include", hdr)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        syms |= set(re.findall(r"\b(h[il]_[a-z_]+)\s*\(", src))
    return sorted(syms)


@pytest.fixture(scope="module")
def lib():
    from paper_2502_12574_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2502_12574_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_the_north_star_calls():
    syms = _declared_symbols()
    for name in ("hi_init", "hi_prefill_chunk", "hi_decode", "hi_free"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2502_12574_b200 import _lib
    syms = _declared_symbols()
    assert sorted(_lib.EXPORTS) == syms
    for name in syms:
        assert hasattr(lib, name), name


def test_status_strings(lib):
    names = [lib.hi_status_str(i).decode() for i in range(8)]
    assert names == ["HI_OK", "HI_EINVAL", "HI_ESHAPE", "HI_ECAPACITY", "HI_ENOMEM_HOST", "HI_ENOMEM_DEV",
                     "HI_ECUDA", "HI_ESTATE"]


def test_free_null_and_bad_handles(lib):
    assert lib.hi_free(None) == 0
    assert lib.hi_seq_len(None, 0) == -1
    assert lib.hi_prefill_chunk(None, 0, None, None, None, None, 1, None) == 2  # HI_ESHAPE
    assert lib.hi_last_error(None)


@pytest.mark.parametrize("args", [
    (0, 4, 2, 64, 1024, 256, 0, 1),     # layers <= 0
    (1, 5, 2, 64, 1024, 256, 0, 1),     # q_heads % kv_heads
    (1, 4, 2, 96, 1024, 256, 0, 1),     # head_dim not in {64, 128}
    (1, 8, 2, 64, 1024, 256, 0, 4),     # kv_heads % world
    (1, 4, 2, 64, 0, 256, 0, 1),        # max_ctx <= 0
    (1, 4, 2, 64, 1024, 256, 1, 1),     # rank >= world
    (1, 64, 2, 64, 1024, 256, 0, 1),    # g = 32 unsupported
])
def test_init_rejects_invalid_configuration(lib, args):
    h = ctypes.c_void_p()
    assert lib.hi_init(*args, ctypes.byref(h)) == 1  # HI_EINVAL, before touching CUDA
    assert not h.value


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_init_without_gpu_fails_loudly(lib):
    h = ctypes.c_void_p()
    assert lib.hi_init(1, 4, 2, 64, 1024, 256, 0, 1, ctypes.byref(h)) == 6  # HI_ECUDA, no CPU fallback
    assert not h.value
    assert b"CUDA" in lib.hi_last_error(None) or b"device" in lib.hi_last_error(None)


@pytest.mark.parametrize("opts", [dict(head_group=3), dict(head_group=-3), dict(n_slots=1),
                                  dict(resident_kv_heads=-2)])
def test_init_rejects_invalid_options(lib, opts):
    """hi_init_ex validates hi_options before touching CUDA (head_group must divide kv_heads/world)."""
    from paper_2502_12574_b200._lib import hi_options
    h = ctypes.c_void_p()
    o = hi_options(**opts)
    assert lib.hi_init_ex(1, 8, 4, 64, 1024, 256, 0, 1, ctypes.byref(o), ctypes.byref(h)) == 1
    assert not h.value
    assert b"hi_options" in lib.hi_last_error(None)


@pytest.mark.parametrize("flags", [0x10, 0x20, 0x40, 0x1000])
def test_product_build_rejects_comparison_kernel_flags(lib, flags):
    """The comparison prefill kernels (mma.sync, CTA pair, one tile) live only in the variants build; the
    product library refuses their flags before touching CUDA."""
    from paper_2502_12574_b200._lib import hi_options
    h = ctypes.c_void_p()
    o = hi_options(flags=flags)
    assert lib.hi_init_ex(1, 8, 4, 64, 1024, 256, 0, 1, ctypes.byref(o), ctypes.byref(h)) == 1
    assert not h.value
    assert b"variants" in lib.hi_last_error(None)


@pytest.mark.parametrize("opts", [dict(duo_window=-5), dict(duo_window=1 << 21)])
def test_init_rejects_invalid_duo_options(lib, opts):
    """NEXT-3: streaming heads need a window >= 1 and the default (band-masking) prefill kernel."""
    from paper_2502_12574_b200._lib import hi_options
    lab = (ctypes.c_ubyte * 4)(1, 0, 0, 1)
    h = ctypes.c_void_p()
    o = hi_options(streaming_heads=ctypes.cast(lab, ctypes.c_void_p), **opts)
    assert lib.hi_init_ex(1, 8, 4, 64, 1024, 256, 0, 1, ctypes.byref(o), ctypes.byref(h)) == 1
    assert not h.value
    assert b"streaming" in lib.hi_last_error(None)


def test_init_rejects_too_many_local_kv_heads(lib):
    h = ctypes.c_void_p()
    assert lib.hi_init(1, 128, 128, 64, 1024, 256, 0, 1, ctypes.byref(h)) == 1  # > 64 kv heads per launch map
    assert b"64" in lib.hi_last_error(None)


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's hi_options / hi_stats mirror the C layout (size and every field offset), compiled
    from include/headinfer.h with the host C compiler."""
    import subprocess
    from paper_2502_12574_b200._lib import hi_options, hi_stats, hl_weights
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "headinfer.h"', 'int main(void) {']
    lines[2] = '#include "hilayer.h"'
    for st in (hi_options, hi_stats, hl_weights):
        lines.append(f'printf("{st.__name__} %zu\\n", sizeof({st.__name__}));')
        for name, _ in st._fields_:
            lines.append(f'printf("{st.__name__}.{name} %zu\\n", offsetof({st.__name__}, {name}));')
    lines += ["return 0; }"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines())
    for st in (hi_options, hi_stats, hl_weights):
        assert int(got[st.__name__]) == ctypes.sizeof(st), st.__name__
        for name, _ in st._fields_:
            assert int(got[f"{st.__name__}.{name}"]) == getattr(st, name).offset, (st.__name__, name)
