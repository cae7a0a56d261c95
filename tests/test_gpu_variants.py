"""GPU parity of the COMPARISON prefill kernels (csrc/variants/: CTA pair, one tile, mma.sync baseline)
against the fp64 oracle.  They are not in the product library: these tests build the variants library
(build.build_variant("cmp", [])) and run in a subprocess with HI_LIB_VARIANT=cmp.  Opt-in: HI_TEST_VARIANTS=1
(the build takes minutes), so the default `-m gpu` tier covers the product path only."""
import os
import subprocess
import sys

import pytest
import torch

from conftest import cuda_available
from hi_harness import Run, check_host_kv, compare, run_gpu, run_oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IN_VARIANT = os.environ.get("HI_LIB_VARIANT") == "cmp"
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU"),
              pytest.mark.skipif(not os.environ.get("HI_TEST_VARIANTS"), reason="opt-in: HI_TEST_VARIANTS=1")]


@pytest.mark.skipif(IN_VARIANT, reason="runs the variant tests in a subprocess")
def test_variants_in_subprocess():
    sys.path.insert(0, ROOT)
    from paper_2502_12574_b200 import build
    build.build_variant("cmp", [])
    env = dict(os.environ, HI_LIB_VARIANT="cmp")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", __file__, "-k", "not subprocess"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=3600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]


need_variant = pytest.mark.skipif(not IN_VARIANT, reason="needs HI_LIB_VARIANT=cmp")


@need_variant
@pytest.mark.parametrize("g", [1, 4, 8])
def test_cta_pair_kernel(g):
    """The CTA-pair (cta_group::2, M = 256) prefill kernel behind HI_FLAG_PREFILL_2CTA (head_dim 128)."""
    r = Run(layers=2, q_heads=2 * g, kv_heads=2, d=128, chunks=[300, 300, 555], n_decode=2, dist="P",
            opts=dict(slot_tokens=256, flags=0x20))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()


@need_variant
@pytest.mark.parametrize("group,flags", [(4, 0x10), (2, 0x20)])
def test_head_groups_with_single_head_kernels(group, flags):
    r = Run(layers=2, q_heads=16, kv_heads=8, d=128, chunks=[300, 300, 100], n_decode=4, dist="P",
            opts=dict(slot_tokens=128, head_group=group, flags=flags))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()


@need_variant
@pytest.mark.parametrize("g,d", [(1, 64), (4, 64), (2, 128), (4, 128), (8, 128)])
def test_one_tile_kernel(g, d):
    """The one-tile / three-S-buffer prefill kernel behind HI_FLAG_PREFILL_TC1 (k_prefill_tc1.cu): causal
    chunks, ragged tails, many history blocks, K/V multicast across CTA pairs (odd tile counts leave a
    padding CTA)."""
    r = Run(layers=2, q_heads=2 * g, kv_heads=2, d=d, chunks=[300, 300, 555, 77], n_decode=2, dist="P",
            opts=dict(slot_tokens=256, flags=0x40))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()


@need_variant
@pytest.mark.parametrize("dist", ["S", "ONE"])
def test_one_tile_kernel_special(dist):
    """Sink-dominated scores (lazy rescale paths) and V == 1 (exact normalisation) on the one-tile kernel,
    with head groups and resident heads."""
    r = Run(layers=2, q_heads=16, kv_heads=4, d=128, chunks=[256, 512, 100], n_decode=2, dist=dist,
            opts=dict(slot_tokens=192, flags=0x40, head_group=2, resident_kv_heads=1))
    gpu, ctx = run_gpu(r)
    if dist == "ONE":
        assert torch.all(gpu[0] == 1.0)
    ref, _ = run_oracle(r)
    compare(gpu, ref)
    ctx.close()


@need_variant
@pytest.mark.parametrize("dist", ["P", "S"])
@pytest.mark.parametrize("g,d", [(1, 64), (4, 128), (8, 128)])
def test_psmem_kernel(dist, g, d):
    """The P-in-shared-memory prefill kernel behind HI_FLAG_PREFILL_PSMEM (variants/k_prefill_tcp.cu): ragged
    causal chunks, many history blocks, head groups."""
    r = Run(layers=2, q_heads=4 * g, kv_heads=4, d=d, chunks=[300, 300, 555, 77], n_decode=2, dist=dist,
            opts=dict(slot_tokens=256, flags=0x1000, head_group=2))
    gpu, ctx = run_gpu(r)
    ref, inputs = run_oracle(r)
    compare(gpu, ref)
    check_host_kv(ctx, r, inputs)
    ctx.close()
