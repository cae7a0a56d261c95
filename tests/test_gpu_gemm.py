"""NEXT-4 projections: the library's tcgen05 GEMM / GEMV (k_gemm.cu, through the C ABI hl_gemm) against the
mathematical definition y = bf16((beta ? y0 : 0) + x w^T) computed in fp64 on the CPU: at most one bf16 ulp
(fp32 accumulation order) and a tiny fraction of elements off by one ulp.  Shapes: ragged token counts (M tails),
out features not a multiple of the 256-wide tile (N tails), K not a multiple of the 64-deep stage, the Llama-3-8B
projection shapes at a 1024-token chunk, and the decode GEMV."""
import pytest
import torch

from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a GPU")]


def _check(n, mo, kd, beta, seed=0):
    from paper_2502_12574_b200.layer import hl_gemm
    g = torch.Generator().manual_seed(seed)
    x = (torch.rand(n, kd, generator=g) * 2 - 1).bfloat16()
    w = ((torch.rand(mo, kd, generator=g) * 2 - 1) / kd ** 0.5).bfloat16()
    y0 = (torch.rand(n, mo, generator=g) * 2 - 1).bfloat16()
    ref = (x.double() @ w.double().T + (y0.double() if beta else 0)).to(torch.bfloat16)
    y = y0.cuda() if beta else torch.full((n, mo), float("nan"), dtype=torch.bfloat16, device="cuda")
    hl_gemm(w.cuda(), x.cuda(), y, beta=beta)
    got = y.cpu()
    assert torch.isfinite(got.float()).all()
    diff = (got.double() - ref.double()).abs()
    ulp = ref.double().abs().clamp_min(2 ** -14) * 2 ** -7   # one bf16 ulp at the reference magnitude (upper bound)
    # fp32 accumulation in another order (the tensor core's adds need not round like IEEE fp32) plus the fp32 add
    # of the residual: |err| <= 2^-20 * (sum_k |x_k w_k| + |y0|), ~16 fp32 ulps of the magnitudes involved
    acc_err = 2.0 ** -20 * (x.double().abs() @ w.double().abs().T + (y0.double().abs() if beta else 0))
    bound = ulp + acc_err
    assert (diff <= bound).all(), float((diff / bound).max())
    assert (diff > 0).double().mean() < 0.05   # almost everything rounds the same way
    return got


@pytest.mark.parametrize("n,mo,kd,beta", [
    (128, 256, 64, False),       # one tile, one stage
    (300, 640, 200, True),       # M, N and K tails, residual
    (2, 64, 8, False),           # the smallest GEMM (tails everywhere)
    (2048, 4096, 64, True),      # 256 tiles on 148 CTAs: the persistent loop and both TMEM accumulators
    (4096, 8192, 128, True),     # ~7 pair tiles per CTA pair: each accumulator buffer drained and re-filled 3+ times
    (1024, 6144, 4096, False),   # Llama-3-8B QKV at a 1024-token chunk
    (1024, 4096, 4096, True),    # O projection + residual
    (517, 4096, 14336, True),    # down projection + residual, ragged chunk
])
def test_gemm_tc(n, mo, kd, beta):
    _check(n, mo, kd, beta)


@pytest.mark.parametrize("mo,kd,beta", [(6144, 4096, False), (4096, 14336, True), (64, 8, True), (28672, 4096, False)])
def test_gemv_decode(mo, kd, beta):
    _check(1, mo, kd, beta)


def test_gemm_rejects_bad_sizes():
    from paper_2502_12574_b200 import _lib
    lib = _lib.load()
    assert lib.hl_gemm(1, 1, 1, 100, 4, 64, 0, None) == _lib.HI_EINVAL   # mo % 64
    assert lib.hl_gemm(None, 1, 1, 128, 4, 64, 0, None) == _lib.HI_EINVAL
