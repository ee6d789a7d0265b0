"""PARITY projection GEMM on the int8 tensor cores (gemm_oz.cu, Ozaki scheme II)
against the reference's arithmetic: fp32 operands, fp64 accumulation, one
rounding to fp32 (vec_mat, tensor.hpp:31-41).

The exact product (fp64 here, computed by torch on the GPU in float64) is the
oracle; the DFMA kernel (gemm_f64acc.cu, bit-exact with vec_mat) is the
baseline.  The Ozaki result must stay within its stated error bound of the
exact value, and its fp32 outputs must equal the DFMA kernel's except for a
tiny fraction of 1-ulp rounding-boundary cases.
"""
import math
import os

import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu


MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def oz_bits(K):
    """gemm_oz.cu oz_bits: integer bits per operand with K 2^2b <= M / 4."""
    n = int(os.environ.get("KEEP_OZ_MODULI", "14"))
    lm = sum(math.log2(m) for m in MODULI[:n])
    return int(math.floor((lm - 2.0 - math.log2(K)) / 2.0))


def run(A, B, mode):
    import torch
    M, K = A.shape
    N = B.shape[1]
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    lib = kb.load_library()
    rc = lib.keep_debug_gemm_parity(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, mode)
    assert rc == 0, lib.keep_last_error()
    return C


@pytest.mark.parametrize("M,N,K", [
    (128, 256, 128), (300, 512, 512), (64, 96, 64), (1000, 15360, 5120), (777, 5120, 13824),
    (2049, 1024, 1024), (130, 288, 4096), (256, 5120, 27648),
])
def test_ozaki_matches_fp64_accumulation(M, N, K):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 31 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g, dtype=torch.float32)
    A[:, ::7] *= 1e-3  # a wide dynamic range inside rows
    A = torch.relu(A) if K % 2 else A
    B = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float32) / np.sqrt(K)
    oz = run(A, B, 1)
    df = run(A, B, 2)
    exact = A.double() @ B.double()
    assert not torch.isnan(oz).any()
    # error bound: each operand rounded to b integer bits of its row / column
    # maximum (|error| <= 2^-b max), the CRT reconstruction exact, the fp64
    # Horner within a few ulp, plus the final fp32 rounding
    b = oz_bits(K)
    amax = A.abs().amax(dim=1, keepdim=True).double()
    bmax = B.abs().amax(dim=0, keepdim=True).double()
    bound = K * 2.0 ** (1 - b) * amax * bmax + exact.abs() * 2.0 ** -24
    assert bool(((oz.double() - exact).abs() <= bound).all())
    # fp32 outputs equal the DFMA (vec_mat) ones except rounding-boundary ties
    diff = (oz != df).double().mean().item()
    assert diff <= 1e-4, diff
    ulps = ((oz - df).abs() / torch.clamp(df.abs(), min=1e-30)).max().item()
    assert ulps <= 2.0 ** -22, ulps


def test_ozaki_zero_rows_and_tiny_values():
    import torch
    M, N, K = 256, 512, 256
    A = torch.zeros(M, K, device="cuda")
    A[1] = 1e-30
    A[2, 5] = 3.0e30
    A[3] = torch.arange(K, device="cuda", dtype=torch.float32) - 100
    B = torch.randn(K, N, device="cuda")
    oz = run(A, B, 1)
    exact = (A.double() @ B.double()).float()
    assert torch.equal(oz[0], torch.zeros_like(oz[0]))
    assert torch.allclose(oz, exact, rtol=1e-6, atol=0)


@pytest.mark.parametrize("M,N,K", [(1, 96, 64), (8, 512, 260), (9, 512, 1024), (17, 160, 5120), (32, 2048, 996),
                                   (8, 5120, 5120)])
def test_dfma_skinny_is_vec_mat(M, N, K):
    """Few rows (the deep layers): the DFMA weight-stream kernel keeps vec_mat's
    exact arithmetic -- fp64 accumulation in ascending k, one rounding."""
    import torch
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32)
    acc = np.zeros((M, N), np.float64)
    for k in range(K):  # tensor.hpp:36-39, k ascending
        acc += A[:, k:k + 1].astype(np.float64) * B[k].astype(np.float64)
    got = run(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), 2).cpu().numpy()
    assert np.array_equal(got, acc.astype(np.float32))


@pytest.mark.parametrize("K", [64, 5120, 13824])
def test_ozaki_crt_range_extremes(K):
    """The largest product sums the CRT range must hold: every operand at its
    row / column maximum with one sign (|X| = K 2^2b), and alternating signs."""
    import torch
    M, N = 128, 256
    A = torch.ones(M, K, device="cuda")
    A[1::2] = -1.0
    A[2] = 0.75
    B = torch.ones(K, N, device="cuda")
    B[:, 1::3] = -0.5
    oz = run(A, B, 1)
    exact = (A.double() @ B.double()).float()
    assert torch.equal(oz, exact)
