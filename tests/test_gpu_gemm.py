"""tcgen05 GEMM (FAST projections) against a torch fp32 reference of the same op."""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K,bn", [
    (128, 256, 64, 256), (128, 64, 64, 64), (1, 64, 64, 64), (300, 512, 512, 256), (300, 512, 512, 64),
    (16, 5120, 5120, 0), (1000, 15360, 5120, 0), (17, 13824, 5120, 0), (4100, 5120, 13824, 0),
    (2049, 1024, 1024, 256),
    # small-M path (deep layers): 32-row A stages, 32-wide N tiles
    (8, 5120, 5120, 32), (1, 32, 64, 32), (32, 13824, 5120, 32), (8, 5120, 13824, 0), (9, 15360, 5120, 0),
    # skinny weight-stream path (M <= 16, mma.sync over TMA stages): ragged K stages / n-blocks
    (8, 5120, 5120, 16), (1, 32, 64, 16), (16, 13824, 5120, 16), (5, 1920, 5120, 16), (3, 96, 320, 16),
    (16, 5120, 13824, 16),
    # few 128x256 tiles: one wave, or split along K
    (1108, 3584, 18944, 0), (300, 5120, 5120, 0), (200, 3584, 13824, 0),
    # two m16 tiles (17..32 rows)
    (24, 5120, 5120, 16), (32, 13824, 5120, 16), (17, 96, 320, 16),
])
def test_gemm_bf16_tcgen05(M, N, K, bn):
    import torch
    torch.manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    lib = kb.load_library()
    rc = lib.keep_debug_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, bn)
    assert rc == 0, lib.keep_last_error()
    ref = A.float() @ B.float().T
    err = (C - ref).abs().max().item()
    # fp32 accumulation in a different order: |err| << sqrt(K) * |a||b|
    assert err <= 2e-3 * np.sqrt(K), (err, M, N, K, bn)
    assert not torch.isnan(C).any()
