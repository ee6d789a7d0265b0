"""PARITY weight-stream GEMM microbenchmark (keep_debug_gemm_parity mode 3: the
few-row DFMA path with split K): us and GB/s of fp32 weights per launch at the
C3 deep-layer shapes (M = 8 query rows), four weight copies (> L2) in rotation.
KEEP_PARITY_STREAM=0 selects the smem-staged skinny kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_23592_b200 as kb

lib = kb.load_library()
for (M, N, K) in [(8, 15360, 5120), (8, 5120, 5120), (8, 13824, 5120), (8, 5120, 13824), (16, 15360, 5120),
                  (32, 5120, 5120)]:
    A = torch.randn(M, K, device="cuda")
    Bs = [torch.randn(K, N, device="cuda") for _ in range(4)]
    C = torch.empty(M, N, device="cuda")
    ref = (A.double() @ Bs[0].double()).float()
    assert lib.keep_debug_gemm_parity(A.data_ptr(), Bs[0].data_ptr(), C.data_ptr(), M, N, K, 3) == 0
    err = float((C - ref).abs().max() / ref.abs().max())
    for i in range(3):
        lib.keep_debug_gemm_parity(A.data_ptr(), Bs[i % 4].data_ptr(), C.data_ptr(), M, N, K, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record()
    for i in range(it):
        lib.keep_debug_gemm_parity(A.data_ptr(), Bs[i % 4].data_ptr(), C.data_ptr(), M, N, K, 3)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"stream={os.environ.get('KEEP_PARITY_STREAM', '1')} M={M} N={N} K={K}: {ms * 1e3:.1f} us "
          f"{4 * N * K / ms / 1e6:.0f} GB/s  rel err {err:.1e}", flush=True)
