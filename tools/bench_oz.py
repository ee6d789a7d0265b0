"""Ozaki int8 GEMM microbenchmark (keep_debug_gemm_parity mode 1) at the C3
layer-0 shapes; KEEP_OZ_MODULI / KEEP_OZ_PAIR select the variant (read once
per process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_23592_b200 as kb

lib = kb.load_library()
shapes = [(16288, 15360, 5120, "qkv L0"), (16288, 5120, 5120, "wo L0"), (16288, 13824, 5120, "mlp_in L0"),
          (16288, 5120, 13824, "mlp_out L0")]
if len(sys.argv) > 1:
    shapes = shapes[:int(sys.argv[1])]
U = int(os.environ.get("KEEP_OZ_MODULI", "14"))
for (M, N, K, name) in shapes:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(2):
        assert lib.keep_debug_gemm_parity(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 5
    e0.record()
    for _ in range(it):
        lib.keep_debug_gemm_parity(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"U={U} pair={os.environ.get('KEEP_OZ_PAIR', '1')} {name:10s} M={M} N={N} K={K}: {ms:.2f} ms  "
          f"{2 * M * N * K * U / ms / 1e9:.0f} int8 TOP/s", flush=True)
