"""tcgen05 GEMM microbenchmark at the C3 layer shapes (plain fp32-store epilogue)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_23592_b200 as kb
lib = kb.load_library()
for (M, N, K, name) in [(8450, 15360, 5120, "qkv"), (8450, 5120, 5120, "wo"), (8450, 13824, 5120, "mlp_in"),
                        (8450, 5120, 13824, "mlp_out"), (16280, 5120, 5120, "wo L0")]:
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.float32)
    for i in range(3):
        lib.keep_debug_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1000)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record()
    for i in range(it):
        lib.keep_debug_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1000)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"{name:8s} M={M} N={N} K={K}: {ms*1e3:.0f} us  {2*M*N*K/ms/1e9:.0f} TFLOP/s")
