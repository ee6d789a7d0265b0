"""Weight-stream GEMM microbenchmark (M <= 16): GB/s of the skinny path vs the
tcgen05 split-K path, CUDA events, weights larger than L2."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_23592_b200 as kb
lib = kb.load_library()
for (M, N, K) in [(8, 15360, 5120), (8, 13824, 5120), (8, 5120, 13824), (8, 5120, 5120), (8, 1920, 5120)]:
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    Bs = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(4)]  # > L2 in total
    C = torch.empty(M, N, device="cuda", dtype=torch.float32)
    for bn in (16, 32):
        for i in range(3):
            lib.keep_debug_gemm_bf16(A.data_ptr(), Bs[i % 4].data_ptr(), C.data_ptr(), M, N, K, bn + 1000)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 40
        e0.record()
        for i in range(it):
            lib.keep_debug_gemm_bf16(A.data_ptr(), Bs[i % 4].data_ptr(), C.data_ptr(), M, N, K, bn + 1000)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        print(f"M={M} N={N} K={K} path={'skinny' if bn == 16 else 'tc-splitk'} {ms*1e3:.1f} us {2*N*K/ms/1e6:.0f} GB/s")
