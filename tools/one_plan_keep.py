"""One C3 plan_keep (for ncu captures): python tools/one_plan_keep.py [fast|parity] [c3|c2|...]
The setup (weights, canonical KV) runs before cudaProfilerStart, so
`ncu --profile-from-start off` captures only the plan_keep launches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, paper_2602_23592_b200 as kb
mode = kb.PARITY if len(sys.argv) > 1 and sys.argv[1] == "parity" else kb.FAST
cfg = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c3"]
lay, q = bench.workload(cfg, 20250807)
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode)
ctx.model_init(); ctx.memory_compute_layout(lay)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ctx.plan_keep(lay, q, kb.ratio_schedule(cfg["L"], cfg["r_avg"]), final_hidden=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
