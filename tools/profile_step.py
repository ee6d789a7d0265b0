"""One KEEP prefill under the CUDA profiler API (for ncu --profile-from-start off).

    python tools/profile_step.py [--config c3] [--layers L]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2602_23592_b200 as kb

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--numerics", default="fast")
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
if args.layers:
    cfg["L"] = args.layers
layout, query = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], max(cfg["r_avg"], 1.0 / cfg["L"]))
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807,
                 kb.FAST if args.numerics == "fast" else kb.PARITY)
ctx.model_init()
ctx.memory_compute_layout(layout)
res = ctx.plan_keep(layout, query, r, final_hidden=False)  # warm-up
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.steps):
    res = ctx.plan_keep(layout, query, r, final_hidden=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ttft_ms", res["ttft_ms"], "rows", res["rows_per_layer"].tolist()[:6])
