"""TTFT with and without the per-phase profiler (host-gap probe)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2602_23592_b200 as kb
cfg = bench.CONFIGS["c3"]
layout, query = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.FAST)
ctx.model_init()
ctx.memory_compute_layout(layout)
for _ in range(3):
    ctx.plan_keep(layout, query, r, final_hidden=False)
a = [ctx.plan_keep(layout, query, r, final_hidden=False)["ttft_ms"] for _ in range(3)]
ctx.profile_enable(True)
b = [ctx.plan_keep(layout, query, r, final_hidden=False)["ttft_ms"] for _ in range(3)]
ctx.profile_enable(False)
t0 = time.perf_counter()
res = ctx.plan_keep(layout, query, r, final_hidden=False)
wall = (time.perf_counter() - t0) * 1e3
print("no-prof", np.round(a, 2), "prof", np.round(b, 2), "wall", round(wall, 2))
lm = res["layer_ms"]
print("layer ms", np.round(lm[:4], 3), np.round(lm[18:22], 3), np.round(lm[-3:], 3), "sum", round(float(np.sum(lm)), 2))
