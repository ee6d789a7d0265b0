"""Host vs device time of the in-place canonical refresh (bench --updates)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
cfg = bench.CONFIGS["c3"]
lay, q = bench.workload(cfg, 20250807)
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.FAST)
ctx.model_init(); ctx.memory_compute_layout(lay)
own = lay.owners(); dyn = [i for i, o in enumerate(own) if o[0] == kb.SEGMENT]
rng = np.random.default_rng(1)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
for it in range(4):
    pick = [u for u in dyn if rng.random() < 0.35]
    ctx.profile_enable(True); ctx.profile_read(reset=True)
    t0 = time.perf_counter(); ctx.memory_refresh(lay, pick, 2 + it); t1 = time.perf_counter()
    res = ctx.plan_keep(lay, q, r, final_hidden=False); t2 = time.perf_counter()
    pr = ctx.profile_read(reset=True)
    print(f"refresh wall {1e3*(t1-t0):.1f} ms (device {pr['refresh']['ms']:.1f})  plan_keep wall {1e3*(t2-t1):.1f} ms (ttft {res['ttft_ms']:.1f})")
