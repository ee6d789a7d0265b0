import os, sys
import numpy as np
sys.path.insert(0, '.')
import bench
import paper_2602_23592_b200 as kb
cfg = bench.CONFIGS["c3"]
layout, query = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
with kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.FAST) as ctx:
    ctx.model_init(); ctx.memory_compute_layout(layout)
    for name, sch in (("keep", r), ("full", np.ones(cfg["L"]))):
        res = ctx.plan_keep(layout, query, sch, final_hidden=True)
        row = res["final_hidden"][-1]
        lg = res["last_logits"]
        print(name, "row finite", np.isfinite(row).all(), "max|row|", float(np.max(np.abs(row[np.isfinite(row)]))) if np.isfinite(row).any() else None,
              "logits finite", np.isfinite(lg).all(), "max|lg|", float(np.nanmax(np.abs(lg))))
