"""C3 PARITY plan_keep TTFT and per-layer device times (layer_ms): the lazy
summary on (default) or off (KEEP_LAZY_SUMMARY=0)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2602_23592_b200 as kb
cfg = bench.CONFIGS["c3"]
layout, query = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.PARITY)
ctx.model_init()
ctx.memory_compute_layout(layout)
ctx.plan_keep(layout, query, r, final_hidden=False)
res = [ctx.plan_keep(layout, query, r, final_hidden=False) for _ in range(3)]
lm = np.mean([x["layer_ms"] for x in res], axis=0)
print("lazy", os.environ.get("KEEP_LAZY_SUMMARY", "1"), "ttft", [round(x["ttft_ms"], 1) for x in res],
      "layer ms 0,1,19,20", np.round([lm[0], lm[1], lm[19], lm[20]], 2), "hops19", int(res[-1]["hops"][19]))
