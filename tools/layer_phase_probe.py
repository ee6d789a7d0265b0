"""Per-layer phase times of the C3 prefill through the cursor (device events)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2602_23592_b200 as kb
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
layout, query = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.FAST)
ctx.model_init()
ctx.memory_compute_layout(layout)
res = ctx.plan_keep(layout, query, r, final_hidden=False)
plan = res["plan"]
ctx.profile_enable(True)
rows = []
for rep in range(2):
    ctx.prefill_begin(layout, query)
    ctx.profile_read(reset=True)
    for l in range(cfg["L"]):
        ctx.prefill_layer(plan[l], summary=False)
        pr = ctx.profile_read(reset=True)
        if rep == 1:
            rows.append({k: (round(v["ms"], 4), v["bytes"], v["flops"]) for k, v in pr.items() if v["launches"]})
    ctx.prefill_finish(kv=False)
for l in sorted(set([0, 1, 5, 10, 19, 20, 27, 30, 47]) & set(range(cfg["L"]))):
    print(l, json.dumps(rows[l]))
a = [(r_["attn_decode"][0], r_["attn_decode"][1]) for r_ in rows[20 if cfg["L"] > 40 else 10:]]
ms = np.mean([x[0] for x in a]); by = np.mean([x[1] for x in a])
print("deep attn ms", ms, "bytes", by, "GB/s", by / ms / 1e6)
