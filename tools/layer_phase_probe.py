"""Per-layer phase times of the C3 prefill through the cursor (device events):
python tools/layer_phase_probe.py [c2|c3|c4] [fast|parity]"""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2602_23592_b200 as kb
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
mode = kb.PARITY if len(sys.argv) > 2 and sys.argv[2] == "parity" else kb.FAST
layout, query = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode)
ctx.model_init()
ctx.memory_compute_layout(layout)
res = ctx.plan_keep(layout, query, r, final_hidden=False)
plan = res["plan"]
need = [l for l in range(cfg["L"]) if l + 1 < cfg["L"] and res["orders"][l] is not None]
ctx.profile_enable(True)
rows = []
for rep in range(2):
    ctx.prefill_begin(layout, query)
    ctx.profile_read(reset=True)
    for l in range(cfg["L"]):
        ctx.prefill_layer(plan[l], summary=(l in need))
        pr = ctx.profile_read(reset=True)
        if rep == 1:
            rows.append({k: (round(v["ms"], 4), v["bytes"], v["flops"]) for k, v in pr.items() if v["launches"]})
    ctx.prefill_finish(kv=False)
print("summary layers", need)
tot = {}
for l in range(cfg["L"]):
    for k, v in rows[l].items():
        tot[k] = tot.get(k, 0.0) + v[0]
    a = rows[l].get("attn")
    if a:
        print(l, "attn ms %.3f TF/s %.2f" % (a[0], a[2] / a[0] / 1e9 if a[0] else 0),
              "gemm ms %.3f" % sum(rows[l].get(p, (0,))[0] for p in ("qkv", "wo", "mlp_in", "mlp_out")),
              json.dumps({k: v[0] for k, v in rows[l].items()}))
print("totals", json.dumps({k: round(v, 2) for k, v in tot.items()}))
