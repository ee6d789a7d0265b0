"""Per-layer device times of one C3 plan_keep: python tools/layer_times.py [fast|parity] [c3|c2|...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
mode = kb.PARITY if len(sys.argv) > 1 and sys.argv[1] == "parity" else kb.FAST
cfg = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c3"]
lay, q = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
with kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    ctx.plan_keep(lay, q, r, final_hidden=False)
    res = ctx.plan_keep(lay, q, r, final_hidden=False)
    lm = np.asarray(res["layer_ms"])
    print(json.dumps({"ttft_ms": res["ttft_ms"], "layer_ms": [round(float(x), 3) for x in lm],
                      "rows": [int(x) for x in res["rows_per_layer"]], "hops": [int(x) for x in res["hops"]]}))
