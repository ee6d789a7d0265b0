"""Full-scale selection parity and the realised-plan fixture.

Runs plan_keep on a BASELINE config in PARITY (the reference's arithmetic)
and in FAST (bf16) on the same synthetic weights, memory and query; writes
  * <out>: bench.selection_parity of FAST against PARITY (plans, walk orders,
    hops per layer, the PARITY walks' decision margins) plus both TTFTs;
  * tests/golden/<config>_realized_plan.json (with --fixture): the PARITY
    plan as runs of layers sharing one segment set -- the realised workload
    the CPU reference arm of bench.py extrapolates to.

    python tools/c3_parity.py [c3] [gpurun_out/c3_parity.json] [--fixture]
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfgname = args[0] if args else "c3"
out = args[1] if len(args) > 1 else "gpurun_out/c3_parity.json"
cfg = bench.CONFIGS[cfgname]
lay, q = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
res = {}
for name, mode in (("parity", kb.PARITY), ("fast", kb.FAST)):
    t0 = time.time()
    with kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        ctx.plan_keep(lay, q, r, final_hidden=False)  # warm
        res[name] = ctx.plan_keep(lay, q, r, final_hidden=True, summaries=(name == "parity"))
    res[name]["wall_s"] = time.time() - t0
    print(name, "ttft_ms", res[name]["ttft_ms"], "wall", res[name]["wall_s"], flush=True)
P, F = res["parity"], res["fast"]
summ = {"qts": P.pop("qts"), "sts": P.pop("sts")}
sel = bench.selection_parity(P, F, summ)
hp, hf = P["final_hidden"][-len(q):].astype(np.float64), F["final_hidden"][-len(q):].astype(np.float64)
summary = {"config": cfgname, "S": lay.S, "T": int(np.sum(lay.seg_len)) + len(q),
           "parity_ttft_ms": P["ttft_ms"], "fast_ttft_ms": F["ttft_ms"],
           "oz_moduli": int(os.environ.get("KEEP_OZ_MODULI", "14")),
           "plan_segments_per_layer_parity": [int(x) for x in P["plan"].sum(axis=1)],
           "plan_segments_per_layer_fast": [int(x) for x in F["plan"].sum(axis=1)],
           "hops_parity": [int(x) for x in P["hops"]], "hops_fast": [int(x) for x in F["hops"]],
           "selection_parity": sel,
           "query_rows_rel_max_diff": float(np.max(np.abs(hp - hf)) / max(np.max(np.abs(hp)), 1e-300)),
           "logits_top1_parity": int(np.argmax(P["last_logits"])), "logits_top1_fast": int(np.argmax(F["last_logits"])),
           "parity_orders": {str(l): P["orders"][l] for l in range(cfg["L"]) if P["orders"][l] is not None}}
print(json.dumps({k: v for k, v in summary.items() if k != "parity_orders"}))
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump(bench._finite(summary), f, indent=1)
if "--fixture" in sys.argv:
    runs, l = [], 0
    plan = P["plan"]
    while l < cfg["L"]:
        e = l + 1
        while e < cfg["L"] and np.array_equal(plan[e], plan[l]):
            e += 1
        runs.append([l, e, [int(i) for i in np.nonzero(plan[l])[0]]])
        l = e
    fx = {"generator": "tools/c3_parity.py (GPU PARITY plan_keep; layers 0-1 pinned to oracle/_ref by "
                       "tests/golden/c3_width_golden.npz)", "config": cfgname, "seed": 20250807,
          "S": lay.S, "L": cfg["L"], "runs": runs,
          "rows_per_layer": [int(x) for x in P["rows_per_layer"]], "hops": [int(x) for x in P["hops"]]}
    path = os.path.join(bench.ROOT, "tests", "golden", f"{cfgname}_realized_plan.json")
    with open(path, "w") as f:
        json.dump(fx, f, separators=(",", ":"))
    print("wrote", path)
