"""Full-scale selection parity: the C3 plan_keep in PARITY (fp32 storage,
fp64 accumulation -- the reference's arithmetic) against FAST (bf16 tensor
cores) on the same synthetic weights, memory and query.  Writes a JSON
summary (plans per layer, walk orders, hops, last-row drift, logits top-1)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/c3_parity.json"
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
        res[name] = ctx.plan_keep(lay, q, r, final_hidden=True)
    res[name]["wall_s"] = time.time() - t0
    print(name, "ttft_ms", res[name]["ttft_ms"], "wall", res[name]["wall_s"], flush=True)
P, F = res["parity"], res["fast"]
L = cfg["L"]
same_plan = [bool(np.array_equal(P["plan"][l], F["plan"][l])) for l in range(L)]
same_order = [P["orders"][l] == F["orders"][l] for l in range(L)]
hp, hf = P["final_hidden"][-len(q):].astype(np.float64), F["final_hidden"][-len(q):].astype(np.float64)
summary = {
    "config": cfgname, "S": lay.S, "T": int(np.sum(lay.seg_len)) + len(q),
    "parity_ttft_ms": P["ttft_ms"], "fast_ttft_ms": F["ttft_ms"],
    "plan_segments_per_layer_parity": [int(x) for x in P["plan"].sum(axis=1)],
    "plan_segments_per_layer_fast": [int(x) for x in F["plan"].sum(axis=1)],
    "layers_with_identical_plan": int(sum(same_plan)), "layers": L,
    "walk_orders_identical": [i for i, x in enumerate(same_order) if x and P["orders"][i] is not None],
    "walk_orders_differ": [i for i, x in enumerate(same_order) if not x],
    "hops_parity": [int(x) for x in P["hops"]], "hops_fast": [int(x) for x in F["hops"]],
    "query_rows_rel_max_diff": float(np.max(np.abs(hp - hp * 0 - hf)) / max(np.max(np.abs(hp)), 1e-300)),
    "logits_top1_parity": int(np.argmax(P["last_logits"])), "logits_top1_fast": int(np.argmax(F["last_logits"])),
}
print(json.dumps(summary))
os.makedirs(os.path.dirname(out), exist_ok=True)
with open(out, "w") as f:
    json.dump(summary, f, indent=1)
