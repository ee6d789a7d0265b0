"""Per-layer device time of one batched plan_keep (cursor-free): layer_ms and
the CACHED phase per call, C3/C4, HBM or host memory."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
cfgname, mem, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = bench.CONFIGS[cfgname]
lay, q = bench.workload(cfg, 20250807)
r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
rng = np.random.default_rng(7)
Q = rng.integers(0, cfg["V"], size=(B, len(q))).astype(np.int32)
Q[0] = q
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.FAST)
ctx.model_init()
ctx.memory_compute_layout(lay, tier=kb.TIER_HOST if mem == "host" else kb.TIER_DEVICE)
ctx.plan_keep_batch(lay, Q, r)
ctx.profile_enable(True)
ctx.profile_read(reset=True)
res = ctx.plan_keep_batch(lay, Q, r)
pr = ctx.profile_read(reset=True)
print("ttft", res[0]["ttft_ms"])
print("layer_ms", np.round(res[0]["layer_ms"], 2).tolist())
print({k: (round(v["ms"], 2), v["launches"]) for k, v in pr.items() if v["launches"]})
