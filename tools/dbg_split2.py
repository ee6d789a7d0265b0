import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle
ko = Oracle("ko")
def rel(a, b): return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
for seed, S, L, H, d, mlp, V in [(51, 40, 3, 4, 512, 1024, 700), (52, 100, 2, 2, 256, 256, 512), (53, 300, 2, 1, 128, 128, 256)]:
    p = ko.make_instance(seed, S, L, H, d, mlp, V)
    w = ko.model_init(L, H, d, mlp, V, seed)
    sched = ko.ratio_schedule(L, 0.5)
    refp = ko.plan_keep(p, w, sched, kv=True)
    lay = kb.Layout(p.seg_len, p.tokens)
    with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as ctx:
        ctx.model_init(); ctx.memory_compute_layout(lay)
        sel = ctx.selective_prefill(lay, p.query, refp["plan"])
    print(os.environ.get("KEEP_ATTN_SPLITS"), seed, "T", p.T, "rows/layer", refp["plan"].sum(1), "hidden", round(rel(sel["final_hidden"], refp["final_hidden"]),4),
          "kv", [round(rel(sel["kv"][l], refp["kv"][l]),4) for l in range(L)], "sts", round(rel(sel["sts"], refp["sts"]), 4))
