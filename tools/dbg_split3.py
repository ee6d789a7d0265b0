import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle
ko = Oracle("ko")
def rel(a, b): return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
seed, S, L, H, d, mlp, V = 51, 40, 2, 4, 512, 1024, 700
p = ko.make_instance(seed, S, L, H, d, mlp, V)
w = ko.model_init(L, H, d, mlp, V, seed)
for act in [S, 15, 1, 0]:
    plan = np.ones((L, S), np.uint8)
    plan[1, :] = 0
    plan[1, :act] = 1
    ref = ko.selective_prefill(p, w, plan)
    lay = kb.Layout(p.seg_len, p.tokens)
    with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as ctx:
        ctx.model_init(); ctx.memory_compute_layout(lay)
        got = ctx.selective_prefill(lay, p.query, plan)
    print(os.environ.get("KEEP_ATTN_SPLITS"), "active@1", act, "hidden", round(rel(got["final_hidden"], ref["final_hidden"]), 4),
          "qts1", round(rel(got["qts"][1], ref["qts"][1]), 4), "sts1", round(rel(got["sts"][1], ref["sts"][1]), 4))
