import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle
ko = Oracle("ko")
seed, S, L, H, d, mlp, V = 50, 20, 4, 2, 256, 512, 512
p = ko.make_instance(seed, S, L, H, d, mlp, V)
w = ko.model_init(L, H, d, mlp, V, seed)
plan = np.ones((L, S), np.uint8)
ref = ko.selective_prefill(p, w, plan)
lay = kb.Layout(p.seg_len, p.tokens)
with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as ctx:
    ctx.model_init(); ctx.memory_compute_layout(lay)
    got = ctx.selective_prefill(lay, p.query, plan)
def rel(a, b): return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
print(os.environ.get("KEEP_ATTN_SPLITS"), "T", p.T, "hidden", rel(got["final_hidden"], ref["final_hidden"]), "kv", [rel(got["kv"][l], ref["kv"][l]) for l in range(L)], "qts", rel(got["qts"], ref["qts"]))
