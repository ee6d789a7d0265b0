"""Per-layer summaries of one golden instance through the cursor (for A/B of
the PARITY attention kernels): python tools/summ_ab.py out.npz [seed S L H d mlp V]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle
ko = Oracle("ko")
out = sys.argv[1]
seed, S, L, H, d, mlp, V = [int(x) for x in (sys.argv[2:9] if len(sys.argv) > 8 else [103, 12, 16, 4, 32, 64, 128])]
p = ko.make_instance(seed, S, L, H, d, mlp, V)
plan = np.ones((L, S), np.uint8)
lay = kb.Layout(p.seg_len, p.tokens)
with kb.Context(L, H, d, mlp, V, seed, kb.PARITY) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    res = ctx.selective_prefill(lay, p.query, plan)
w = ko.model_init(L, H, d, mlp, V, seed)
ref = ko.selective_prefill(p, w, plan)
np.savez(out, qts=res["qts"], sts=res["sts"], rq=ref["qts"], rs=ref["sts"], fh=res["final_hidden"], rfh=ref["final_hidden"])
for l in range(L):
    print(l, "qts sum got %.17g ref %.17g  max|dq| %.3g  max|ds| %.3g" % (res["qts"][l].sum(), ref["qts"][l].sum(),
          np.max(np.abs(res["qts"][l] - ref["qts"][l])), np.max(np.abs(res["sts"][l] - ref["sts"][l]))))
