"""Compare the FAST summary (qts, sts) against the fp64 oracle for one
instance; run with KEEP_ATTN_V1=1 / unset to A/B the bins path."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle

ko = Oracle("ko")
seed, S, L, H, d, mlp, V = int(sys.argv[1]) if len(sys.argv) > 1 else 50, 60, 2, 2, 256, 256, 512
p = ko.make_instance(seed, S, L, H, d, mlp, V)
w = ko.model_init(L, H, d, mlp, V, seed)
plan = np.ones((L, S), np.uint8)
ref = ko.selective_prefill(p, w, plan)
lay = kb.Layout(p.seg_len, p.tokens)
with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    got = ctx.selective_prefill(lay, p.query, plan)
for l in range(L):
    q, s = got["qts"][l], got["sts"][l]
    rq, rs = ref["qts"][l], ref["sts"][l]
    print(f"layer {l}: qts rel {np.max(np.abs(q-rq))/np.max(np.abs(rq)):.3e}  sts rel {np.max(np.abs(s-rs))/np.max(np.abs(rs)):.3e}"
          f"  sts sum got {s.sum():.6f} ref {rs.sum():.6f}  zeros got {(s[np.tril_indices(S,-1)]==0).sum()} ref {(rs[np.tril_indices(S,-1)]==0).sum()}")
    bad = np.argwhere(np.abs(s - rs) > 0.05 * np.abs(rs).max())
    print("  first bad (src,dst):", bad[:10].tolist())
    if len(bad):
        i, j = bad[0]
        print("  got", s[i, max(0,j-3):j+4], "\n  ref", rs[i, max(0,j-3):j+4])
