"""Step-by-step GPU bring-up trace (prints after every ABI call)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.time()
def log(*a):
    print(f"[{time.time()-t0:7.2f}s]", *a, flush=True)
import numpy as np
log("numpy")
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle
ko = Oracle("ko")
log("libs")
seed, S, L, H, d, mlp, V = 2, 8, 4, 4, 32, 64, 128
p = ko.make_instance(seed, S, L, H, d, mlp, V)
w = ko.model_init(L, H, d, mlp, V, seed)
sched = ko.ratio_schedule(L, 0.5)
ref = ko.plan_keep(p, w, sched)
log("oracle done")
ctx = kb.Context(L, H, d, mlp, V, seed, kb.PARITY)
log("ctx")
ctx.model_init(); log("model_init")
ew = ctx.export_weights(); log("export", np.array_equal(ew, w))
lay = kb.Layout(p.seg_len, p.tokens)
ctx.memory_compute_layout(lay); log("memory_compute")
ctx.prefill_begin(lay, p.query); log("begin")
for l in range(L):
    q, s = ctx.prefill_layer(ref["plan"][l]); log("layer", l, q[:3])
fh, kv = ctx.prefill_finish(); log("finish", float(np.abs(fh - ref["final_hidden"]).max()))
o = ctx.importance_evaluation([0.05,0.10,0.15,0.70], [[0,0,0,0],[0.8,0,0,0],[0,0,0,0],[0.1,0.75,0.1,0]], 3); log("select", o)
got = ctx.plan_keep(lay, p.query, sched); log("plan_keep", got["plan"].sum(1), got["hops"], got["ttft_ms"])
