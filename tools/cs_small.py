import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import make_instance_layout
S, L, H, d, V = 24, 3, 2, 256, 256
inst = make_instance_layout(5, S, V)
lay = kb.Layout(inst.seg_len, inst.tokens)
with kb.Context(L, H, d, 2 * d, V, 5, kb.FAST) as ctx:
    ctx.model_init(); ctx.memory_compute_layout(lay)
    r = ctx.plan_keep(lay, inst.query, kb.ratio_schedule(L, 0.5))
    Q = np.stack([inst.query, inst.query[::-1].copy(), inst.query])
    plans = np.zeros((3, L, S), np.uint8); plans[:, 0] = 1; plans[1, 1, :4] = 1
    b = ctx.plan_keep_batch(lay, Q, None, plans=plans)
print("ok", r["ttft_ms"])
