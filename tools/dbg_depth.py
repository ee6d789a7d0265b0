"""Where do hidden states stop being finite with depth (C3 dims, small memory)?"""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import make_instance_layout
H, d, mlp, V, seed = 40, 5120, 13824, 152064, 20250807
inst = make_instance_layout(7, 50, V)
lay = kb.Layout(inst.seg_len, inst.tokens)
for mode, name in ((kb.FAST, "FAST"), (kb.PARITY, "PARITY")):
    for L in (8, 16, 24, 32, 40, 48):
        with kb.Context(L, H, d, mlp, V, seed, mode) as ctx:
            ctx.model_init(); ctx.memory_compute_layout(lay)
            res = ctx.plan_keep(lay, inst.query, np.ones(L), final_hidden=True)
            row = res["final_hidden"][-1]
            fin = np.isfinite(row)
            print(name, L, "finite", bool(fin.all()), "max|row|", float(np.max(np.abs(row[fin]))) if fin.any() else None,
                  "logits finite", bool(np.isfinite(res["last_logits"]).all()), flush=True)
