import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import make_instance_layout
H, d, mlp, V, seed = 40, 5120, 13824, 152064, 20250807
inst = make_instance_layout(7, 50, V)
lay = kb.Layout(inst.seg_len, inst.tokens)
L = 24
out = {}
for mode, name in ((kb.FAST, "FAST"), (kb.PARITY, "PARITY")):
    with kb.Context(L, H, d, mlp, V, seed, mode) as ctx:
        ctx.model_init(); ctx.memory_compute_layout(lay)
        sel = ctx.selective_prefill(lay, inst.query, np.ones((L, lay.S), np.uint8))
        out[name] = sel
for l in range(L):
    kf, kp = out["FAST"]["kv"][l, 0], out["PARITY"]["kv"][l, 0]
    vf = out["FAST"]["kv"][l, 1]
    print(l, "K finite", bool(np.isfinite(kf).all()), "V finite", bool(np.isfinite(vf).all()), "max|K| fast", float(np.nanmax(np.abs(kf))), "parity", float(np.max(np.abs(kp))),
          "rel", float(np.nanmax(np.abs(kf - kp)) / np.max(np.abs(kp))))
