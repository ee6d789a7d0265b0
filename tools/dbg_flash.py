"""Tiny FLASH-attention runs (cursor, no summary), one per process argument set."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import make_instance_layout
S, H, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
L, V, seed = 2, 512, 70
inst = make_instance_layout(seed, S, V)
lay = kb.Layout(inst.seg_len, inst.tokens)
with kb.Context(L, H, d, 2 * d, V, seed, kb.FAST) as ctx:
    ctx.model_init()
    print("init", flush=True)
    ctx.memory_compute_layout(lay)
    print("memory", flush=True)
    ctx.prefill_begin(lay, inst.query)
    for l in range(L):
        print("layer", l, flush=True)
        ctx.prefill_layer(np.ones(S, np.uint8), summary=False)
    fh, kv = ctx.prefill_finish()
print("ok", np.isfinite(fh).all(), float(np.abs(fh).max()), flush=True)
