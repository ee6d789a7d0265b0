"""A/B the FAST summary bins between the v1 (scan) and v2 (tensor-core)
attention at a large shape: python tools/debug_bins2.py out.npz"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import make_instance_layout

S, L, H, d, mlp, V = int(os.environ.get("S", 1638)), 1, int(os.environ.get("H", 40)), int(os.environ.get("D", 5120)), 1024, 1024
inst = make_instance_layout(7, S, V)
lay = kb.Layout(inst.seg_len, inst.tokens)
with kb.Context(L, H, d, mlp, V, 7, kb.FAST) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    ctx.prefill_begin(lay, inst.query)
    q, s = ctx.prefill_layer(np.ones(S, np.uint8))
np.savez(sys.argv[1], q=q, s=s)
