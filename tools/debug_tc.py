import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_23592_b200 as kb
from oracle.oracle import Oracle
ko = Oracle("ko")
seed, S, L, H, d, mlp, V = 50, 20, 4, 2, 256, 512, 512
p = ko.make_instance(seed, S, L, H, d, mlp, V)
lay = kb.Layout(p.seg_len, p.tokens)
print("T", p.T, flush=True)
with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as ctx:
    ctx.model_init()
    print("init ok", flush=True)
    ctx.memory_compute_layout(lay)
    print("refresh ok", flush=True)
