"""Finite-ness of the final hidden state with depth (C3 dims, the bench's memory
and query): plan_keep on the first L layers (weights are per-name, so the
L-layer model is a prefix of the 48-layer one) for several L.
    python tools/depth_probe.py [parity|fast] [L1,L2,...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
mode = kb.FAST if len(sys.argv) > 1 and sys.argv[1] == "fast" else kb.PARITY
Ls = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 16, 24, 32, 40, 44, 48]
cfg = bench.CONFIGS["c3"]
lay, q = bench.workload(cfg, 20250807)
r48 = kb.ratio_schedule(48, cfg["r_avg"])
for L in Ls:
    with kb.Context(L, cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        res = ctx.plan_keep(lay, q, r48[:L], final_hidden=True)
    fh = res["final_hidden"]
    qr = fh[-len(q):]
    print(json.dumps({"L": L, "query_finite": bool(np.isfinite(qr).all()), "all_finite": bool(np.isfinite(fh).all()),
                      "query_max": float(np.max(np.abs(qr[np.isfinite(qr)]))) if np.isfinite(qr).any() else None,
                      "nonfinite_rows": int(np.sum(~np.isfinite(fh).all(axis=1))),
                      "logits_finite": bool(np.isfinite(res["last_logits"]).all()),
                      "top1": int(np.argmax(res["last_logits"]))}), flush=True)
