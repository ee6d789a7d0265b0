"""Layer-by-layer cursor (prefill_layer with summaries) over the C3 realised
plan: the first layer whose summary is non-finite.  python tools/summary_probe.py L"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
L = int(sys.argv[1])
cfg = bench.CONFIGS["c3"]
lay, q = bench.workload(cfg, 20250807)
plan = bench.plan_from_fixture("c3", lay.S, 48)[:L]
with kb.Context(L, cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.PARITY) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    ctx.prefill_begin(lay, q)
    for l in range(L):
        qts, sts = ctx.prefill_layer(plan[l], summary=True)
        print(json.dumps({"layer": l, "qts_finite": bool(np.isfinite(qts).all()), "sts_finite": bool(np.isfinite(sts).all()),
                          "qts_sum": float(np.nansum(qts)), "qts_max": float(np.nanmax(qts)) if qts.size else 0}), flush=True)
    fh, _ = ctx.prefill_finish(kv=False)
    print("final finite", bool(np.isfinite(fh).all()), float(np.nanmax(np.abs(fh[-8:]))))
