"""A/B of the PARITY kernels at C3 width (env KEEP_PARITY_GEMM / KEEP_PARITY_ATTN /
KEEP_OZ_MODULI select them): final query rows, logits top-1, plans / orders.
    python tools/parity_ab.py L out.npz [summaries]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench, paper_2602_23592_b200 as kb
L = int(sys.argv[1]); out = sys.argv[2]; summ = len(sys.argv) > 3
cfg = bench.CONFIGS["c3"]
lay, q = bench.workload(cfg, 20250807)
r48 = kb.ratio_schedule(48, cfg["r_avg"])
with kb.Context(L, cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, kb.PARITY) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    res = ctx.plan_keep(lay, q, r48[:L], final_hidden=True, summaries=summ)
fh = res["final_hidden"]
np.savez(out, q=fh[-len(q):], logits=res["last_logits"], plan=res["plan"], hops=res["hops"],
         order0=np.array(res["orders"][0] or [], np.int32), ttft=res["ttft_ms"],
         qts0=res["qts"][0] if summ else np.zeros(1))
print(json.dumps({"L": L, "env": {k: os.environ.get(k) for k in ("KEEP_PARITY_GEMM", "KEEP_PARITY_ATTN", "KEEP_OZ_MODULI")},
                  "ttft_ms": res["ttft_ms"], "finite": bool(np.isfinite(fh).all()), "top1": int(np.argmax(res["last_logits"])),
                  "qmax": float(np.nanmax(np.abs(fh[-len(q):]))), "hops": [int(x) for x in res["hops"][:21]]}), flush=True)
