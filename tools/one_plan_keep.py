"""One C3 plan_keep (for ncu captures): python tools/one_plan_keep.py [fast|parity]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2602_23592_b200 as kb
mode = kb.PARITY if len(sys.argv) > 1 and sys.argv[1] == "parity" else kb.FAST
cfg = bench.CONFIGS["c3"]
lay, q = bench.workload(cfg, 20250807)
ctx = kb.Context(cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode)
ctx.model_init(); ctx.memory_compute_layout(lay)
ctx.plan_keep(lay, q, kb.ratio_schedule(cfg["L"], cfg["r_avg"]), final_hidden=False)
