"""Lazy summary (abi.cu run_layer + attn_dmma.cu walk_probe_kernel): a walk
layer whose candidate segments provably receive no query probability (every
candidate key's score is more than 746 + an fp64 error margin below its query
row's max, so its exponential underflows to 0) skips the summary; the
reference's first hop then adds nothing (recompute.hpp:110-121).

C3 at full width with the first 21 layers and r[0..20] of the 48-layer
schedule (the weights are per-name counter streams: these are C3's layers
0-20).  At layer 19 the scores reach ~1e18 and the walk for layer 20 stops at
its first hop.  Plans, walk orders and hop counts must equal the run that
always computes the summary (KEEP_LAZY_SUMMARY=0) and PARITY_EXACT's.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import bench, paper_2602_23592_b200 as kb
cfg = bench.CONFIGS["c3"]
L = 21
lay, q = bench.workload(cfg, 20250807)
sched = kb.ratio_schedule(cfg["L"], cfg["r_avg"])[:L]
mode = kb.PARITY_EXACT if sys.argv[1] == "exact" else kb.PARITY
with kb.Context(L, cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], 20250807, mode) as ctx:
    ctx.model_init()
    ctx.memory_compute_layout(lay)
    ctx.plan_keep(lay, q, sched, final_hidden=False)
    r = ctx.plan_keep(lay, q, sched, final_hidden=False)
print(json.dumps({"plan": r["plan"].astype(int).tolist(), "orders": r["orders"],
                  "hops": [int(x) for x in r["hops"]], "layer_ms": [float(x) for x in r["layer_ms"]]}))
""" % ROOT


def run(mode, env):
    p = subprocess.run([sys.executable, "-c", SCRIPT, mode], cwd=ROOT, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_lazy_summary_keeps_c3_selections():
    lazy = run("parity", {})
    full = run("parity", {"KEEP_LAZY_SUMMARY": "0"})
    exact = run("exact", {})
    assert lazy["hops"][19] == 1 and lazy["orders"][19] == [] and sum(lazy["plan"][20]) == 0
    for other in (full, exact):
        assert lazy["plan"] == other["plan"]
        assert lazy["orders"] == other["orders"]
        assert lazy["hops"] == other["hops"]
    # the skipped summary shows in layer 19's device time; the probe costs little at layer 0
    assert lazy["layer_ms"][19] < full["layer_ms"][19] - 5.0, (lazy["layer_ms"][19], full["layer_ms"][19])
    assert lazy["layer_ms"][0] < full["layer_ms"][0] + 3.0, (lazy["layer_ms"][0], full["layer_ms"][0])
