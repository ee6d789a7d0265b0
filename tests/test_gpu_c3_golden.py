"""BASELINE configs[2] (C3: Qwen2.5-14B dims, the bench's 16,280-token memory
and query) pinned to the UNMODIFIED reference at full width.

tests/golden/c3_width_golden.npz comes from oracle/_ref (the reference
headers compiled in place) by tests/golden/make_c3_golden.py: plan_keep on the
first two layers with r[0..1] of the 48-layer schedule.  The weights are
per-name counter streams (model.hpp:54-73), so these are the 48-layer model's
layers 0 and 1 exactly: the layer-0 summary, the ~850-hop layer-0 walk
(converge, recompute.hpp:130-138) that decides the whole C3 plan, and the
layer-1 plan.  Both PARITY modes must reproduce the plan, the walk order and
the hop counts bit-exactly; summaries and hidden states within the fp64
re-ordering tolerances of tests/test_gpu_parity.py.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import bench
import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c3_width_golden.npz")


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)))) / max(float(np.max(np.abs(b))), 1e-300)


SHA = GOLD + ".sha256"  # recorded when the generated golden is adopted


@pytest.fixture(scope="module")
def gold():
    if not os.path.exists(GOLD):
        pytest.skip("C3-width golden not generated (tests/golden/make_c3_golden.py)")
    if not os.path.exists(SHA):
        pytest.skip("C3-width golden generated but not adopted (no recorded sha256)")
    with open(GOLD, "rb") as f:
        digest = hashlib.sha256(f.read()).hexdigest()
    with open(SHA) as f:
        assert digest == f.read().split()[0], "c3_width_golden.npz differs from its recorded sha256"
    g = np.load(GOLD)
    return g, json.loads(bytes(g["meta"]).decode())


@pytest.mark.parametrize("mode", [kb.PARITY, kb.PARITY_EXACT], ids=["parity", "exact"])
def test_c3_width_layers_0_1_match_reference(gold, mode):
    g, meta = gold
    cfg = bench.CONFIGS["c3"]
    L = 2
    lay, q = bench.workload(cfg, meta["config"]["seed"])
    assert lay.S == meta["S"] and int(np.sum(lay.seg_len)) == meta["Tm"]
    with kb.Context(L, cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], meta["config"]["seed"], mode) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        res = ctx.plan_keep(lay, q, np.array(meta["sched"]), final_hidden=True, summaries=True)
        # the canonical KV of the first owner (static group 0: a joint prefill of segments 0..7)
        kind, oid, b, e = lay.owners()[0]
        n0 = int(np.sum(lay.seg_len[b:e]))
        cached0 = [ctx.memory_read(kind, oid, l, n0) for l in range(L)]
    # selections: bit-exact with the reference
    assert np.array_equal(res["plan"], g["plan"])
    assert res["orders"][0] == [int(x) for x in g["order0"]]
    assert res["orders"][1] is None and meta["orders_none"][1]
    assert np.array_equal(res["hops"], g["hops"])
    # summaries (fp64, summation order only)
    assert float(np.max(np.abs(res["qts"] - g["qts"]))) <= 1e-12
    assert np.allclose(res["sts"][0].sum(axis=1), g["sts0_rowsum"], rtol=1e-12, atol=1e-15)
    assert np.allclose(res["sts"][1].sum(axis=1), g["sts1_rowsum"], rtol=1e-12, atol=1e-15)
    picks = g["order0"][:16]
    assert float(np.max(np.abs(res["sts"][0][picks] - g["sts0_rows"]))) <= 1e-12
    # hidden states / canonical KV: fp32 outputs of fp64 sums
    assert rel(res["final_hidden"][-len(q):], g["final_query_rows"]) <= 2e-6
    step = max(1, (meta["T"]) // 64)
    assert rel(res["final_hidden"][::step], g["final_rows_sample"]) <= 2e-6
    for l in range(L):
        k, v = cached0[l]
        assert rel(k[0], g["cached_rows_sample"][l, 0, 0]) <= 2e-6
        assert rel(v[0], g["cached_rows_sample"][l, 1, 0]) <= 2e-6
