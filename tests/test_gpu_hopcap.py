"""The optional converge hop cap (BASELINE configs[3]: "3-hop recompute").

The reference's converge has no hop parameter: it runs until the budget is
filled, the set stabilises, or S hops (recompute.hpp:130-138).  A capped walk
is the one-line variant `hop < min(S, max_hops)`, restated in the CPU oracle
(ko_set_max_hops, oracle/keep_oracle.c) and passed to the device selector as
keep_config.max_hops; 0 keeps the reference's walk.
"""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cap", [1, 2, 3, 5])
@pytest.mark.parametrize("seed,S", [(2, 8), (101, 16), (7, 24)])
def test_capped_plan_keep_matches_restatement(ko, cap, seed, S):
    L, H, d, mlp, V = 6, 4, 32, 64, 128
    p = ko.make_instance(seed, S, L, H, d, mlp, V)
    w = ko.model_init(L, H, d, mlp, V, seed)
    sched = ko.ratio_schedule(L, 0.5)
    try:
        ko.set_max_hops(cap)
        ref = ko.plan_keep(p, w, sched)
    finally:
        ko.set_max_hops(0)
    lay = kb.Layout(p.seg_len, p.tokens)
    with kb.Context(L, H, d, mlp, V, seed, kb.PARITY, max_hops=cap) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        got = ctx.plan_keep(lay, p.query, sched)
    assert np.array_equal(got["plan"], ref["plan"])
    assert got["orders"] == ref["orders"]
    assert np.array_equal(got["hops"], ref["hops"])
    assert int(np.max(got["hops"])) <= cap


def test_uncapped_is_the_reference(ko, golden):
    c = next(x for x in golden["instances"] if x["S"] == 16)
    p = ko.make_instance(c["seed"], c["S"], c["L"], c["H"], c["d"], c["mlp"], c["V"], c["lo"], c["hi"], c["qlen"])
    lay = kb.Layout(p.seg_len, p.tokens)
    with kb.Context(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"], kb.PARITY, max_hops=0) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        got = ctx.plan_keep(lay, p.query, np.array(c["sched"]))
    assert got["plan"].tolist() == c["plan"] and got["orders"] == c["orders"]


def test_selector_cap_on_known_answer():
    # the hand trace (test_recompute.cpp:55-68) walks {3, 1, 0} in 3 hops; capped at 2: {3, 1}
    q = [0.05, 0.10, 0.15, 0.70]
    a = [[0, 0, 0, 0], [0.80, 0, 0, 0], [0, 0, 0, 0], [0.10, 0.75, 0.10, 0]]
    with kb.Context(2, 2, 16, 16, 16, 1, kb.PARITY, max_hops=2) as ctx:
        assert ctx.importance_evaluation(q, a, 3) == ([3, 1], 2)
