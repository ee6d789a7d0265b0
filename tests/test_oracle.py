"""Pin the plain-C oracle restatement (oracle/keep_oracle.c).

Checked against (1) the golden vectors generated from the unmodified reference
(tests/golden/reference_golden.json) and (2) the reference
itself behind the C shim (oracle/_ref) on fresh random instances where that
shim is built.  Bit-exact throughout: the restatement performs the same fp64
operation sequence as the reference.
"""
import hashlib

import numpy as np
import pytest

from oracle.oracle import OracleError


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem_of(ko, c):
    p = ko.make_instance(c["seed"], c["S"], c["L"], c["H"], c["d"], c["mlp"], c["V"], c["lo"], c["hi"], c["qlen"])
    p.units = [tuple(u) for u in c["units"]]
    return p


def test_weights_match_golden(ko, golden):
    for c in golden["weights"]:
        w = ko.model_init(*c["cfg"])
        assert w.size == c["count"]
        assert sha(w) == c["sha"], c["cfg"]
        assert [float(x) for x in w[:16]] == c["head"]


def test_ratio_schedule_and_budgets(ko, golden):
    for c in golden["ratio_schedule"]:
        if "error" in c:
            with pytest.raises(OracleError) as ei:
                ko.ratio_schedule(c["L"], c["r_avg"])
            assert ei.value.kind == c["error"]
        else:
            assert [float(x) for x in ko.ratio_schedule(c["L"], c["r_avg"])] == c["r"]
    for c in golden["layer_budget"]:
        assert ko.layer_budget(c["ratio"], c["S"]) == c["budget"]
    # test_recompute.cpp:134-157: mean and geometric profile
    r = ko.ratio_schedule(4, 0.55)
    assert abs(r.mean() - 0.55) <= 1e-6 and r[0] == 1.0
    assert abs(r[2] / r[1] - r[1] / r[0]) < 1e-9


def test_converge_known_answers(ko, golden):
    for c in golden["converge"]:
        order, hops = ko.converge(c["qts"], c["sts"], c["budget"], c.get("candidates"))
        assert (order, hops) == (c["order"], c["hops"]), c["name"]
    hand = next(c for c in golden["converge"] if c["name"] == "hand_trace")
    assert hand["order"] == [3, 1, 0] and hand["hops"] == 3


def test_instances_match_golden(ko, golden):
    for c in golden["instances"]:
        p = problem_of(ko, c)
        assert [int(x) for x in p.seg_len] == c["seg_len"] and sha(p.tokens) == c["tokens_sha"]
        w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
        res = ko.plan_keep(p, w, np.array(c["sched"]), multihop=c["multihop"], kv=True)
        tag = (c["seed"], c["S"], c["r_avg"], c["multihop"])
        assert res["plan"].tolist() == c["plan"], tag
        assert res["orders"] == c["orders"], tag
        assert res["hops"].tolist() == c["hops"], tag
        assert res["qts"].tolist() == c["qts"], tag
        assert res["sts"].tolist() == c["sts"], tag
        assert sha(res["final_hidden"]) == c["final_hidden_sha"], tag
        assert sha(res["kv"]) == c["kv_sha"], tag
        assert sha(ko.canonical_kv(p, w)) == c["canonical_kv_sha"], tag
        full = ko.full_prefill(p, w, kv=False)
        assert sha(full["final_hidden"]) == c["full_final_hidden_sha"], tag
        l2, kl = ko.divergence(p, w, res["final_hidden"][-1], full["final_hidden"][-1])
        assert np.array_equal([l2, kl], [c["div_l2"], c["div_kl"]], equal_nan=True), tag


def test_witness_and_acceptance_properties(ko, golden):
    inst = golden["instances"]
    # seed 2 keep@0.5 plan (acceptance.cpp:84-110)
    w2 = next(c for c in inst if c["seed"] == 2 and c["r_avg"] == 0.5 and c["multihop"] and not c["units"])
    assert w2["plan"] == [[1] * 8, [1, 1, 1, 1, 0, 0, 0, 1], [1, 0, 0, 1, 0, 0, 0, 1], [0, 0, 0, 1, 0, 0, 0, 1]]
    assert abs(w2["div_l2"] - 2.1777) < 1e-4
    # oracle degeneracy: keep@1.0 == full prefill (acceptance.cpp:39-58)
    for c in inst:
        if c["r_avg"] == 1.0:
            assert c["final_hidden_sha"] == c["full_final_hidden_sha"]
            assert c["div_l2"] == 0.0 and c["div_kl"] == 0.0


def test_errors(ko):
    p = ko.make_instance(15, 2)
    w = ko.model_init(4, 4, 32, 64, 128, 15)
    bad = p.tokens.copy()
    bad[0] = 128 + 3
    p2 = type(p)(**{**p.__dict__, "tokens": bad})
    with pytest.raises(OracleError) as ei:
        ko.full_prefill(p2, w)
    assert ei.value.kind == "InputError"
    grow = np.zeros((4, 2), np.uint8)
    grow[1, 0] = 1
    with pytest.raises(OracleError) as ei:
        ko.selective_prefill(p, w, grow)
    assert ei.value.kind == "PlanError"
    with pytest.raises(OracleError) as ei:
        ko.model_init(4, 3, 32, 64, 128, 1)
    assert ei.value.kind == "ConfigError"


@pytest.mark.parametrize("seed", [7, 19, 404])
def test_restatement_equals_reference_random(ko, kr, seed):
    rng = np.random.default_rng(seed)
    L, H = int(rng.integers(1, 7)), int(rng.choice([1, 2, 4, 8]))
    d = H * int(rng.choice([2, 4, 8]))
    mlp, V = int(rng.integers(4, 80)), int(rng.integers(16, 300))
    S = int(rng.integers(1, 14))
    p = kr.make_instance(seed, S, L, H, d, mlp, V, 1, 9, int(rng.integers(0, 9)))
    cuts = sorted(set(int(x) for x in rng.integers(1, S, size=2))) if S > 2 else []
    bounds = [0] + cuts + [S]
    p.units = [(bounds[i], bounds[i + 1], int(rng.integers(0, 2))) for i in range(len(bounds) - 1)]
    w = kr.model_init(L, H, d, mlp, V, seed)
    assert np.array_equal(w, ko.model_init(L, H, d, mlp, V, seed))
    r = kr.ratio_schedule(L, max(1.0 / L, float(rng.uniform(0.2, 1.0))))
    a = ko.plan_keep(p, w, r, kv=True)
    b = kr.plan_keep(p, w, r, kv=True)
    for k in ["plan", "hops", "qts", "sts", "final_hidden", "kv"]:
        assert np.array_equal(a[k], b[k]), k
    assert a["orders"] == b["orders"]


def test_hop_cap_restatement(ko, golden):
    """ko_set_max_hops: the capped walk stops at max_hops hops; a cap >= S is the reference."""
    c = next(x for x in golden["converge"] if x["name"] == "hand_trace")
    try:
        ko.set_max_hops(2)
        assert ko.converge(c["qts"], c["sts"], c["budget"]) == ([3, 1], 2)
        ko.set_max_hops(1)
        assert ko.converge(c["qts"], c["sts"], c["budget"]) == ([3], 1)
        ko.set_max_hops(100)
        assert ko.converge(c["qts"], c["sts"], c["budget"]) == (c["order"], c["hops"])
    finally:
        ko.set_max_hops(0)
    assert ko.converge(c["qts"], c["sts"], c["budget"]) == (c["order"], c["hops"])
