"""bench.py host logic on CPU: strict JSON, the attention work model, the
reference arm's workload model and its one-layer extrapolation."""
import json
import math

import numpy as np

import bench
import paper_2602_23592_b200 as kb


def test_finite_makes_strict_json():
    line = {"a": float("nan"), "b": [1.0, float("inf")], "c": {"d": -float("inf"), "e": 2}}
    out = bench._finite(line)
    assert out == {"a": None, "b": [1.0, None], "c": {"d": None, "e": 2}}
    json.loads(json.dumps(out, allow_nan=False))


def test_attention_pairs_counts_visible_keys():
    lay = kb.Layout(np.array([3, 2, 4], np.int32), np.arange(9, dtype=np.int32) % 7)
    plan = np.array([[1, 1, 1], [0, 1, 0]], np.uint8)
    pairs = bench.attention_pairs(lay, 2, plan)
    # layer 0: every row t of 9 memory + 2 query rows sees t + 1 keys
    assert pairs[0] == sum(t + 1 for t in range(11))
    # layer 1: segment 1 (rows 3, 4) and the query (rows 9, 10)
    assert pairs[1] == (4 + 5) + (10 + 11)


def test_plan_fixture_roundtrip(tmp_path, monkeypatch):
    fx = {"config": "c1", "S": 5, "L": 3, "runs": [[0, 1, [0, 1, 2, 3, 4]], [1, 3, [1, 3]]]}
    path = tmp_path / "c1_plan.json"
    path.write_text(json.dumps(fx))
    monkeypatch.setattr(bench, "PLAN_FIXTURE", str(tmp_path / "{}_plan.json"))
    plan = bench.plan_from_fixture("c1", 5, 3)
    assert plan.tolist() == [[1, 1, 1, 1, 1], [0, 1, 0, 1, 0], [0, 1, 0, 1, 0]]
    assert bench.plan_from_fixture("c3", 5, 3) is None  # another config: no fixture


def test_committed_c3_plan_fixture_is_monotone():
    cfg = bench.CONFIGS["c3"]
    plan = bench.plan_from_fixture("c3", cfg["S"], cfg["L"])
    if plan is None:
        import pytest
        pytest.skip("no committed C3 plan fixture")
    assert plan[0].all()  # layer 0 recomputes everything (recompute.hpp:149)
    assert all(((plan[l + 1] <= plan[l]).all()) for l in range(cfg["L"] - 1))  # prefill.hpp:227-231


def test_walk_margins_follow_converge():
    # the hand trace of test_recompute.cpp:55-68: order {3, 1, 0}, scores 0.70 / 0.75 / 0.45 vs 0.05
    q = np.array([0.05, 0.10, 0.15, 0.70])
    a = np.array([[0, 0, 0, 0], [0.80, 0, 0, 0], [0, 0, 0, 0], [0.10, 0.75, 0.10, 0]])
    g = bench.walk_margins(q, a, [3, 1, 0], np.ones(4, bool))
    assert math.isclose(g[0], (0.70 - 0.15) / 0.70)
    assert math.isclose(g[1], (0.75 - 0.10) / 0.75)
    assert math.isclose(g[2], (0.45 - 0.05) / 0.45)


def test_selection_parity_reports_first_difference():
    L, S = 2, 4
    q = np.array([0.05, 0.10, 0.15, 0.70])
    a = np.array([[0, 0, 0, 0], [0.80, 0, 0, 0], [0, 0, 0, 0], [0.10, 0.75, 0.10, 0]])
    plan = np.array([[1, 1, 1, 1], [1, 1, 0, 1]], np.uint8)
    ref = {"plan": plan, "orders": [[3, 1, 0], None], "hops": np.array([3, 0])}
    oth = {"plan": plan.copy(), "orders": [[3, 0, 1], None], "hops": np.array([3, 0])}
    out = bench.selection_parity(ref, oth, {"qts": np.stack([q, q]), "sts": np.stack([a, a])})
    assert out["plans_equal"] == 2 and out["orders_equal"] == 1 and out["hops_equal"]
    assert out["walks"][0]["first_differing_hop"] == 1
    assert math.isclose(out["walks"][0]["margin_at_first_difference"], (0.75 - 0.10) / 0.75)


def test_both_arms_print_the_same_config():
    import argparse
    cfg = bench.CONFIGS["c1"]
    lay, q = bench.workload(cfg, 20250807)
    args = argparse.Namespace(config="c1", seed=20250807, memory="hbm")
    assert (bench.workload_config(args, cfg, lay, q, 1, "parity") ==
            bench.workload_config(args, cfg, lay, q, 1, "reference"))
    assert bench.host_cpu()["logical_cores"] >= 1


def test_cpu_extrapolation_is_linear_in_work():
    cfg = bench.CONFIGS["c3"]
    sample = {"rate": 1.0e9}
    rows = np.array([100, 50], np.int64)
    pairs = np.array([1.0e4, 2.0e3])
    ex = bench.cpu_extrapolate(sample, cfg, rows, pairs)
    d, mlp = cfg["d"], cfg["mlp"]
    macs = 150 * (4.0 * d * d + 2.0 * d * mlp) + 2.0 * d * 1.2e4
    assert math.isclose(ex["ttft_s"], macs / 1.0e9)
    assert math.isclose(ex["tokens_per_s"], 150 / ex["ttft_s"])
