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


def test_budget_plan_follows_the_schedule():
    cfg = dict(bench.CONFIGS["c1"])
    lay = kb.Layout(np.full(16, 8, np.int32), np.zeros(128, np.int32))
    r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
    plan = bench.budget_plan(cfg, lay, r)
    sizes = plan.sum(axis=1)
    assert sizes[0] == 16
    assert all(sizes[l] == min(16, kb.layer_budget(r[l], 16)) for l in range(1, cfg["L"]))
    assert all(a >= b for a, b in zip(sizes, sizes[1:]))  # monotone


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
