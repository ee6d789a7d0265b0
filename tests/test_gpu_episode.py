"""Episode replay on the GPU: the memory control plane
drives the B200 prefill engine through the C ABI and reproduces the
UNMODIFIED reference harness (oracle/_ref/libkeep_ref_episode.so).

* compare_csv of the reference's golden episode (seed 20250807, 12 segments,
  4 steps, k=5; test_harness.cpp:231-241) equals proj/tests/golden/
  compare_golden.csv byte for byte (tests/golden/compare_golden.csv);
* every strategy's per-step report -- TTFT time units, refresh charge, plan
  sizes, reuse accounting, invalidated tokens, slow bytes -- equals the
  reference's exactly; divergences (fp64 softmax/KL of GPU logits) within
  1e-9 relative;
* the ablations of test_harness.cpp:255-290 (fixed-block grouping, overlap
  instead of balanced loading) keep the reference's orderings.
"""
import os

import numpy as np
import pytest

import paper_2602_23592_b200 as kb
from paper_2602_23592_b200 import episode as ep
from test_episode_cpu import base_config

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "compare_golden.csv")


@pytest.fixture(scope="module")
def kre():
    from oracle.episode_oracle import EpisodeOracle, available
    if not available():
        pytest.skip("reference episode shim not built (oracle/_ref/libkeep_ref_episode.so)")
    return EpisodeOracle()


_CTX = {}


def ctx_for(cfg, numerics=kb.PARITY):
    key = (cfg.model_seed, numerics, cfg.num_layers, cfg.num_heads, cfg.model_dim, cfg.mlp_dim, cfg.vocab_size)
    if key not in _CTX:
        c = kb.Context(cfg.num_layers, cfg.num_heads, cfg.model_dim, cfg.mlp_dim, cfg.vocab_size, cfg.model_seed,
                       numerics)
        c.model_init()
        _CTX[key] = c
    return _CTX[key]


def close(a, b, rel=1e-9):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def assert_report_equal(got, ref):
    assert len(got["per_step"]) == len(ref["per_step"])
    for g, r in zip(got["per_step"], ref["per_step"]):
        for k in ("step", "realized_segments", "ttft_tu", "makespan_tu", "refresh_tu", "plan_sizes", "reused_tokens",
                  "recomputed_tokens", "memory_tokens", "invalidated_tokens_delta", "bytes_loaded_slow_delta"):
            assert g[k] == r[k], (k, g[k], r[k], g["step"])
        assert close(g["div_l2"], r["div_l2"]) and close(g["div_kl"], r["div_kl"]), (g, r)
    ga, ra = got["aggregate"], ref["aggregate"]
    for k in ("steps", "mean_ttft_tu", "p95_ttft_tu", "reuse_ratio", "mean_realized_segments", "invalidated_tokens",
              "bytes_slow"):
        assert ga[k] == ra[k], (k, ga[k], ra[k])
    assert close(ga["mean_div_l2"], ra["mean_div_l2"]) and close(ga["mean_div_kl"], ra["mean_div_kl"])


def test_compare_csv_reproduces_reference_golden(kre):
    cfg = base_config(20250807, 12, 4, 5)
    tr = ep.generate_episode(cfg)
    got = ep.compare_csv(ctx_for(cfg), tr, ["full", "full-reuse", "keep"], cfg)
    with open(GOLD) as f:
        gold = f.read()
    assert got == gold, (got, gold)
    # and the live reference on the same trace text
    assert got == kre.compare_csv(cfg.to_json(), tr.to_jsonl(), ["full", "full-reuse", "keep"])


@pytest.mark.parametrize("strategy", list(ep.STRATEGIES))
@pytest.mark.parametrize("seed", [7, 20250807, 1003])
def test_run_episode_matches_reference(kre, strategy, seed):
    cfg = base_config(seed)
    if seed == 1003:  # update-heavy (test_harness.cpp:262-268)
        cfg.categories[0].update_prob_per_step = 0.5
        cfg.categories[1].update_prob_per_step = 0.35
    tr = ep.generate_episode(cfg)
    got = ep.run_episode(ctx_for(cfg), tr, strategy, cfg)
    ref = kre.run_episode(cfg.to_json(), tr.to_jsonl(), strategy)
    assert_report_equal(got, ref)
    assert all(s["wall_ms"] > 0 for s in got["per_step"])


@pytest.mark.parametrize("variant", ["fixed", "overlap", "single-hop", "seq", "k-sweep", "r-sweep"])
def test_episode_ablations_match_reference(kre, variant):
    cfg = base_config(1001)
    cfg.categories[0].update_prob_per_step = 0.5
    cfg.categories[1].update_prob_per_step = 0.35
    if variant == "fixed":
        cfg.grouping = "fixed"
    elif variant == "overlap":
        cfg.balanced_loading = False
    elif variant == "single-hop":
        cfg.multihop = False
    elif variant == "seq":
        cfg.schedule_override = "seq"
    tr = ep.generate_episode(cfg)
    if variant.endswith("sweep"):
        ks, rs = ([4, 8], []) if variant == "k-sweep" else ([], [0.3, 0.75])
        got = ep.compare_csv(ctx_for(cfg), tr, ["keep", "full-reuse"], cfg, ks, rs)
        assert got == kre.compare_csv(cfg.to_json(), tr.to_jsonl(), ["keep", "full-reuse"], ks, rs)
        return
    got = ep.run_episode(ctx_for(cfg), tr, "keep", cfg)
    assert_report_equal(got, kre.run_episode(cfg.to_json(), tr.to_jsonl(), "keep"))


def test_ablation_orderings_hold_on_gpu():
    """test_harness.cpp:255-290 (fewer paired seeds): on update-heavy traces,
    fixed-block grouping costs TTFT and fidelity, and overlap loading is never
    faster than balanced loading."""
    ttft_sem = ttft_fix = div_sem = div_fix = ttft_bal = ttft_ovl = 0.0
    for i in range(6):
        cfg = base_config(1000 + i)
        cfg.categories[0].update_prob_per_step = 0.5
        cfg.categories[1].update_prob_per_step = 0.35
        tr = ep.generate_episode(cfg)
        c = ctx_for(cfg)
        a = ep.run_episode(c, tr, "keep", cfg)["aggregate"]
        ttft_sem += a["mean_ttft_tu"]
        div_sem += a["mean_div_l2"]
        ttft_bal += a["mean_ttft_tu"]
        cfg.grouping = "fixed"
        b = ep.run_episode(c, tr, "keep", cfg)["aggregate"]
        ttft_fix += b["mean_ttft_tu"]
        div_fix += b["mean_div_l2"]
        cfg.grouping = "semantic"
        cfg.balanced_loading = False
        ttft_ovl += ep.run_episode(c, tr, "keep", cfg)["aggregate"]["mean_ttft_tu"]
    assert ttft_fix > ttft_sem and div_fix > div_sem
    assert ttft_ovl >= ttft_bal


def test_episode_at_head_dim_128_runs_the_tensor_core_paths(kre):
    """The same replay at head_dim 128 (the Ozaki / DMMA PARITY kernels and
    the tcgen05 FAST kernels): PARITY reproduces the reference; FAST keeps
    every TTFT / reuse figure (its plans may differ only at near-ties)."""
    cfg = base_config(7, num_segments=16, num_steps=3, k=6, num_heads=2, model_dim=256, mlp_dim=256,
                      vocab_size=256)
    tr = ep.generate_episode(cfg)
    ref = kre.run_episode(cfg.to_json(), tr.to_jsonl(), "keep")
    assert_report_equal(ep.run_episode(ctx_for(cfg), tr, "keep", cfg), ref)
    fast = ep.run_episode(ctx_for(cfg, kb.FAST), tr, "full-reuse", cfg)
    ref_fr = kre.run_episode(cfg.to_json(), tr.to_jsonl(), "full-reuse")
    for g, r in zip(fast["per_step"], ref_fr["per_step"]):
        assert g["ttft_tu"] == r["ttft_tu"] and g["plan_sizes"] == r["plan_sizes"]
        assert abs(g["div_l2"] - r["div_l2"]) <= 3e-2 * max(r["div_l2"], 1.0)
