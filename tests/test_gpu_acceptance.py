"""The reference's acceptance-level properties, on the device (PARITY):
  - divergence non-increasing along nested plans, 20 pinned seeds
    (test_prefill.cpp:309-330);
  - oracle degeneracy: keep at r_avg 1 is the full prefill
    (acceptance.cpp:39-58);
  - sandwich: div(full) = 0 <= div(keep@0.5) <= div(full reuse), 21 pinned
    seeds (acceptance.cpp:63-79);
  - multi-hop beats single-hop on the chain-structured seeds {2, 6, 8, 15}
    (test_harness.cpp:296-308).
The strategies run as run_strategy does (recompute.hpp:313-334):
selective_prefill of the plan through the cursor, then divergence of the
last row against the full prefill."""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import make_instance_layout

pytestmark = pytest.mark.gpu

L, H, D, MLP, V = 4, 4, 32, 64, 128
SANDWICH_SEEDS = [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 22, 23]


def setup(seed, S, lo=8, hi=12, qlen=8):
    inst = make_instance_layout(seed, S, V, lo, hi, qlen)
    lay = kb.Layout(inst.seg_len, inst.tokens)
    ctx = kb.Context(L, H, D, MLP, V, seed)
    ctx.model_init()
    ctx.memory_compute_layout(lay)  # per-segment canonical KV (segment_prefill)
    full = ctx.selective_prefill(lay, inst.query, np.ones((L, S), np.uint8))["final_hidden"]
    return inst, lay, ctx, full


def div(ctx, lay, query, plan, full):
    fh = ctx.selective_prefill(lay, query, np.asarray(plan, np.uint8))["final_hidden"]
    return ctx.divergence(fh[-1], full[-1]), fh


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 8, 10, 11, 12, 15, 17, 19, 20, 22, 23, 24, 25, 26, 27, 29])
def test_divergence_monotone_along_nested_plans(seed):
    S = 6
    inst, lay, ctx, full = setup(seed, S, 6, 9, 6)
    with ctx:
        prev = 1e300
        for n in range(S + 1):
            plan = np.zeros((L, S), np.uint8)
            plan[:, :n] = 1
            (l2, _), _ = div(ctx, lay, inst.query, plan, full)
            assert l2 <= prev + 1e-9, (seed, n, l2, prev)
            prev = l2
        assert prev <= 1e-6


@pytest.mark.parametrize("seed", SANDWICH_SEEDS)
def test_oracle_degeneracy_and_sandwich(seed):
    S = 8
    inst, lay, ctx, full = setup(seed, S)
    with ctx:
        keep1 = ctx.plan_keep(lay, inst.query, kb.ratio_schedule(L, 1.0))
        assert np.max(np.abs(keep1["final_hidden"] - full)) <= 1e-6
        (l2_full, kl_full), _ = div(ctx, lay, inst.query, np.ones((L, S)), full)
        keep = ctx.plan_keep(lay, inst.query, kb.ratio_schedule(L, 0.5))
        (l2_keep, _), _ = div(ctx, lay, inst.query, keep["plan"], full)
        (l2_reuse, _), _ = div(ctx, lay, inst.query, np.zeros((L, S)), full)
    assert l2_full == 0.0 and kl_full == 0.0
    assert l2_keep <= l2_reuse, (seed, l2_keep, l2_reuse)


@pytest.mark.parametrize("seed", [2, 6, 8, 15])
def test_multihop_beats_single_hop(seed):
    S = 8
    inst, lay, ctx, full = setup(seed, S)
    sched = kb.ratio_schedule(L, 0.5)
    with ctx:
        multi = ctx.plan_keep(lay, inst.query, sched, multihop=True)
        single = ctx.plan_keep(lay, inst.query, sched, multihop=False)
        (l2_m, _), _ = div(ctx, lay, inst.query, multi["plan"], full)
        (l2_s, _), _ = div(ctx, lay, inst.query, single["plan"], full)
    assert l2_m < l2_s, (seed, l2_m, l2_s)
