"""Batched multi-query prefill (keep_plan_keep_batch): B
planning queries over one memory layout.  Every query of the batch gets
exactly what a lone plan_keep gives it -- plans, walk orders, hops, rows per
layer, summaries and (PARITY) bit-identical final hidden states and logits --
although layer 0's memory rows are computed once for the whole batch, the
projections run once per layer over all queries' rows, and all-reused layers
read the in-order arena in place.  plan_keep itself is pinned to the
reference oracle by test_gpu_parity.py."""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb
from paper_2602_23592_b200.synth import group_units, make_instance_layout

pytestmark = pytest.mark.gpu


def batch_queries(seed, B, qlen, V, first):
    rng = np.random.default_rng(seed)
    Q = rng.integers(0, V, size=(B, qlen)).astype(np.int32)
    Q[0] = first
    return Q


def layout(inst, S, groups):
    if groups:
        return kb.Layout(inst.seg_len, inst.tokens, group_units(S, 4, 0.5))
    return kb.Layout(inst.seg_len, inst.tokens)


@pytest.mark.parametrize("seed,S,L,H,d,B,groups,r_avg", [
    (5, 16, 4, 4, 32, 3, False, 0.5), (6, 40, 5, 2, 64, 5, True, 0.4), (7, 12, 3, 2, 32, 1, False, 0.5),
    (8, 60, 6, 4, 64, 4, True, 0.3),
])
def test_batch_parity_matches_single(seed, S, L, H, d, B, groups, r_avg):
    mlp, V = 2 * d, 256
    inst = make_instance_layout(seed, S, V)
    lay = layout(inst, S, groups)
    Q = batch_queries(seed, B, len(inst.query), V, inst.query)
    sched = kb.ratio_schedule(L, r_avg)
    with kb.Context(L, H, d, mlp, V, seed) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        batch = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True, summaries=True)
        singles = [ctx.plan_keep(lay, Q[b], sched, summaries=True) for b in range(B)]
        again = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)  # workspace reuse
    for b, (g, r) in enumerate(zip(batch, singles)):
        assert np.array_equal(g["plan"], r["plan"]), b
        assert g["orders"] == r["orders"], b
        assert np.array_equal(g["hops"], r["hops"]), b
        assert np.array_equal(g["rows_per_layer"], r["rows_per_layer"]), b
        assert np.array_equal(g["qts"], r["qts"]) and np.array_equal(g["sts"], r["sts"]), b
        assert np.array_equal(g["final_hidden"], r["final_hidden"]), b
        assert np.array_equal(g["last_logits"], r["last_logits"]), b
        assert np.array_equal(again[b]["final_hidden"], r["final_hidden"]), b
    assert len({round(g["ttft_ms"], 9) for g in batch}) == 1  # one device time for the batch


@pytest.mark.parametrize("seed,S,L,H,d,B,groups,r_avg", [
    (5, 16, 4, 4, 32, 3, False, 0.5), (8, 60, 6, 4, 64, 4, True, 0.3), (9, 48, 3, 2, 256, 3, True, 0.5),
    (10, 120, 3, 1, 128, 4, True, 0.4),
])
def test_batch_parity_matches_oracle(ko, seed, S, L, H, d, B, groups, r_avg):
    """Every query of a PARITY batch against the CPU oracle's own plan_keep
    (recompute.hpp:140-180) on that query: selections bit-exact, summaries
    within the fp64 summation-order tolerance, hidden states within 2e-6
    (head_dim 128 rows: the Ozaki / DMMA kernels with the fused bins)."""
    from oracle.oracle import Problem
    mlp, V = 2 * d, 256
    inst = make_instance_layout(seed, S, V)
    lay = layout(inst, S, groups)
    units = [(u[0], u[1], 1 if u[2] == kb.GROUP else 0) for u in lay.units] if groups else []
    Q = batch_queries(seed + 100, B, len(inst.query), V, inst.query)
    sched = kb.ratio_schedule(L, r_avg)
    with kb.Context(L, H, d, mlp, V, seed) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        batch = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True, summaries=True)
    w = ko.model_init(L, H, d, mlp, V, seed)
    for b in range(B):
        ref = ko.plan_keep(Problem(L, H, d, mlp, V, seed, inst.seg_len, inst.tokens, Q[b], units), w, sched)
        g = batch[b]
        assert np.array_equal(g["plan"], ref["plan"]), b
        assert g["orders"] == ref["orders"] and np.array_equal(g["hops"], ref["hops"]), b
        assert float(np.max(np.abs(g["qts"] - ref["qts"]))) <= 1e-12, b
        assert float(np.max(np.abs(g["sts"] - ref["sts"]))) <= 1e-12, b
        scale = float(np.max(np.abs(ref["final_hidden"])))
        assert float(np.max(np.abs(g["final_hidden"].astype(np.float64) - ref["final_hidden"]))) <= 2e-6 * scale, b


def test_batch_fast_tc_matches_single():
    # head_dim 128: tensor-core attention, decode kernel on the query-only layers
    seed, S, L, H, d, V, B = 31, 50, 6, 2, 256, 512, 4
    inst = make_instance_layout(seed, S, V)
    lay = layout(inst, S, True)
    Q = batch_queries(seed, B, len(inst.query), V, inst.query)
    sched = kb.ratio_schedule(L, 0.3)
    with kb.Context(L, H, d, 2 * d, V, seed, kb.FAST) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        batch = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
        singles = [ctx.plan_keep(lay, Q[b], sched) for b in range(B)]
    agree = np.mean([np.mean(g["plan"] == r["plan"]) for g, r in zip(batch, singles)])
    assert agree >= 0.95
    for g, r in zip(batch, singles):
        if np.array_equal(g["plan"], r["plan"]):
            q = slice(-len(inst.query), None)
            a, e = g["final_hidden"][q].astype(np.float64), r["final_hidden"][q].astype(np.float64)
            assert np.max(np.abs(a - e)) <= 3e-2 * np.max(np.abs(e))


def test_batch_host_memory_matches_hbm():
    """Memory in pinned host DRAM (BASELINE configs[4]): the batch streams one
    layer sheet per layer over PCIe for all queries (staged one layer ahead)
    and computes exactly what it computes over HBM-resident memory --
    walks, and (given plans) all-reused layers on the staged sheet."""
    seed, S, L, H, d, V, B = 21, 30, 5, 2, 64, 256, 4
    inst = make_instance_layout(seed, S, V)
    lay = layout(inst, S, True)
    Q = batch_queries(seed, B, len(inst.query), V, inst.query)
    sched = kb.ratio_schedule(L, 0.4)
    plans = np.zeros((B, L, S), np.uint8)
    plans[:, 0] = 1
    plans[1, 1:3, :7] = 1
    plans[2, 1] = 1
    with kb.Context(L, H, d, 2 * d, V, seed) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1)
        dev = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
        dev_sel = ctx.plan_keep_batch(lay, Q, None, final_hidden=True, plans=plans)
        ctx.memory_compute_layout(lay, version=2, tier=kb.TIER_HOST)
        st0 = ctx.memory_stats()
        host = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
        st1 = ctx.memory_stats()
        host_sel = ctx.plan_keep_batch(lay, Q, None, final_hidden=True, plans=plans)
        with pytest.raises(kb.KeepError):
            ctx.plan_keep_batch(lay, np.zeros((2, 0), np.int32), sched)
    for g, r in list(zip(host, dev)) + list(zip(host_sel, dev_sel)):
        assert np.array_equal(g["plan"], r["plan"]) and g["orders"] == r["orders"]
        assert np.array_equal(g["final_hidden"], r["final_hidden"])
        assert np.array_equal(g["last_logits"], r["last_logits"])
    Tm = int(np.sum(inst.seg_len))
    # every layer after the first crosses PCIe once for the whole batch
    assert st1["bytes_loaded_slow"] - st0["bytes_loaded_slow"] == (L - 1) * 2 * Tm * d * 4


@pytest.mark.parametrize("mode", [kb.PARITY, kb.FAST])
def test_batch_selective_prefill_alias_layers(mode):
    """Given plans (keep_selective_prefill_batch): queries whose later layers
    reuse all memory run those layers on the in-order arena (their query rows
    copied into its spare rows one query at a time), the others on their own
    merged KV; each equals the cursor's selective_prefill of its plan."""
    seed, S, L, V, B = 12, 24, 5, 256, 4
    H, d = (4, 32) if mode == kb.PARITY else (2, 256)
    inst = make_instance_layout(seed, S, V)
    lay = kb.Layout(inst.seg_len, inst.tokens)
    Q = batch_queries(seed, B, len(inst.query), V, inst.query)
    plans = np.zeros((B, L, S), np.uint8)
    plans[:, 0] = 1
    plans[0, 1] = 1                  # everything, then nothing
    plans[1, 1:3, :5] = 1            # a prefix for two layers
    plans[2] = 1                     # full recompute
    plans[3, 1, ::3] = 1             # scattered, then nothing
    with kb.Context(L, H, d, 2 * d, V, seed, mode) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        batch = ctx.plan_keep_batch(lay, Q, None, final_hidden=True, summaries=True, plans=plans)
        refs = [ctx.selective_prefill(lay, Q[b], plans[b]) for b in range(B)]
        with pytest.raises(kb.KeepError):  # not monotone
            bad = plans.copy()
            bad[0, 3, 0] = 1
            ctx.plan_keep_batch(lay, Q, None, plans=bad)
    for b in range(B):
        g, r = batch[b], refs[b]
        assert np.array_equal(g["plan"], plans[b])
        if mode == kb.PARITY:
            assert np.array_equal(g["final_hidden"], r["final_hidden"]), b
            assert np.array_equal(g["qts"], r["qts"]) and np.array_equal(g["sts"], r["sts"]), b
        else:
            q = slice(-len(inst.query), None)
            a, e = g["final_hidden"][q].astype(np.float64), r["final_hidden"][q].astype(np.float64)
            assert np.max(np.abs(a - e)) <= 3e-2 * np.max(np.abs(e)), b


@pytest.mark.parametrize("B,qlen,multihop", [(1, 1, True), (3, 1, False), (20, 5, True)])
def test_batch_edges(B, qlen, multihop):
    """One query, one-token queries, the single-hop ablation
    (recompute.hpp:166-176) and more queries than one logits launch covers."""
    seed, S, L, H, d, V = 44, 14, 4, 2, 32, 128
    inst = make_instance_layout(seed, S, V, qlen=qlen)
    lay = kb.Layout(inst.seg_len, inst.tokens)
    Q = batch_queries(seed, B, qlen, V, inst.query)
    sched = kb.ratio_schedule(L, 0.5)
    with kb.Context(L, H, d, 2 * d, V, seed) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        batch = ctx.plan_keep_batch(lay, Q, sched, multihop=multihop, final_hidden=True)
        singles = [ctx.plan_keep(lay, Q[b], sched, multihop=multihop) for b in range(B)]
    for g, r in zip(batch, singles):
        assert np.array_equal(g["plan"], r["plan"]) and g["orders"] == r["orders"]
        assert np.array_equal(g["final_hidden"], r["final_hidden"])
        assert np.array_equal(g["last_logits"], r["last_logits"])


def test_trim_releases_and_regrows_workspaces():
    """keep_ctx_trim frees the prefill / batch / refresh workspaces; the next
    calls regrow them and compute the same results."""
    seed, S, L, H, d, V, B = 9, 18, 4, 2, 64, 256, 3
    inst = make_instance_layout(seed, S, V)
    lay = kb.Layout(inst.seg_len, inst.tokens)
    Q = batch_queries(seed, B, len(inst.query), V, inst.query)
    sched = kb.ratio_schedule(L, 0.5)
    with kb.Context(L, H, d, 2 * d, V, seed) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        a = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
        s1 = ctx.plan_keep(lay, Q[1], sched)
        ctx.trim()
        with pytest.raises(kb.KeepError):  # no prefill in progress after a trim
            ctx.prefill_layer(np.ones(S, np.uint8))
        b = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
        s2 = ctx.plan_keep(lay, Q[1], sched)
    for x, y in zip(a, b):
        assert np.array_equal(x["plan"], y["plan"]) and np.array_equal(x["final_hidden"], y["final_hidden"])
    assert np.array_equal(s1["final_hidden"], s2["final_hidden"])
