"""KV-head sharding on one B200: G logical ranks, one host
thread each, exchanging through the loopback collectives (the same
run_layer code path the NCCL communicator drives across GPUs).

PARITY: plans, walk orders and hop counts of every rank are bit-exact with the
reference; hidden states within the fp64-reordering tolerance; each rank's KV
is its head-column slice of the reference merged KV.  FAST: the sharded path
agrees with the single-GPU FAST path to the FAST tolerance."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

HIDDEN_RTOL = 2e-6
RTOL_FAST = 3e-2


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)))) / max(float(np.max(np.abs(b))), 1e-30)


def run_sharded(G, cfg, numerics, body):
    """body(ctx) on G ranks concurrently; returns the per-rank results."""
    L, H, d, mlp, V, seed = cfg
    grp = kb.LoopbackGroup(G)
    ctxs = [kb.Context(L, H, d, mlp, V, seed, numerics, world=G, rank=r, loopback=grp) for r in range(G)]
    try:
        with ThreadPoolExecutor(G) as ex:
            return list(ex.map(body, ctxs))
    finally:
        for c in ctxs:
            c.close()
        grp.close()


def problem(ko, c):
    p = ko.make_instance(c["seed"], c["S"], c["L"], c["H"], c["d"], c["mlp"], c["V"], c["lo"], c["hi"], c["qlen"])
    return p


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("idx", [0, 5, 11, 20, 40, 56])
def test_sharded_parity_plan_keep(ko, golden, G, idx):
    if idx >= len(golden["instances"]):
        pytest.skip("fewer golden instances")
    c = golden["instances"][idx]
    if c["H"] % G:
        pytest.skip("heads do not divide")
    p = problem(ko, c)
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    sched = np.array(c["sched"])
    ref = ko.plan_keep(p, w, sched, kv=True)
    lay = kb.Layout(p.seg_len, p.tokens)

    def body(ctx):
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        res = ctx.plan_keep(lay, p.query, sched)
        sel = ctx.selective_prefill(lay, p.query, res["plan"])
        return res, sel["final_hidden"], sel["kv"]

    out = run_sharded(G, (c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"]), kb.PARITY, body)
    dl = c["d"] // G
    for r, (res, fh, kv) in enumerate(out):
        assert np.array_equal(res["plan"], ref["plan"]), (r, res["plan"].sum(1), ref["plan"].sum(1))
        assert res["orders"] == ref["orders"] and np.array_equal(res["hops"], ref["hops"])
        assert rel(res["final_hidden"], ref["final_hidden"]) <= HIDDEN_RTOL
        assert rel(fh, ref["final_hidden"]) <= HIDDEN_RTOL
        assert rel(kv, ref["kv"][..., r * dl:(r + 1) * dl]) <= HIDDEN_RTOL


def test_sharded_summaries_identical_across_ranks(ko, golden):
    c = golden["instances"][3]
    p = problem(ko, c)
    lay = kb.Layout(p.seg_len, p.tokens)
    S = c["S"]

    def body(ctx):
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        ctx.prefill_begin(lay, p.query)
        return [ctx.prefill_layer(np.ones(S, np.uint8)) for _ in range(c["L"])]

    out = run_sharded(4, (c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"]), kb.PARITY, body)
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ref = ko.selective_prefill(p, w, np.ones((c["L"], S), np.uint8))
    for l in range(c["L"]):
        for r in range(1, 4):  # identical bits on every rank: converge runs replicated
            assert np.array_equal(out[r][l][0], out[0][l][0]) and np.array_equal(out[r][l][1], out[0][l][1])
        assert np.max(np.abs(out[0][l][0] - ref["qts"][l])) <= 1e-12
        assert np.max(np.abs(out[0][l][1] - ref["sts"][l])) <= 1e-12


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_fast_matches_single_gpu(ko, G):
    # head_dim 128: the tcgen05 attention on each rank's head slice
    seed, S, L, H, d, mlp, V = 61, 40, 3, 4, 512, 1024, 700
    p = ko.make_instance(seed, S, L, H, d, mlp, V)
    w = ko.model_init(L, H, d, mlp, V, seed)
    sched = ko.ratio_schedule(L, 0.5)
    ref = ko.plan_keep(p, w, sched, kv=True)
    lay = kb.Layout(p.seg_len, p.tokens)
    with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as one:
        one.model_init()
        one.memory_compute_layout(lay)
        single = one.selective_prefill(lay, p.query, ref["plan"])

    def body(ctx):
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        return ctx.selective_prefill(lay, p.query, ref["plan"]), ctx.plan_keep(lay, p.query, sched)

    out = run_sharded(G, (L, H, d, mlp, V, seed), kb.FAST, body)
    dl = d // G
    for r, (sel, pk) in enumerate(out):
        assert rel(sel["final_hidden"], ref["final_hidden"]) <= RTOL_FAST
        assert rel(sel["final_hidden"], single["final_hidden"]) <= RTOL_FAST
        assert rel(sel["kv"], ref["kv"][..., r * dl:(r + 1) * dl]) <= RTOL_FAST
        assert rel(sel["sts"], single["sts"]) <= 1e-2
        assert np.array_equal(pk["plan"], out[0][1]["plan"])  # replicated selection


@pytest.mark.parametrize("G", [2, 4])
def test_sharded_few_row_layers_split_weights(ko, G):
    """Layers of <= 32 rows split the Wo / MLP weights across the ranks
    (row- / column-parallel, fixed-order fp64 all-reduces): a plan that keeps
    only the query from layer 1 on runs every later layer that way.  Hidden
    states within the fp64 re-ordering tolerance of the oracle, identical on
    every rank."""
    seed, S, L, H, d, mlp, V = 91, 12, 5, 4, 256, 512, 300
    p = ko.make_instance(seed, S, L, H, d, mlp, V)
    w = ko.model_init(L, H, d, mlp, V, seed)
    plan = np.zeros((L, S), np.uint8)
    plan[0] = 1
    ref = ko.selective_prefill(p, w, plan)
    lay = kb.Layout(p.seg_len, p.tokens)

    def body(ctx):
        ctx.model_init()
        ctx.memory_compute_layout(lay)
        return ctx.selective_prefill(lay, p.query, plan)["final_hidden"]

    outs = run_sharded(G, (L, H, d, mlp, V, seed), kb.PARITY, body)
    for o in outs:
        assert np.array_equal(o, outs[0])
        assert rel(o[-len(p.query):], ref["final_hidden"][-len(p.query):]) <= HIDDEN_RTOL
