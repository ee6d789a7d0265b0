"""GPU parity of the CUDA path against the CPU oracle (runs on a B200).

PARITY numerics: selections (plans, walk orders, hop counts) must be
bit-exact with the reference on every golden instance; device weights and
layer-0 KV are bit-exact; hidden states / merged KV / summaries within the
fp64-reordering tolerance stated below (the only differences are fp64
summation order and exp ulps inside attention).
"""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

# fp32 outputs: relative tolerance on max-normalised differences
HIDDEN_RTOL = 2e-6
# fp64 summaries: summation order only (the Q.K^T and P.V products run on the
# fp64 tensor cores in their own order; every rounding step of the softmax is
# the reference's: s = dot * scale, s - max, e * (1/sum), p * (1/H)).
SUMMARY_ATOL = 1e-12
SUMMARY_RTOL = 0.0


def summary_close(got, ref):
    """per layer: |got - ref| <= atol + rtol * max|ref of that layer|"""
    got, ref = np.asarray(got), np.asarray(ref)
    for l in range(ref.shape[0]):
        tol = SUMMARY_ATOL + SUMMARY_RTOL * float(np.max(np.abs(ref[l])))
        if float(np.max(np.abs(got[l] - ref[l]))) > tol:
            return False
    return True


def problem(ko, c):
    p = ko.make_instance(c["seed"], c["S"], c["L"], c["H"], c["d"], c["mlp"], c["V"], c["lo"], c["hi"], c["qlen"])
    p.units = [tuple(u) for u in c["units"]]
    return p


def layout_of(p):
    units = []
    for u, (b, e, g) in enumerate(p.units):
        units.append((b, e, kb.GROUP if g else kb.SEGMENT, u if g else b))
        if not g and e - b > 1:  # dynamic unit of several segments: one owner per segment
            units.pop()
            units += [(i, i + 1, kb.SEGMENT, i) for i in range(b, e)]
    return kb.Layout(p.seg_len, p.tokens, units)


def rel(a, b):
    scale = max(float(np.max(np.abs(b))), 1e-30)
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)))) / scale


@pytest.fixture(scope="module")
def ctx_cache():
    cache = {}
    yield cache
    for c in cache.values():
        c.close()


def gpu_ctx(cache, c, numerics=kb.PARITY):
    key = (c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"], numerics)
    if key not in cache:
        cache[key] = kb.Context(*key[:6], numerics=numerics).model_init()
    return cache[key]


def test_weights_bit_exact(ko, golden, ctx_cache):
    for c in golden["weights"]:
        L, H, d, mlp, V, seed = c["cfg"]
        with kb.Context(L, H, d, mlp, V, seed) as ctx:
            w = ctx.model_init().export_weights()
        assert np.array_equal(w, ko.model_init(L, H, d, mlp, V, seed))


def test_selector_known_answers(golden, ctx_cache):
    ctx = gpu_ctx(ctx_cache, golden["instances"][0])
    for c in golden["converge"]:
        order, hops = ctx.importance_evaluation(c["qts"], c["sts"], c["budget"], c.get("candidates"))
        assert (order, hops) == (c["order"], c["hops"]), c["name"]


def test_selector_random_large(ko, ctx_cache, golden):
    ctx = gpu_ctx(ctx_cache, golden["instances"][0])
    rng = np.random.default_rng(5)
    for S in [1, 2, 33, 700, 1025, 3000]:
        qts = rng.random(S) * (rng.random(S) > 0.3)
        sts = np.tril(rng.random((S, S)) * (rng.random((S, S)) > 0.5) / S, -1)
        # exact ties: quantised values
        if S > 100:
            sts = np.round(sts * 64) / 64
        cand = (rng.random(S) > 0.2).astype(np.uint8)
        for budget in [1, max(1, S // 3), S]:
            assert ctx.importance_evaluation(qts, sts, budget, cand) == ko.converge(qts, sts, budget, cand), (S, budget)


def test_canonical_kv(ko, golden, ctx_cache):
    for c in golden["instances"][:12] + golden["instances"][-12:]:
        p = problem(ko, c)
        w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
        ref = ko.canonical_kv(p, w)
        ctx = gpu_ctx(ctx_cache, c)
        lay = layout_of(p)
        ctx.memory_compute_layout(lay, version=1)
        starts = np.concatenate([[0], np.cumsum(p.seg_len)])
        for kind, oid, b, e in lay.owners():
            n = int(starts[e] - starts[b])
            for l in range(c["L"]):
                k, v = ctx.memory_read(kind, oid, l, n)
                rk, rv = ref[l, 0, starts[b]:starts[e]], ref[l, 1, starts[b]:starts[e]]
                if l == 0:  # embedding-only KV: bit-exact (prefill.hpp / test_prefill.cpp:175-195)
                    assert np.array_equal(k, rk) and np.array_equal(v, rv)
                else:
                    assert rel(k, rk) <= HIDDEN_RTOL and rel(v, rv) <= HIDDEN_RTOL


@pytest.mark.parametrize("mode", [kb.PARITY, kb.PARITY_EXACT], ids=["parity", "exact"])
@pytest.mark.parametrize("idx", range(57))
def test_plan_keep_parity(ko, golden, ctx_cache, idx, mode):
    if idx >= len(golden["instances"]):
        pytest.skip("fewer golden instances")
    c = golden["instances"][idx]
    p = problem(ko, c)
    ctx = gpu_ctx(ctx_cache, c, mode)
    lay = layout_of(p)
    ctx.memory_compute_layout(lay, version=1)
    got = ctx.plan_keep(lay, p.query, np.array(c["sched"]), multihop=c["multihop"], summaries=True)
    tag = (c["seed"], c["S"], c["r_avg"], c["multihop"])
    # selections: bit-exact
    assert got["plan"].tolist() == c["plan"], tag
    assert got["orders"] == c["orders"], tag
    assert got["hops"].tolist() == c["hops"], tag
    # summaries: fp64, summation order only
    assert summary_close(got["qts"], np.array(c["qts"])), tag
    assert summary_close(got["sts"], np.array(c["sts"])), tag
    # last row vs the golden, whole final hidden vs the oracle
    assert rel(got["final_hidden"][-1], np.array(c["last_row"], np.float32)) <= HIDDEN_RTOL, tag
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ref = ko.plan_keep(p, w, np.array(c["sched"]), multihop=c["multihop"])
    assert rel(got["final_hidden"], ref["final_hidden"]) <= HIDDEN_RTOL, tag
    # first-token logits (model.hpp:76-85): fp64 over the final row
    lg = ko.logits(p, w, got["final_hidden"][-1])
    assert np.allclose(got["last_logits"], lg, rtol=1e-12, atol=1e-12), tag


def test_selective_prefill_plans(ko, golden, ctx_cache):
    """selective_prefill with fixed plans (full, reuse-all, prefix, drop after 0)."""
    c = next(x for x in golden["instances"] if x["seed"] == 18 and x["r_avg"] == 0.5)
    p = problem(ko, c)
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ctx = gpu_ctx(ctx_cache, c)
    lay = layout_of(p)
    ctx.memory_compute_layout(lay, version=1)
    cached = ko.canonical_kv(p, w)
    L, S = c["L"], c["S"]
    plans = {
        "full": np.ones((L, S), np.uint8),
        "reuse": np.zeros((L, S), np.uint8),
        "prefix2": np.tile((np.arange(S) < 2).astype(np.uint8), (L, 1)),
        "drop_after_0": np.vstack([np.ones(S, np.uint8)] + [(np.arange(S) < 2).astype(np.uint8)] * (L - 1)),
        # all memory reused after layer 1: those layers run on the arena sheets (no merged-KV copy)
        "empty_after_1": np.vstack([np.ones((2, S), np.uint8), np.zeros((L - 2, S), np.uint8)]),
    }
    for name, plan in plans.items():
        got = ctx.selective_prefill(lay, p.query, plan)
        ref = ko.selective_prefill(p, w, plan, cached=cached)
        assert rel(got["final_hidden"], ref["final_hidden"]) <= HIDDEN_RTOL, name
        assert rel(got["kv"], ref["kv"]) <= HIDDEN_RTOL, name
        assert summary_close(got["sts"], ref["sts"]), name
        assert summary_close(got["qts"], ref["qts"]), name
        # merged KV takes the (device) cached rows verbatim (test_prefill.cpp:273-287)
        starts = np.concatenate([[0], np.cumsum(p.seg_len)])
        for l in range(L):
            for i in range(S):
                if plan[l, i]:
                    continue
                k, v = ctx.memory_read(kb.SEGMENT, i, l, int(p.seg_len[i]))
                assert np.array_equal(got["kv"][l][0][starts[i]:starts[i + 1]], k), (name, l, i)
                assert np.array_equal(got["kv"][l][1][starts[i]:starts[i + 1]], v), (name, l, i)


def test_errors(ko, golden, ctx_cache):
    c = golden["instances"][0]
    p = problem(ko, c)
    ctx = gpu_ctx(ctx_cache, c)
    lay = layout_of(p)
    L, S = c["L"], c["S"]
    ctx.invalidate(kb.SEGMENT, 1, 5)
    ctx.memory_compute_layout(lay, version=1)
    # owner s1 is now stale (current version 5 > 1): reuse of segment 1 misses
    ctx.prefill_begin(lay, p.query)
    with pytest.raises(kb.KeepError) as ei:
        ctx.prefill_layer(np.zeros(S, np.uint8))
    assert ei.value.kind == "CacheMissError"
    # non-monotone plan
    ctx.prefill_begin(lay, p.query)
    a = np.ones(S, np.uint8)
    a[0] = 0
    ctx.prefill_layer(a)
    with pytest.raises(kb.KeepError) as ei:
        ctx.prefill_layer(np.ones(S, np.uint8))
    assert ei.value.kind == "PlanError"
    # stepping past the last layer / finishing early
    ctx.prefill_begin(lay, p.query)
    with pytest.raises(kb.KeepError) as ei:
        ctx.prefill_finish()
    assert ei.value.kind == "PlanError"
    # token out of vocabulary
    bad = kb.Layout(p.seg_len, np.where(np.arange(len(p.tokens)) == 0, c["V"] + 3, p.tokens))
    with pytest.raises(kb.KeepError) as ei:
        ctx.prefill_begin(bad, p.query)
    assert ei.value.kind == "InputError"
    # load_memory surface: miss, stale, hit
    with pytest.raises(kb.KeepError) as ei:
        ctx.load_memory(kb.SEGMENT, 1, 0)
    assert ei.value.kind == "CacheMissError"
    v = ctx.load_memory(kb.SEGMENT, 0, 1)
    assert v.tokens == p.seg_len[0] and v.keys and v.values
    assert ctx.has_current(kb.SEGMENT, 0, 1) and not ctx.has_current(kb.SEGMENT, 1, 1)


def test_host_tier_load(ko, golden, ctx_cache):
    c = golden["instances"][0]
    p = problem(ko, c)
    ctx = gpu_ctx(ctx_cache, c)
    lay = layout_of(p)
    ctx.memory_compute_layout(lay, version=3, tier=kb.TIER_HOST)
    st0 = ctx.memory_stats()
    v = ctx.load_memory(kb.SEGMENT, 2, 1)
    assert v.tier == kb.TIER_HOST and v.load_ms >= 0
    st1 = ctx.memory_stats()
    assert st1["bytes_loaded_slow"] > st0["bytes_loaded_slow"]
    v2 = ctx.load_memory(kb.SEGMENT, 2, 1)  # promoted: now a fast hit
    assert v2.tier == kb.TIER_DEVICE
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ref = ko.canonical_kv(p, w)
    starts = np.concatenate([[0], np.cumsum(p.seg_len)])
    k, _ = ctx.memory_read(kb.SEGMENT, 2, 1, int(p.seg_len[2]))
    assert rel(k, ref[1, 0, starts[2]:starts[3]]) <= HIDDEN_RTOL


def test_host_tier_load_async(ko, golden, ctx_cache):
    """keep_load_memory_async: the promotion copy is only enqueued; after the
    completion event the HBM block equals the canonical KV."""
    c = golden["instances"][1]
    p = problem(ko, c)
    ctx = gpu_ctx(ctx_cache, c)
    lay = layout_of(p)
    ctx.memory_compute_layout(lay, version=4, tier=kb.TIER_HOST)
    owner = (kb.SEGMENT, 3) if (kb.SEGMENT, 3) in [(o[0], o[1]) for o in lay.owners()] else lay.owners()[-1][:2]
    v, ev = ctx.load_memory_async(owner[0], owner[1], 0)
    assert ev and v.tier == kb.TIER_HOST and v.load_ms < 0
    ctx.load_wait()
    assert ctx.load_memory(owner[0], owner[1], 0).tier == kb.TIER_DEVICE  # promoted
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ref = ko.canonical_kv(p, w)
    starts = np.concatenate([[0], np.cumsum(p.seg_len)])
    b, e = [(o[2], o[3]) for o in lay.owners() if (o[0], o[1]) == tuple(owner)][0]
    n = int(starts[e] - starts[b])
    k, vv = ctx.memory_read(owner[0], owner[1], 0, n)
    assert rel(k, ref[0, 0, starts[b]:starts[e]]) <= HIDDEN_RTOL
    assert rel(vv, ref[0, 1, starts[b]:starts[e]]) <= HIDDEN_RTOL


def test_determinism(ko, golden, ctx_cache):
    c = golden["instances"][-3]
    p = problem(ko, c)
    ctx = gpu_ctx(ctx_cache, c)
    lay = layout_of(p)
    ctx.memory_compute_layout(lay)
    a = ctx.plan_keep(lay, p.query, np.array(c["sched"]), summaries=True)
    b = ctx.plan_keep(lay, p.query, np.array(c["sched"]), summaries=True)
    assert np.array_equal(a["final_hidden"], b["final_hidden"])
    assert np.array_equal(a["sts"], b["sts"]) and np.array_equal(a["plan"], b["plan"])


def test_divergence_matches_reference(ko, golden, ctx_cache):
    """divergence (prefill.hpp:501-531) on the device against the reference's
    values for the golden instances (keep vs full prefill, last row)."""
    checked = 0
    for c in golden["instances"][::4]:
        p = problem(ko, c)
        w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
        res = ko.plan_keep(p, w, np.array(c["sched"]), multihop=c["multihop"])
        full = ko.full_prefill(p, w, kv=False)
        ctx = gpu_ctx(ctx_cache, c)
        l2, kl = ctx.divergence(res["final_hidden"][-1], full["final_hidden"][-1])
        for got, want in ((l2, c["div_l2"]), (kl, c["div_kl"])):
            if np.isnan(want):
                assert np.isnan(got)
            else:
                assert abs(got - want) <= 1e-9 * max(1.0, abs(want)), (c["seed"], got, want)
        checked += 1
    assert checked >= 10
