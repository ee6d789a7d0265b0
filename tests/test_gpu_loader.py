"""K10: memory KV resident in pinned host DRAM, loaded layer by layer into the
merged KV (loader.cu).  The prefill must be identical to the HBM-resident
run (PARITY: bit-exact plans, walk orders, hops and hidden states), and the
realised load schedule must satisfy the reference's timeline rules
(pipeline_sim.hpp:340-428):
  P   every workload item (layer l, owner with a member outside plan[l]) is
      loaded exactly once, with its whole block (derive_workload, 103-154);
  D1  the batch carrying an item of layer l completes before compute(l);
  S   a pre-load (item of layer >= l+2 issued behind compute(l)) only touches
      owners whose members all left the plan by layer l."""
import numpy as np
import pytest

import paper_2602_23592_b200 as kb

pytestmark = pytest.mark.gpu

EPS_MS = 1e-3


def problem(ko, c):
    p = ko.make_instance(c["seed"], c["S"], c["L"], c["H"], c["d"], c["mlp"], c["V"], c["lo"], c["hi"], c["qlen"])
    p.units = [tuple(u) for u in c["units"]]
    return p


def layout_of(p):
    units = []
    for u, (b, e, g) in enumerate(p.units):
        if g:
            units.append((b, e, kb.GROUP, u))
        else:
            units += [(i, i + 1, kb.SEGMENT, i) for i in range(b, e)]
    return kb.Layout(p.seg_len, p.tokens, units)


def check_schedule(trace, plan, lay, d, elem):
    L, S = plan.shape
    owners = lay.owners()
    tokens = {(k, o): int(np.sum(lay.seg_len[b:e])) for k, o, b, e in owners}
    members = {(k, o): list(range(b, e)) for k, o, b, e in owners}
    want = {(l, own) for l in range(L) for own, ms in members.items() if any(not plan[l, m] for m in ms)}
    got = [(r["layer"], r["owner"]) for r in trace]
    assert len(got) == len(set(got)), "an item was loaded twice"
    assert set(got) == want, (sorted(want - set(got))[:5], sorted(set(got) - want)[:5])  # P
    for r in trace:
        own = r["owner"]
        assert r["bytes"] == 2 * tokens[own] * d * elem  # whole block, K + V
        assert r["end_ms"] <= r["compute_start_ms"] + EPS_MS, r  # D1
        if r["kind"] == "preload":  # S
            assert r["layer"] >= r["at_layer"] + 2
            assert all(not plan[r["at_layer"], m] for m in members[own]), r


@pytest.mark.parametrize("idx", [0, 7, 21, 40, 56])
def test_host_memory_parity(ko, golden, idx):
    if idx >= len(golden["instances"]):
        pytest.skip("fewer golden instances")
    c = golden["instances"][idx]
    p = problem(ko, c)
    lay = layout_of(p)
    sched = np.array(c["sched"])
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ref = ko.plan_keep(p, w, sched)
    with kb.Context(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"]) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1, tier=kb.TIER_DEVICE)
        dev = ctx.plan_keep(lay, p.query, sched)
        ctx.memory_compute_layout(lay, version=2, tier=kb.TIER_HOST)
        st0 = ctx.memory_stats()
        host = ctx.plan_keep(lay, p.query, sched)
        trace = ctx.loader_trace()
        st1 = ctx.memory_stats()
    assert np.array_equal(host["plan"], ref["plan"]) and host["orders"] == ref["orders"]
    assert np.array_equal(host["hops"], ref["hops"])
    assert np.array_equal(host["final_hidden"], dev["final_hidden"])  # same arithmetic, other tier
    assert np.array_equal(host["last_logits"], dev["last_logits"])
    check_schedule(trace, host["plan"], lay, c["d"], 4)
    assert st1["bytes_loaded_slow"] - st0["bytes_loaded_slow"] == sum(r["bytes"] for r in trace)


def test_host_memory_fast_tc():
    # head_dim 128, tensor-core attention; preloads exercised by a deep plan
    seed, S, L, H, d, mlp, V = 71, 60, 6, 2, 256, 512, 512
    from paper_2602_23592_b200.synth import group_units, make_instance_layout
    inst = make_instance_layout(seed, S, V)
    lay = kb.Layout(inst.seg_len, inst.tokens, group_units(S, 4, 0.5))
    sched = kb.ratio_schedule(L, 0.3)
    with kb.Context(L, H, d, mlp, V, seed, kb.FAST) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1)
        dev = ctx.plan_keep(lay, inst.query, sched)
        ctx.memory_compute_layout(lay, version=2, tier=kb.TIER_HOST)
        host = ctx.plan_keep(lay, inst.query, sched)
        trace = ctx.loader_trace()
    assert np.array_equal(host["plan"], dev["plan"])
    assert np.max(np.abs(host["final_hidden"] - dev["final_hidden"])) <= 1e-3 * np.max(np.abs(dev["final_hidden"]))
    check_schedule(trace, host["plan"], lay, d, 2)
    assert len(trace) > 0


def test_inplace_refresh(ko, golden):
    """An update refreshes owners in place (no new arena): the blocks, the
    versions and the prefill stay exactly as a fresh computation's."""
    c = golden["instances"][11]
    p = problem(ko, c)
    lay = layout_of(p)
    sched = np.array(c["sched"])
    w = ko.model_init(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"])
    ref = ko.plan_keep(p, w, sched)
    owners = lay.owners()
    pick = list(range(0, len(owners), 2))
    with kb.Context(c["L"], c["H"], c["d"], c["mlp"], c["V"], c["seed"]) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1)
        before = {u: ctx.memory_read(owners[u][0], owners[u][1], 1, int(np.sum(lay.seg_len[owners[u][2]:owners[u][3]])))
                  for u in range(len(owners))}
        dev0 = ctx.memory_stats()["device_bytes"]
        ctx.memory_refresh(lay, pick, version=2)
        assert ctx.memory_stats()["device_bytes"] == dev0  # refreshed in place
        for u, (kind, oid, b, e) in enumerate(owners):
            assert ctx.has_current(kind, oid, 2 if u in pick else 1)
            k, v = ctx.memory_read(kind, oid, 1, int(np.sum(lay.seg_len[b:e])))
            assert np.array_equal(k, before[u][0]) and np.array_equal(v, before[u][1])
        got = ctx.plan_keep(lay, p.query, sched)
    assert np.array_equal(got["plan"], ref["plan"]) and got["orders"] == ref["orders"]


def validate_real_timeline(kr, ctx, lay, plan, qlen, block_bytes):
    """The reference's own validate_timeline over the device's timeline."""
    evs, frac = ctx.timeline_trace()
    L = plan.shape[0]
    units = [(b, e, int(k == kb.GROUP), o) for k, o, b, e in lay.owners()]
    slow = np.array([[block_bytes(b, e)] * L for b, e, _, _ in units], np.uint64)
    return kr.validate_timeline(plan, lay.seg_len, qlen, units, slow, frac, evs), evs, frac, units, slow


@pytest.mark.parametrize("numerics", [kb.PARITY, kb.FAST])
def test_reference_validate_timeline_on_device_trace(kr, numerics):
    """pipeline_sim.hpp:340-428 (R, D1, D2, P, S) run by the unmodified
    reference on the realised copy / compute / selector-stream timeline."""
    seed, S, L, H, d, mlp, V = 71, 60, 6, 2, 256, 512, 512
    from paper_2602_23592_b200.synth import group_units, make_instance_layout
    inst = make_instance_layout(seed, S, V)
    lay = kb.Layout(inst.seg_len, inst.tokens, group_units(S, 4, 0.5))
    sched = kb.ratio_schedule(L, 0.3)
    elem = 2 if numerics == kb.FAST else 4
    with kb.Context(L, H, d, mlp, V, seed, numerics) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1, tier=kb.TIER_HOST)
        res = ctx.plan_keep(lay, inst.query, sched)
        bb = lambda b, e: 2 * int(np.sum(lay.seg_len[b:e])) * d * elem  # noqa: E731
        codes, evs, frac, units, slow = validate_real_timeline(kr, ctx, lay, res["plan"], len(inst.query), bb)
    assert codes == [], codes
    kinds = {e["kind"] for e in evs}
    assert kinds == {0, 1, 2} and 0.0 < frac <= 1.0
    # fault injection (test_pipeline.cpp:276-335): the same checker flags broken timelines
    comp = {e["layer"]: e for e in evs if e["kind"] == 1}
    load = next(e for e in evs if e["kind"] == 0 and e["layer"] > 0)
    late = [dict(e) for e in evs]
    for e in late:
        if e is not None and e["kind"] == 0 and e["layer"] == load["layer"] and e["owner"] == load["owner"]:
            e["end"] = comp[load["layer"]]["start"] + 1.0
    assert "D1" in kr.validate_timeline(res["plan"], lay.seg_len, len(inst.query), units, slow, frac, late)
    dup = evs + [dict(load)]
    assert "P" in kr.validate_timeline(res["plan"], lay.seg_len, len(inst.query), units, slow, frac, dup)


@pytest.mark.parametrize("idx,frac", [(7, 0.5), (40, 0.25), (56, 1.0)])
def test_hbm_residency_budget(ko, golden, idx, frac):
    """keep_memory_residency: the deepest layers of the pinned-host memory
    stay in HBM (the capacity-bounded fast tier, cache_manager.hpp:23-35).
    The prefill is bit-identical, no item of a resident layer is loaded, every
    other workload item still is (rule P over the slow layers), and a write
    to the memory drops the HBM copy."""
    if idx >= len(golden["instances"]):
        pytest.skip("fewer golden instances")
    c = golden["instances"][idx]
    p = problem(ko, c)
    lay = layout_of(p)
    sched = np.array(c["sched"])
    L = c["L"]
    with kb.Context(L, c["H"], c["d"], c["mlp"], c["V"], c["seed"]) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1, tier=kb.TIER_HOST)
        full = ctx.plan_keep(lay, p.query, sched)
        per_layer = 2 * int(np.sum(lay.seg_len)) * c["d"] * 4 + 2 * 128 * c["d"] * 4  # (arena pad rows)
        m = int(frac * L)
        got = ctx.memory_residency(m * per_layer + per_layer // 2)
        assert got == m * per_layer
        res = ctx.plan_keep(lay, p.query, sched)
        trace = ctx.loader_trace()
        assert np.array_equal(res["final_hidden"], full["final_hidden"])
        assert np.array_equal(res["plan"], full["plan"]) and res["orders"] == full["orders"]
        assert all(r["layer"] < L - m for r in trace)
        owners = lay.owners()
        members = {(k, o): list(range(b, e)) for k, o, b, e in owners}
        want = {(l, own) for l in range(L - m) for own, ms in members.items() if any(not res["plan"][l, mm] for mm in ms)}
        assert {(r["layer"], r["owner"]) for r in trace} == want
        # a write to the memory drops the HBM copy; results stay identical
        ctx.memory_compute_layout(lay, version=2, tier=kb.TIER_HOST)
        again = ctx.plan_keep(lay, p.query, sched)
        assert np.array_equal(again["final_hidden"], full["final_hidden"])
        assert ctx.memory_residency(0) == 0


@pytest.mark.parametrize("numerics", [kb.PARITY, kb.FAST])
def test_split_host_arena_chunked(ko, numerics, monkeypatch):
    """A pinned-host memory created under an HBM budget: computed in owner
    chunks (KEEP_HOST_CHUNK_ROWS forces them at test size) into ONE in-order
    arena whose deepest layers live in HBM only.  plan_keep and the batched
    prefill over it equal the HBM-resident runs bit for bit; resident layers
    are never loaded."""
    from paper_2602_23592_b200.synth import group_units, make_instance_layout
    seed, S, L, H, d, V = 23, 40, 6, 2, 256, 512
    inst = make_instance_layout(seed, S, V)
    lay = kb.Layout(inst.seg_len, inst.tokens, group_units(S, 4, 0.5))
    sched = kb.ratio_schedule(L, 0.4)
    rng = np.random.default_rng(seed)
    Q = rng.integers(0, V, size=(3, len(inst.query))).astype(np.int32)
    Q[0] = inst.query
    elem = 4 if numerics == kb.PARITY else 2
    per_layer = 2 * (int(np.sum(inst.seg_len)) + 128) * d * elem
    with kb.Context(L, H, d, 2 * d, V, seed, numerics) as ctx:
        ctx.model_init()
        ctx.memory_compute_layout(lay, version=1, tier=kb.TIER_DEVICE)
        dev = ctx.plan_keep(lay, Q[0], sched)
        devb = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
    with kb.Context(L, H, d, 2 * d, V, seed, numerics) as ctx:
        ctx.model_init()
        assert ctx.memory_residency(2 * per_layer + 10) == 0  # (no host memory yet: the budget is for new arenas)
        monkeypatch.setenv("KEEP_HOST_CHUNK_ROWS", "97")
        ctx.memory_compute_layout(lay, version=1, tier=kb.TIER_HOST)
        monkeypatch.delenv("KEEP_HOST_CHUNK_ROWS")
        st = ctx.memory_stats()
        assert st["device_bytes"] >= 2 * per_layer and st["host_bytes"] == (L - 2) * per_layer
        host = ctx.plan_keep(lay, Q[0], sched)
        trace = ctx.loader_trace()
        hostb = ctx.plan_keep_batch(lay, Q, sched, final_hidden=True)
    assert all(r["layer"] < L - 2 for r in trace)
    assert np.array_equal(host["plan"], dev["plan"]) and host["orders"] == dev["orders"]

    def same(a, b):
        if numerics == kb.PARITY:  # the chunks' canonical KV is bit-identical (row-local arithmetic)
            return np.array_equal(a, b)
        # FAST: the chunks' bf16 GEMMs tile / split K differently from one pass
        return float(np.max(np.abs(a - b))) <= 3e-2 * float(np.max(np.abs(b)))

    assert same(host["final_hidden"], dev["final_hidden"])
    for a, b in zip(hostb, devb):
        assert np.array_equal(a["plan"], b["plan"])
        assert same(a["final_hidden"], b["final_hidden"])
