"""The loading-schedule specification the K10 loader follows (oracle/pipeline_sim.py,
a restatement of pipeline_sim.hpp), pinned against the reference's own fixtures
(tests/test_pipeline.cpp) and fault injections; plus the online rule the real
loader applies, checked on random monotone plans: every item it issues is a
workload item, each exactly once, pre-loads only of fully-out owners (S)."""
import numpy as np
import pytest

from oracle.pipeline_sim import (LoadItem, Workload, simulate_balanced, simulate_overlap, simulate_sequential,
                                 validate_timeline)

PLAN = [{3}, set(), set()]  # kFixturePlan: owners 1, 2 never recomputed, 3 only at layer 0


def fixture(compute, items, plan=PLAN):
    w = Workload(len(compute), list(compute), [0.0] * len(compute), 0.5)
    for layer, owner, tu in items:
        w.items.append(LoadItem(layer, (0, owner), int(tu * 1024), tu))
    return w, plan


def valid(w, plan, tl):
    return validate_timeline(tl, plan, w) == []


def test_hand_fixture_1():  # test_pipeline.cpp:98-106
    w, plan = fixture([4, 4, 4], [(1, 1, 2.0), (2, 2, 3.0)])
    assert simulate_sequential(w).makespan == pytest.approx(17.0)
    assert simulate_overlap(w).makespan == pytest.approx(12.0)
    assert simulate_balanced(w, plan).makespan == pytest.approx(12.0)
    for tl in (simulate_sequential(w), simulate_overlap(w), simulate_balanced(w, plan)):
        assert valid(w, plan, tl)


def test_hand_fixture_2_balanced_preload():  # test_pipeline.cpp:108-133
    w, plan = fixture([4, 4, 4], [(1, 1, 2.0), (2, 2, 2.0), (2, 3, 4.0)])
    assert simulate_sequential(w).makespan == pytest.approx(20.0)  # (SPEC.md:516 says 19; the code says 20)
    assert simulate_overlap(w).makespan == pytest.approx(14.0)
    tl = simulate_balanced(w, plan)
    assert tl.makespan == pytest.approx(12.0)
    pre = [e for e in tl.events if e.kind == "load" and e.layer == 2 and e.end <= 4.0 + 1e-9]
    assert len(pre) == 1 and pre[0].owner == (0, 2) and pre[0].start == pytest.approx(2.0)
    for t in (simulate_sequential(w), simulate_overlap(w), tl):
        assert valid(w, plan, t)


def test_zero_loads():  # test_pipeline.cpp:135-140
    w, plan = fixture([4, 4, 4], [])
    assert simulate_sequential(w).makespan == simulate_overlap(w).makespan == simulate_balanced(w, plan).makespan == 12


def test_eval_dependencies():  # test_pipeline.cpp:257-274
    w, plan = fixture([4, 4, 4], [(1, 1, 2.0), (2, 2, 3.0)])
    w.eval_tu = [1.0, 1.0, 0.0]
    assert simulate_sequential(w).makespan == pytest.approx(19.0)
    ovl = simulate_overlap(w)
    assert valid(w, plan, ovl) and valid(w, plan, simulate_sequential(w))
    ev = [e for e in ovl.events if e.kind == "eval" and e.layer == 0]
    assert ev and ev[0].start == pytest.approx(2.0)


def test_validator_flags_corruption():  # test_pipeline.cpp:276-335
    w, plan = fixture([4, 4, 4], [(1, 1, 2.0), (2, 2, 2.0), (2, 3, 4.0)])

    def codes(tl):
        return {c for c, _ in validate_timeline(tl, plan, w)}

    tl = simulate_overlap(w)
    for e in tl.events:
        if e.kind == "compute" and e.layer == 2:
            e.start -= 3.0
    assert "D1" in codes(tl)
    tl = simulate_overlap(w)
    for e in tl.events:
        if e.kind == "load" and e.layer == 2 and e.owner == (0, 3):
            e.start -= 1.5
    assert "R" in codes(tl)
    tl = simulate_overlap(w)
    tl.events = [e for e in tl.events if e.kind != "load"]
    assert "P" in codes(tl)
    tl = simulate_balanced(w, plan)
    for e in tl.events:
        if e.kind == "load" and e.owner == (0, 3):
            e.start, e.end = 2.0, 4.0
    assert "S" in codes(tl)
    w.eval_tu = [1.0, 1.0, 0.0]
    tl = simulate_overlap(w)
    for e in tl.events:
        if e.kind == "eval" and e.layer == 0:
            e.start -= 1.5
    assert "D2" in codes(tl)


def online_schedule(plan, owners):
    """The K10 loader's issue rule (loader.cu), replayed on the host: returns
    (layer, owner, kind, at_layer) in issue order."""
    L = len(plan)
    loaded, out_from, issued = set(), {}, []
    for l in range(L):
        for o, ms in owners.items():  # urgent: needed at l, not loaded yet
            if any(m not in plan[l] for m in ms) and (l, o) not in loaded:
                loaded.add((l, o))
                issued.append((l, o, "urgent", l))
        if l + 1 >= L:
            continue
        for o, ms in sorted(owners.items()):
            if all(m not in plan[l] for m in ms):
                out_from.setdefault(o, l)
            if any(m not in plan[l] for m in ms) and (l + 1, o) not in loaded:
                loaded.add((l + 1, o))
                issued.append((l + 1, o, "ahead", l))
        for l2 in range(l + 2, L):  # (unbounded window: every eligible pre-load)
            for o in sorted(owners):
                if out_from.get(o, L) <= l and (l2, o) not in loaded:
                    loaded.add((l2, o))
                    issued.append((l2, o, "preload", l))
    return issued


@pytest.mark.parametrize("seed", range(40))
def test_online_loader_rule_issues_exactly_the_workload(seed):
    rng = np.random.default_rng(seed)
    L, S = int(rng.integers(1, 8)), int(rng.integers(1, 10))
    plan, live = [], set(range(S))
    for l in range(L):
        live = {s for s in live if (l == 0 and rng.random() < 0.8) or (l > 0 and rng.random() < 0.7)}
        plan.append(set(live))
    # owners: consecutive runs, some groups
    owners, i = {}, 0
    while i < S:
        j = min(S, i + int(rng.integers(1, 4)))
        owners[(1, i) if j - i > 1 else (0, i)] = list(range(i, j))
        i = j
    issued = online_schedule(plan, owners)
    items = [(l, o) for l, o, _, _ in issued]
    want = {(l, o) for l in range(L) for o, ms in owners.items() if any(m not in plan[l] for m in ms)}
    assert len(items) == len(set(items)) and set(items) == want  # P
    for l, o, kind, at in issued:
        if kind == "preload":  # S
            assert l >= at + 2 and all(m not in plan[at] for m in owners[o])
        if kind == "ahead":  # monotone plans: an owner out at `at` is needed at at + 1
            assert l == at + 1 and any(m not in plan[at] for m in owners[o])
