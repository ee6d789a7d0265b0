"""The memory control plane's host logic (include/keep_episode.h) against the
UNMODIFIED reference harness (oracle/_ref/libkeep_ref_episode.so) -- no GPU.

* generate_episode (harness.hpp:362-413): our traces equal the reference's
  event for event (tokens, embeddings bit-for-bit, query seeds);
* MemoryStore (memory_store.hpp:274-496) driven as run_episode drives it:
  k-means groups, invalidation records, static transitions and versions,
  retrieval sets and state soundness equal the reference's at every step;
* the error taxonomy of the config / trace checks.
"""
import json
import os

import numpy as np
import pytest

import paper_2602_23592_b200 as kb
from paper_2602_23592_b200 import episode as ep


def base_config(seed, num_segments=16, num_steps=6, k=6, **kw):
    """test_harness.cpp:21-45 (base_config)."""
    n4 = num_segments // 4
    cfg = ep.EpisodeConfig(
        seed=seed, num_segments=num_segments, num_steps=num_steps, retrieval_k=k, r_avg=0.5, query_tokens=8,
        embedding_dim=8, fixed_pos_edge_tokens=4, store_t=3, store_num_groups=4, store_seed=seed,
        num_layers=4, num_heads=4, model_dim=32, mlp_dim=64, vocab_size=128, model_seed=seed,
        compute_tu_per_token_per_layer=1.0, eval_tu_per_layer=0.5, attention_fraction=0.5,
        fast_capacity_bytes=32768, fast_bandwidth_bytes_per_tu=8192, slow_to_fast_bandwidth_bytes_per_tu=512,
        categories=[ep.Category("object-state", n4, 8, 0.30), ep.Category("agent-state", n4, 8, 0.20),
                    ep.Category("task-history", n4, 8, 0.02),
                    ep.Category("environment-layout", num_segments - 3 * n4, 8, 0.05)])
    for k_, v in kw.items():
        setattr(cfg, k_, v)
    return cfg


@pytest.fixture(scope="module")
def kre():
    from oracle.episode_oracle import EpisodeOracle, available
    if not available():
        pytest.skip("reference episode shim not built (oracle/_ref/libkeep_ref_episode.so)")
    return EpisodeOracle()


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(kb.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return kb.load_library()


def configs():
    out = [base_config(7), base_config(20250807, 12, 4, 5), base_config(3, 24, 10, 8)]
    heavy = base_config(1003)
    heavy.categories[0].update_prob_per_step = 0.5
    heavy.categories[1].update_prob_per_step = 0.35
    out.append(heavy)
    ones = base_config(5)
    for c in ones.categories:
        c.update_prob_per_step = 1.0
    out.append(ones)
    d = base_config(11, 20, 5, 6)
    d.categories = ep.default_categories(20)
    d.embedding_dim = 16
    out.append(d)
    return out


@pytest.mark.parametrize("i", range(6))
def test_generate_episode_matches_reference(lib, kre, i):
    cfg = configs()[i]
    ref = [json.loads(ln) for ln in kre.generate(cfg.to_json()).splitlines()]
    got = ep.generate_episode(cfg).events()
    assert len(got) == len(ref)
    for a, b in zip(got, ref):
        assert a["type"] == b["type"]
        for key in ("id", "step", "tokens", "embedding_seed", "k", "category"):
            if key in b:
                assert a[key] == b[key], (key, a, b)
        if "embedding" in b:  # doubles round-trip exactly through the JSON text
            assert np.array_equal(np.array(a["embedding"]), np.array(b["embedding"]))


def test_trace_round_trip(lib):
    tr = ep.generate_episode(base_config(7))
    again = ep.Trace.from_jsonl(tr.to_jsonl())
    assert again.events() == tr.events()


@pytest.mark.parametrize("i", range(6))
@pytest.mark.parametrize("grouping", ["semantic", "fixed"])
def test_memory_store_replay_matches_reference(lib, kre, i, grouping):
    cfg = configs()[i]
    cfg.grouping = grouping
    tr = ep.generate_episode(cfg)
    ref = kre.store_replay(cfg.to_json(), tr.to_jsonl())
    events = tr.events()
    segs = [e for e in events if e["type"] == "init-segment"]
    st = ep.MemoryStore(segs, t=cfg.store_t, num_groups=cfg.store_num_groups, seed=cfg.store_seed or cfg.seed,
                        grouping=grouping)

    def groups():
        return [{"members": g["members"], "state": g["state"], "version": g["version"]} for g in st.groups()]

    assert groups() == ref[0]["initial_groups"]
    owner = {0: "s", 1: "g"}
    steps = {}
    for e in events:
        if e["type"] != "init-segment":
            steps.setdefault(e["step"], []).append(e)
    assert len(steps) == len(ref) - 1
    for (step, evs), r in zip(sorted(steps.items()), ref[1:]):
        assert r["step"] == step
        recs = []
        for e in evs:
            if e["type"] == "update":
                rec = st.apply_update(e["id"], e["tokens"], step)
                recs.append({"entries": [[owner[o[0]] + str(o[1]), t] for o, t in rec["entries"]],
                             "new_version": rec["new_segment_version"][1]})
        assert recs == r["updates"]
        assert [list(x) for x in st.advance_step(step)] == r["transitions"]
        for q in r["queries"]:
            units = st.retrieve(q["embedding"], q["k"])
            assert [[owner[o[0]] + str(o[1]), segs_] for o, segs_ in units] == q["units"]
        assert groups() == r["groups"]
        assert st.state_sound() == r["state_sound"]


def test_store_add_segment_joins_nearest_group(lib):
    cfg = base_config(7)
    segs = [e for e in ep.generate_episode(cfg).events() if e["type"] == "init-segment"]
    st = ep.MemoryStore(segs, t=3, num_groups=4, seed=7)
    st.advance_step(5)  # every group static (no updates yet)
    assert all(g["state"] == "static" for g in st.groups())
    new = dict(segs[3], id=100)  # same embedding as segment 3: joins its group, which turns dynamic
    st.add_segment(new, 6)
    g = next(g for g in st.groups() if 100 in g["members"])
    assert 3 in g["members"] and g["state"] == "dynamic"
    assert st.state_sound()
    with pytest.raises(kb.KeepError) as e:
        st.add_segment(new, 7)
    assert e.value.code == kb.CONFIG


def test_config_and_trace_errors(lib):
    bad = base_config(7)
    bad.categories[0].count += 1  # counts no longer sum to num_segments
    with pytest.raises(kb.KeepError) as e:
        ep.generate_episode(bad)
    assert e.value.code == kb.CONFIG
    bad = base_config(7, r_avg=0.1)  # below 1/L
    with pytest.raises(kb.KeepError) as e:
        ep.generate_episode(bad)
    assert e.value.code == kb.CONFIG
    evs = ep.generate_episode(base_config(7)).events()
    with pytest.raises(kb.KeepError) as e:
        ep.Trace.from_events(evs + [evs[0]])  # duplicate init-segment id
    assert e.value.code == kb.TRACE
    q = [x for x in evs if x["type"] == "query"]
    with pytest.raises(kb.KeepError) as e:
        ep.Trace.from_events(evs + [dict(q[0], step=0)])  # steps decrease
    assert e.value.code == kb.TRACE
    with pytest.raises(kb.KeepError) as e:
        ep.Trace.from_events(evs + [{"type": "update", "step": 99, "id": 999, "tokens": [1]}])
    assert e.value.code == kb.TRACE
    segs = [x for x in evs if x["type"] == "init-segment"]
    with pytest.raises(kb.KeepError) as e:
        ep.MemoryStore([dict(segs[0], embedding=[1.0, 1.0])], t=3, num_groups=1)  # not unit norm
    assert e.value.code == kb.CONFIG
    with pytest.raises(kb.KeepError) as e:
        ep.MemoryStore(segs[:2], t=3, num_groups=3)  # more groups than segments
    assert e.value.code == kb.CONFIG


def test_run_episode_needs_a_context(lib):
    cfg = base_config(7)
    tr = ep.generate_episode(cfg)

    class NoCtx:
        _h = None

    with pytest.raises(kb.KeepError) as e:
        ep.run_episode(NoCtx(), tr, "keep", cfg)
    assert e.value.code == kb.CONFIG
