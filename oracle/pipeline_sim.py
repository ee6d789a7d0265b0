"""Restatement of the reference's loading-schedule model (TEST INFRASTRUCTURE ONLY).

The reference simulates layer-balanced loading instead of performing it
(/root/reference/proj/include/keep/pipeline_sim.hpp).  Its functions are the
specification that the real loader (paper_2602_23592_b200/csrc/loader.cu, K10)
follows, so they are restated here, line for line, as the checker:

  derive_workload        pipeline_sim.hpp:103-154
  preload_eligible_from  pipeline_sim.hpp:169-187
  simulate_sequential    pipeline_sim.hpp:191-212
  simulate_overlap       pipeline_sim.hpp:214-259
  simulate_balanced      pipeline_sim.hpp:261-338
  validate_timeline      pipeline_sim.hpp:340-428 (codes R, D1, D2, P, S)

Pinned against the reference's own fixtures (tests/test_pipeline.cpp) in
tests/test_pipeline_spec.py.  Only tests/ import this module.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Set, Tuple

Owner = Tuple[int, int]  # (kind, id): kind 0 segment, 1 group (OwnerRef, memory_store.hpp:61-88)
INF = float("inf")


@dataclass
class LoadItem:
    layer: int
    owner: Owner
    bytes: int
    tu: float


@dataclass
class Workload:
    num_layers: int
    compute_tu: List[float]
    eval_tu: List[float]
    attention_fraction: float = 0.5
    items: List[LoadItem] = field(default_factory=list)
    owner_members: Dict[Owner, List[int]] = field(default_factory=dict)

    def members_of(self, owner: Owner) -> List[int]:  # pipeline_sim.hpp:61-66
        if owner[0] == 0:
            return [owner[1]]
        return list(self.owner_members.get(owner, []))


@dataclass
class Event:
    kind: str      # "load" | "compute" | "eval"
    resource: str  # "load" | "compute" | "eval"
    layer: int
    owner: Owner = (0, 0)
    bytes: int = 0
    start: float = 0.0
    end: float = 0.0


@dataclass
class Timeline:
    events: List[Event] = field(default_factory=list)
    makespan: float = 0.0


def derive_workload(plan: Sequence[Set[int]], seg_tokens: Dict[int, int], units, query_tokens: int,
                    compute_tu_per_token_per_layer: float, eval_tu_per_layer: float,
                    attention_fraction: float, slow_bw: float, with_eval: bool) -> Workload:
    """units: [(owner, [segment ids], [slow bytes per layer])] (LoadUnit)."""
    L = len(plan)
    w = Workload(L, [0.0] * L, [0.0] * L, attention_fraction)
    for l in range(L):
        tokens = query_tokens + sum(seg_tokens[s] for s in plan[l])
        w.compute_tu[l] = float(tokens) * compute_tu_per_token_per_layer
        if with_eval and l + 1 < L:
            w.eval_tu[l] = eval_tu_per_layer
    for owner, segs, slow_bytes in units:
        if owner[0] == 1:
            w.owner_members[owner] = list(segs)
        for l in range(L):
            if not any(s not in plan[l] for s in segs):
                continue
            b = slow_bytes[l] if l < len(slow_bytes) else 0
            if b == 0:
                continue
            w.items.append(LoadItem(l, owner, b, float(b) / slow_bw))
    w.items.sort(key=lambda it: (it.layer, it.owner))
    return w


def _emit(tl: Timeline, kind, res, layer, start, end, owner=(0, 0), nbytes=0):
    if end <= start:  # zero-duration work leaves no event
        return
    tl.events.append(Event(kind, res, layer, owner, nbytes, start, end))
    tl.makespan = max(tl.makespan, end)


def preload_eligible_from(w: Workload, plan, owner: Owner) -> float:
    members = w.members_of(owner)
    if not members:
        return INF
    frm = 0
    for m in members:
        first = INF
        for l in range(len(plan)):
            if m not in plan[l]:
                first = l
                break
        frm = max(frm, first)
        if frm == INF:
            break
    return frm


def simulate_sequential(w: Workload) -> Timeline:
    tl, t = Timeline(), 0.0
    for l in range(w.num_layers):
        for it in w.items:
            if it.layer != l:
                continue
            _emit(tl, "load", "load", l, t, t + it.tu, it.owner, it.bytes)
            t += it.tu
        if l >= 1 and w.eval_tu[l - 1] > 0.0:
            _emit(tl, "eval", "eval", l - 1, t, t + w.eval_tu[l - 1])
            t += w.eval_tu[l - 1]
        _emit(tl, "compute", "compute", l, t, t + w.compute_tu[l])
        t += w.compute_tu[l]
    tl.makespan = max(tl.makespan, t)
    return tl


def _run(w: Workload, plan=None, balanced=False) -> Timeline:
    tl = Timeline()
    L = w.num_layers
    pending = [[it, preload_eligible_from(w, plan, it.owner) if balanced else INF, False] for it in w.items]
    load_last_end = [0.0] * L
    load_free = eval_free = 0.0
    prev_compute_end = prev_eval_end = 0.0
    for p in pending:  # layer-0 loads happen up front
        if p[0].layer != 0:
            continue
        _emit(tl, "load", "load", 0, load_free, load_free + p[0].tu, p[0].owner, p[0].bytes)
        load_free += p[0].tu
        load_last_end[0] = load_free
        p[2] = True
    for l in range(L):
        c_start = max(prev_compute_end, prev_eval_end, load_last_end[l])
        c_end = c_start + w.compute_tu[l]
        _emit(tl, "compute", "compute", l, c_start, c_end)
        prev_eval_end = 0.0
        if w.eval_tu[l] > 0.0:
            attn_done = c_start + w.attention_fraction * w.compute_tu[l]
            e_start = max(attn_done, eval_free)
            e_end = e_start + w.eval_tu[l]
            _emit(tl, "eval", "eval", l, e_start, e_end)
            eval_free = e_end
            prev_eval_end = e_end
        if l + 1 < L:
            for p in pending:
                if p[2] or p[0].layer != l + 1:
                    continue
                start = max(load_free, c_start)
                _emit(tl, "load", "load", l + 1, start, start + p[0].tu, p[0].owner, p[0].bytes)
                load_free = start + p[0].tu
                load_last_end[l + 1] = load_free
                p[2] = True
        if balanced:
            # fill the idle window until this compute finishes with the first
            # eligible future item in (layer, owner) order; an item that would
            # overrun the window stops the fill (pipeline_sim.hpp:314-333)
            while True:
                nxt = None
                for p in pending:
                    if p[2] or p[0].layer < l + 2:
                        continue
                    if p[1] > l:
                        continue
                    nxt = p
                    break
                if nxt is None:
                    break
                start = max(load_free, c_start)
                end = start + nxt[0].tu
                if end > c_end + 1e-12:
                    break
                _emit(tl, "load", "load", nxt[0].layer, start, end, nxt[0].owner, nxt[0].bytes)
                load_free = end
                nxt[2] = True
        prev_compute_end = c_end
    tl.makespan = max(tl.makespan, prev_compute_end)
    return tl


def simulate_overlap(w: Workload) -> Timeline:
    return _run(w)


def simulate_balanced(w: Workload, plan) -> Timeline:
    return _run(w, plan, balanced=True)


def validate_timeline(tl: Timeline, plan, w: Workload) -> List[Tuple[str, str]]:
    eps = 1e-9
    out = []
    for res in ("load", "compute", "eval"):  # R
        evs = sorted((e for e in tl.events if e.resource == res), key=lambda e: e.start)
        for a, b in zip(evs, evs[1:]):
            if b.start < a.end - eps:
                out.append(("R", f"overlapping events on one resource at layer {b.layer}"))
    compute_at = {e.layer: e for e in tl.events if e.kind == "compute"}
    for layer, comp in compute_at.items():  # D1
        for e in tl.events:
            if e.kind == "load" and e.layer == layer and e.end > comp.start + eps:
                out.append(("D1", f"load for layer {layer} ends after compute starts"))
            if e.kind == "eval" and e.layer == layer - 1 and e.end > comp.start + eps:
                out.append(("D1", f"eval of layer {layer - 1} ends after compute of layer {layer}"))
    for e in tl.events:  # D2
        if e.kind != "eval" or e.layer not in compute_at:
            continue
        c = compute_at[e.layer]
        if e.start < c.start + w.attention_fraction * (c.end - c.start) - eps:
            out.append(("D2", f"eval of layer {e.layer} starts before attention completes"))
    loaded: Dict[Tuple[int, Owner], int] = {}
    for e in tl.events:  # P
        if e.kind == "load" and e.bytes > 0:
            loaded[(e.layer, e.owner)] = loaded.get((e.layer, e.owner), 0) + e.bytes
    wanted: Dict[Tuple[int, Owner], int] = {}
    for it in w.items:
        if it.bytes > 0:
            wanted[(it.layer, it.owner)] = wanted.get((it.layer, it.owner), 0) + it.bytes
    if loaded != wanted:
        out.append(("P", "loaded bytes do not match workload items"))
    for e in tl.events:  # S
        if e.kind != "load":
            continue
        for layer, comp in compute_at.items():
            if e.start >= comp.end - eps or e.end <= comp.start + eps:
                continue
            if e.layer < comp.layer + 2:
                continue
            for m in w.members_of(e.owner):
                if comp.layer < len(plan) and m in plan[comp.layer]:
                    out.append(("S", f"pre-load of {e.owner} while segment {m} is planned at layer {comp.layer}"))
    max_end = max((e.end for e in tl.events), default=0.0)
    if tl.makespan + eps < max_end:
        out.append(("P", "makespan smaller than the last event end"))
    return out
