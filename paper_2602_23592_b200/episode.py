"""Memory control plane + episode replay -- Python mirror of
the reference harness over ``include/keep_episode.h``.

    EpisodeConfig, default_categories  harness.hpp:38-113
    generate_episode                   harness.hpp:362-413   (keep_trace_generate)
    trace_to_jsonl / trace_from_jsonl  harness.hpp:297-322
    MemoryStore                        memory_store.hpp:274-496 (keep_store_*)
    run_episode                        harness.hpp:543-817   (keep_run_episode)
    compare_csv                        harness.hpp:828-871   (keep_compare_csv)

The replay runs in the C++ library: canonical KV refreshes, plan_keep, the
selective and full prefills and the divergence on the GPU; the store, the
tier accounting and the pipeline time model on the host.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import KeepError, _check, _p, keep_owner, load_library

STRATEGIES = ("full", "prefix", "full-reuse", "fixed-pos", "deviation", "keep")
SCHEDULES = {None: -1, "seq": 0, "overlap": 1, "balanced": 2}
INIT_SEGMENT, UPDATE, QUERY = 0, 1, 2


class keep_category(C.Structure):
    _fields_ = [("name", C.c_char_p), ("count", C.c_int32), ("tokens_per_segment", C.c_int32),
                ("update_prob_per_step", C.c_double)]


class keep_episode_config(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("num_segments", C.c_int32), ("num_steps", C.c_int32),
                ("retrieval_k", C.c_int32), ("r_avg", C.c_double), ("query_tokens", C.c_int32),
                ("embedding_dim", C.c_int32), ("fixed_pos_edge_tokens", C.c_int32), ("store_t", C.c_int32),
                ("store_num_groups", C.c_int32), ("store_seed", C.c_uint64), ("num_layers", C.c_int32),
                ("num_heads", C.c_int32), ("model_dim", C.c_int32), ("mlp_dim", C.c_int32),
                ("vocab_size", C.c_int32), ("model_seed", C.c_uint64),
                ("compute_tu_per_token_per_layer", C.c_double), ("eval_tu_per_layer", C.c_double),
                ("attention_fraction", C.c_double), ("fast_capacity_bytes", C.c_uint64),
                ("fast_bandwidth_bytes_per_tu", C.c_uint64), ("slow_to_fast_bandwidth_bytes_per_tu", C.c_uint64),
                ("n_categories", C.c_int32), ("categories", C.POINTER(keep_category)), ("grouping", C.c_int32),
                ("multihop", C.c_int32), ("balanced_loading", C.c_int32), ("schedule_override", C.c_int32)]


class keep_trace_event(C.Structure):
    _fields_ = [("type", C.c_int32), ("step", C.c_int64), ("id", C.c_uint32), ("category", C.c_char_p),
                ("n_tokens", C.c_int32), ("tokens", C.POINTER(C.c_int32)), ("embedding_dim", C.c_int32),
                ("embedding", C.POINTER(C.c_double)), ("embedding_seed", C.c_uint64), ("k", C.c_int32)]


class keep_segment(C.Structure):
    _fields_ = [("id", C.c_uint32), ("category", C.c_char_p), ("n_tokens", C.c_int32),
                ("tokens", C.POINTER(C.c_int32)), ("embedding_dim", C.c_int32), ("embedding", C.POINTER(C.c_double))]


class keep_store_config(C.Structure):
    _fields_ = [("t", C.c_int32), ("num_groups", C.c_int32), ("seed", C.c_uint64), ("grouping", C.c_int32)]


class keep_step_report(C.Structure):
    _fields_ = [("step", C.c_int64), ("realized_segments", C.c_int64), ("ttft_tu", C.c_double),
                ("makespan_tu", C.c_double), ("refresh_tu", C.c_double), ("div_l2", C.c_double),
                ("div_kl", C.c_double), ("reused_tokens", C.c_double), ("recomputed_tokens", C.c_double),
                ("memory_tokens", C.c_double), ("invalidated_tokens_delta", C.c_uint64),
                ("bytes_loaded_slow_delta", C.c_uint64), ("num_layers", C.c_int32),
                ("plan_sizes", C.POINTER(C.c_int64)), ("wall_ms", C.c_double)]


class keep_strategy_aggregate(C.Structure):
    _fields_ = [("steps", C.c_int32), ("mean_ttft_tu", C.c_double), ("p95_ttft_tu", C.c_double),
                ("mean_div_l2", C.c_double), ("mean_div_kl", C.c_double), ("reuse_ratio", C.c_double),
                ("mean_realized_segments", C.c_double), ("invalidated_tokens", C.c_uint64),
                ("bytes_slow", C.c_uint64)]


_bound = False


def _lib():
    global _bound
    lib = load_library()
    if _bound:
        return lib
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    cfgp, evp = C.POINTER(keep_episode_config), C.POINTER(keep_trace_event)
    sig = {
        "keep_trace_generate": [cfgp, C.POINTER(vp)],
        "keep_trace_create": [i32, evp, C.POINTER(vp)],
        "keep_trace_size": [vp, C.POINTER(i32)],
        "keep_trace_event_get": [vp, i32, evp],
        "keep_trace_destroy": [vp],
        "keep_store_create": [i32, C.POINTER(keep_segment), C.POINTER(keep_store_config), C.POINTER(vp)],
        "keep_store_destroy": [vp],
        "keep_store_groups": [vp, C.POINTER(i32), i32, C.POINTER(C.c_uint32), C.POINTER(i32), C.POINTER(i32),
                              C.POINTER(u64)],
        "keep_store_apply_update": [vp, C.c_uint32, i32, C.POINTER(i32), i64, i32, C.POINTER(keep_owner),
                                    C.POINTER(u64), C.POINTER(i32), C.POINTER(u64)],
        "keep_store_advance_step": [vp, i64, i32, C.POINTER(C.c_uint32), C.POINTER(u64), C.POINTER(i32)],
        "keep_store_retrieve": [vp, C.POINTER(C.c_double), i32, i32, i32, C.POINTER(keep_owner), C.POINTER(i32),
                                i32, C.POINTER(C.c_uint32), C.POINTER(i32)],
        "keep_store_add_segment": [vp, C.POINTER(keep_segment), i64],
        "keep_store_state_sound": [vp, C.POINTER(i32)],
        "keep_run_episode": [vp, vp, C.c_char_p, cfgp, C.POINTER(vp)],
        "keep_report_aggregate": [vp, C.POINTER(keep_strategy_aggregate)],
        "keep_report_step": [vp, i32, C.POINTER(keep_step_report)],
        "keep_report_json": [vp, C.c_char_p, u64, C.POINTER(u64)],
        "keep_report_destroy": [vp],
        "keep_compare_csv": [vp, vp, i32, C.POINTER(C.c_char_p), cfgp, i32, C.POINTER(i32), i32,
                             C.POINTER(C.c_double), C.c_char_p, u64, C.POINTER(u64)],
        "keep_memory_clear": [vp],
        "keep_ctx_dims": [vp, C.POINTER(i32)],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.restype = C.c_int
        f.argtypes = args
    _bound = True
    return lib


@dataclass
class Category:
    name: str
    count: int = 0
    tokens_per_segment: int = 8
    update_prob_per_step: float = 0.0


def default_categories(num_segments: int) -> List[Category]:
    """harness.hpp:97-113: four categories with different update rates."""
    cats = [Category("object-state", 0, 8, 0.30), Category("agent-state", 0, 8, 0.20),
            Category("task-history", 0, 8, 0.02), Category("environment-layout", 0, 8, 0.05)]
    base, rest = num_segments // 4, num_segments - 4 * (num_segments // 4)
    for c in cats:
        c.count = base + (1 if rest > 0 else 0)
        rest -= 1 if rest > 0 else 0
    return cats


@dataclass
class EpisodeConfig:
    """EpisodeConfig (harness.hpp:53-104); model fields = the context's."""
    seed: int = 0
    num_segments: int = 0
    num_steps: int = 1
    retrieval_k: int = 1
    r_avg: float = 0.5
    query_tokens: int = 8
    embedding_dim: int = 16
    fixed_pos_edge_tokens: int = 4
    store_t: int = 10
    store_num_groups: int = 1
    store_seed: int = 0
    num_layers: int = 4
    num_heads: int = 4
    model_dim: int = 32
    mlp_dim: int = 64
    vocab_size: int = 128
    model_seed: int = 0
    compute_tu_per_token_per_layer: float = 1.0
    eval_tu_per_layer: float = 0.0
    attention_fraction: float = 0.5
    fast_capacity_bytes: int = 0
    fast_bandwidth_bytes_per_tu: int = 0
    slow_to_fast_bandwidth_bytes_per_tu: int = 0
    categories: List[Category] = field(default_factory=list)
    grouping: str = "semantic"
    multihop: bool = True
    balanced_loading: bool = True
    schedule_override: Optional[str] = None

    def c_struct(self):
        cats = (keep_category * max(1, len(self.categories)))()
        names = [c.name.encode() for c in self.categories]
        for i, c in enumerate(self.categories):
            cats[i] = keep_category(names[i], c.count, c.tokens_per_segment, c.update_prob_per_step)
        s = keep_episode_config(
            self.seed, self.num_segments, self.num_steps, self.retrieval_k, self.r_avg, self.query_tokens,
            self.embedding_dim, self.fixed_pos_edge_tokens, self.store_t, self.store_num_groups, self.store_seed,
            self.num_layers, self.num_heads, self.model_dim, self.mlp_dim, self.vocab_size, self.model_seed,
            self.compute_tu_per_token_per_layer, self.eval_tu_per_layer, self.attention_fraction,
            self.fast_capacity_bytes, self.fast_bandwidth_bytes_per_tu, self.slow_to_fast_bandwidth_bytes_per_tu,
            len(self.categories), cats, 1 if self.grouping == "fixed" else 0, int(bool(self.multihop)),
            int(bool(self.balanced_loading)), SCHEDULES[self.schedule_override])
        return s, (cats, names)  # keep the buffers alive with the struct

    def to_json(self) -> str:
        """The reference's config JSON (config_to_json, harness.hpp:131-170)."""
        j = {"seed": self.seed, "num_segments": self.num_segments, "num_steps": self.num_steps,
             "retrieval_k": self.retrieval_k, "r_avg": self.r_avg, "query_tokens": self.query_tokens,
             "embedding_dim": self.embedding_dim, "fixed_pos_edge_tokens": self.fixed_pos_edge_tokens,
             "store": {"t": self.store_t, "num_groups": self.store_num_groups, "seed": self.store_seed or self.seed},
             "model": {"num_layers": self.num_layers, "num_heads": self.num_heads, "model_dim": self.model_dim,
                       "mlp_dim": self.mlp_dim, "vocab_size": self.vocab_size, "seed": self.model_seed},
             "cost": {"compute_tu_per_token_per_layer": self.compute_tu_per_token_per_layer,
                      "eval_tu_per_layer": self.eval_tu_per_layer, "attention_fraction": self.attention_fraction},
             "tier": {"fast_capacity_bytes": self.fast_capacity_bytes,
                      "fast_bandwidth_bytes_per_tu": self.fast_bandwidth_bytes_per_tu,
                      "slow_to_fast_bandwidth_bytes_per_tu": self.slow_to_fast_bandwidth_bytes_per_tu},
             "categories": [{"name": c.name, "count": c.count, "tokens_per_segment": c.tokens_per_segment,
                             "update_prob_per_step": c.update_prob_per_step} for c in self.categories],
             "ablation": {"grouping": self.grouping, "multihop": bool(self.multihop),
                          "balanced_loading": bool(self.balanced_loading)}}
        if self.schedule_override:
            j["schedule_override"] = self.schedule_override
        return json.dumps(j)


class Trace:
    """A replayable episode trace (TraceEvent list, harness.hpp:117-127)."""

    def __init__(self, handle):
        self._h = handle
        self.lib = _lib()

    def __del__(self):
        try:
            if self._h:
                self.lib.keep_trace_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def __len__(self):
        n = C.c_int32()
        _check(self.lib.keep_trace_size(self._h, C.byref(n)))
        return n.value

    def events(self) -> List[dict]:
        out = []
        for i in range(len(self)):
            e = keep_trace_event()
            _check(self.lib.keep_trace_event_get(self._h, i, C.byref(e)))
            if e.type == INIT_SEGMENT:
                out.append({"type": "init-segment", "id": e.id, "category": e.category.decode(),
                            "tokens": [e.tokens[k] for k in range(e.n_tokens)],
                            "embedding": [e.embedding[k] for k in range(e.embedding_dim)]})
            elif e.type == UPDATE:
                out.append({"type": "update", "step": e.step, "id": e.id,
                            "tokens": [e.tokens[k] for k in range(e.n_tokens)]})
            else:
                out.append({"type": "query", "step": e.step, "embedding_seed": e.embedding_seed, "k": e.k})
        return out

    def to_jsonl(self) -> str:
        """trace_to_jsonl (harness.hpp:297-304): one JSON event per line."""
        return "".join(json.dumps(e) + "\n" for e in self.events())

    @classmethod
    def from_events(cls, events: Sequence[dict]) -> "Trace":
        """trace_from_jsonl's checks (harness.hpp:306-322) over parsed events."""
        lib = _lib()
        n = len(events)
        arr = (keep_trace_event * max(n, 1))()
        keep = []
        types = {"init-segment": INIT_SEGMENT, "update": UPDATE, "query": QUERY}
        for i, e in enumerate(events):
            if e["type"] not in types:
                raise KeepError(5, f"unknown trace event type '{e['type']}'")
            t = types[e["type"]]
            toks = np.ascontiguousarray(e.get("tokens", []), np.int32)
            emb = np.ascontiguousarray(e.get("embedding", []), np.float64)
            cat = e.get("category", "").encode()
            keep += [toks, emb, cat]
            arr[i] = keep_trace_event(t, int(e.get("step", 0)), int(e.get("id", 0)), cat, len(toks),
                                      _p(toks, C.c_int32), len(emb), _p(emb, C.c_double),
                                      int(e.get("embedding_seed", 0)), int(e.get("k", 0)))
        h = C.c_void_p()
        _check(lib.keep_trace_create(n, arr, C.byref(h)))
        return cls(h)

    @classmethod
    def from_jsonl(cls, text: str) -> "Trace":
        return cls.from_events([json.loads(ln) for ln in text.splitlines() if ln.strip()])


def generate_episode(cfg: EpisodeConfig) -> Trace:
    """generate_episode (harness.hpp:362-413)."""
    lib = _lib()
    s, keep = cfg.c_struct()
    h = C.c_void_p()
    _check(lib.keep_trace_generate(C.byref(s), C.byref(h)))
    return Trace(h)


def _report(lib, h) -> dict:
    agg = keep_strategy_aggregate()
    _check(lib.keep_report_aggregate(h, C.byref(agg)))
    steps = []
    for i in range(agg.steps):
        s = keep_step_report()
        _check(lib.keep_report_step(h, i, C.byref(s)))
        steps.append({"step": s.step, "realized_segments": s.realized_segments, "ttft_tu": s.ttft_tu,
                      "makespan_tu": s.makespan_tu, "refresh_tu": s.refresh_tu, "div_l2": s.div_l2,
                      "div_kl": s.div_kl, "plan_sizes": [s.plan_sizes[l] for l in range(s.num_layers)],
                      "reused_tokens": s.reused_tokens, "recomputed_tokens": s.recomputed_tokens,
                      "memory_tokens": s.memory_tokens, "invalidated_tokens_delta": s.invalidated_tokens_delta,
                      "bytes_loaded_slow_delta": s.bytes_loaded_slow_delta, "wall_ms": s.wall_ms})
    n = C.c_uint64()
    _check(lib.keep_report_json(h, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib.keep_report_json(h, buf, n.value + 1, C.byref(n)))
    return {"per_step": steps,
            "aggregate": {"steps": agg.steps, "mean_ttft_tu": agg.mean_ttft_tu, "p95_ttft_tu": agg.p95_ttft_tu,
                          "mean_div_l2": agg.mean_div_l2, "mean_div_kl": agg.mean_div_kl,
                          "reuse_ratio": agg.reuse_ratio, "mean_realized_segments": agg.mean_realized_segments,
                          "invalidated_tokens": agg.invalidated_tokens, "bytes_slow": agg.bytes_slow},
            "json": buf.value.decode()}


def run_episode(ctx, trace: Trace, strategy: str, cfg: EpisodeConfig) -> dict:
    """run_episode (harness.hpp:543-817) on the GPU context `ctx` (its memory
    tier is cleared first).  Returns per_step / aggregate like report_to_json."""
    lib = _lib()
    s, keep = cfg.c_struct()
    h = C.c_void_p()
    _check(lib.keep_run_episode(ctx._h, trace._h, strategy.encode(), C.byref(s), C.byref(h)))
    try:
        out = _report(lib, h)
    finally:
        lib.keep_report_destroy(h)
    out["strategy"] = strategy
    return out


def compare_csv(ctx, trace: Trace, strategies: Sequence[str], cfg: EpisodeConfig, ks: Sequence[int] = (),
                rs: Sequence[float] = ()) -> str:
    """compare_csv (harness.hpp:828-871): the strategy comparison table."""
    lib = _lib()
    s, keep = cfg.c_struct()
    names = [x.encode() for x in strategies]
    arr = (C.c_char_p * max(1, len(names)))(*names)
    ka = np.ascontiguousarray(ks, np.int32)
    ra = np.ascontiguousarray(rs, np.float64)
    n = C.c_uint64()
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        _check(lib.keep_compare_csv(ctx._h, trace._h, len(names), arr, C.byref(s), len(ka), _p(ka, C.c_int32),
                                    len(ra), _p(ra, C.c_double), buf, cap, C.byref(n)))
        if n.value < cap:
            return buf.value.decode()
        cap = n.value + 1  # (the episodes are replayed again; results are deterministic)


class MemoryStore:
    """MemoryStore (memory_store.hpp:274-496): grouping, the static/dynamic
    state machine and retrieval.  Host bookkeeping of the device memory tier."""

    def __init__(self, segments: Sequence[dict], t: int = 10, num_groups: int = 1, seed: int = 0,
                 grouping: str = "semantic"):
        self.lib = _lib()
        n = len(segments)
        arr = (keep_segment * max(n, 1))()
        self._keep = []
        for i, sg in enumerate(segments):
            toks = np.ascontiguousarray(sg["tokens"], np.int32)
            emb = np.ascontiguousarray(sg["embedding"], np.float64)
            cat = sg.get("category", "").encode()
            self._keep += [toks, emb, cat]
            arr[i] = keep_segment(int(sg["id"]), cat, len(toks), _p(toks, C.c_int32), len(emb), _p(emb, C.c_double))
        self._h = C.c_void_p()
        cfg = keep_store_config(t, num_groups, seed, 1 if grouping == "fixed" else 0)
        _check(self.lib.keep_store_create(n, arr, C.byref(cfg), C.byref(self._h)))
        self._n = n

    def __del__(self):
        try:
            if self._h:
                self.lib.keep_store_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def groups(self) -> List[dict]:
        n = C.c_int32()
        _check(self.lib.keep_store_groups(self._h, C.byref(n), 0, None, None, None, None))
        cap = self._n + 64
        mem = np.empty(cap, np.uint32)
        cnt = np.empty(n.value, np.int32)
        st = np.empty(n.value, np.int32)
        gv = np.empty(n.value, np.uint64)
        _check(self.lib.keep_store_groups(self._h, C.byref(n), cap, _p(mem, C.c_uint32), _p(cnt, C.c_int32),
                                          _p(st, C.c_int32), _p(gv, C.c_uint64)))
        out, k = [], 0
        for g in range(n.value):
            out.append({"id": g, "members": [int(x) for x in mem[k:k + cnt[g]]],
                        "state": "static" if st[g] else "dynamic", "version": int(gv[g])})
            k += cnt[g]
        return out

    def apply_update(self, seg_id: int, tokens, step: int) -> dict:
        toks = np.ascontiguousarray(tokens, np.int32)
        cap = self._n + 1
        owners = (keep_owner * cap)()
        tk = np.empty(cap, np.uint64)
        n, ver = C.c_int32(), C.c_uint64()
        _check(self.lib.keep_store_apply_update(self._h, seg_id, len(toks), _p(toks, C.c_int32), step, cap, owners,
                                                _p(tk, C.c_uint64), C.byref(n), C.byref(ver)))
        return {"entries": [((owners[i].kind, owners[i].id), int(tk[i])) for i in range(n.value)],
                "new_segment_version": (seg_id, ver.value)}

    def advance_step(self, step: int) -> List[tuple]:
        cap = self._n
        gs = np.empty(cap, np.uint32)
        vs = np.empty(cap, np.uint64)
        n = C.c_int32()
        _check(self.lib.keep_store_advance_step(self._h, step, cap, _p(gs, C.c_uint32), _p(vs, C.c_uint64),
                                                C.byref(n)))
        return [(int(gs[i]), int(vs[i])) for i in range(n.value)]

    def retrieve(self, query_embedding, k: int) -> List[tuple]:
        q = np.ascontiguousarray(query_embedding, np.float64)
        cap = self._n
        units = (keep_owner * cap)()
        cnt = np.empty(cap, np.int32)
        segs = np.empty(cap, np.uint32)
        n = C.c_int32()
        _check(self.lib.keep_store_retrieve(self._h, _p(q, C.c_double), len(q), k, cap, units, _p(cnt, C.c_int32),
                                            cap, _p(segs, C.c_uint32), C.byref(n)))
        out, j = [], 0
        for i in range(n.value):
            out.append(((units[i].kind, units[i].id), [int(x) for x in segs[j:j + cnt[i]]]))
            j += cnt[i]
        return out

    def add_segment(self, segment: dict, step: int):
        toks = np.ascontiguousarray(segment["tokens"], np.int32)
        emb = np.ascontiguousarray(segment["embedding"], np.float64)
        cat = segment.get("category", "").encode()
        s = keep_segment(int(segment["id"]), cat, len(toks), _p(toks, C.c_int32), len(emb), _p(emb, C.c_double))
        _check(self.lib.keep_store_add_segment(self._h, C.byref(s), step))
        self._n += 1

    def state_sound(self) -> bool:
        out = C.c_int32()
        _check(self.lib.keep_store_state_sound(self._h, C.byref(out)))
        return bool(out.value)
