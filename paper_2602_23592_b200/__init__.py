"""KEEP per-layer memory prefill on B200 -- Python mirror of the reference interface.

A thin ctypes layer over the C ABI in ``include/keep_b200.h`` (the product is
``paper_2602_23592_b200/lib/libkeep_b200.so``: C++ host engine + sm_100a CUDA
kernels).  Names follow the reference (``/root/reference/proj/include/keep``):

    Model.init            -> Context.model_init          (model.hpp:54-73)
    CacheManager.put/load -> Context.memory_put / load_memory (cache_manager.hpp:69-130)
    compute_and_put       -> Context.memory_compute      (harness.hpp:512-532)
    PrefillCursor.step    -> Context.prefill_layer       (prefill.hpp:224-322)
    converge              -> Context.importance_evaluation (recompute.hpp:130-138)
    plan_keep             -> Context.plan_keep           (recompute.hpp:140-180)

There is no CPU fallback: importing works without a GPU (so the ABI can be
inspected), but creating a Context without the built library or without a
B200 raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libkeep_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "keep_b200.h")

OK, CONFIG, INPUT, PLAN, CACHE_MISS, TRACE, CUDA = range(7)
ERROR_NAMES = {CONFIG: "ConfigError", INPUT: "InputError", PLAN: "PlanError",
               CACHE_MISS: "CacheMissError", TRACE: "TraceError", CUDA: "CudaError"}
PARITY, FAST, PARITY_EXACT = 0, 1, 2
SEGMENT, GROUP = 0, 1
TIER_DEVICE, TIER_HOST = 0, 1


class KeepError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERROR_NAMES.get(code, str(code))


class keep_config(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_heads", C.c_int32), ("model_dim", C.c_int32),
                ("mlp_dim", C.c_int32), ("vocab_size", C.c_int32), ("numerics", C.c_int32),
                ("seed", C.c_uint64), ("device", C.c_int32), ("world_size", C.c_int32),
                ("rank", C.c_int32), ("max_hops", C.c_int32), ("nccl_id", C.c_void_p),
                ("nccl_comm", C.c_void_p), ("loopback", C.c_void_p)]


class keep_owner(C.Structure):
    _fields_ = [("kind", C.c_int32), ("id", C.c_uint32)]


class keep_layout(C.Structure):
    _fields_ = [("num_segments", C.c_int32), ("num_units", C.c_int32),
                ("seg_len", C.POINTER(C.c_int32)), ("tokens", C.POINTER(C.c_int32)),
                ("unit_begin", C.POINTER(C.c_int32)), ("unit_end", C.POINTER(C.c_int32)),
                ("unit_owner", C.POINTER(keep_owner))]


class keep_kv_view(C.Structure):
    _fields_ = [("keys", C.c_void_p), ("values", C.c_void_p), ("tokens", C.c_int64),
                ("tier", C.c_int32), ("elem_bytes", C.c_int32), ("load_ms", C.c_double),
                ("row_elems", C.c_int32), ("col0", C.c_int32)]


class keep_memory_stats(C.Structure):
    _fields_ = [("bytes_loaded_slow", C.c_uint64), ("cache_misses", C.c_uint64),
                ("tokens_invalidated", C.c_uint64), ("blocks", C.c_uint64),
                ("device_bytes", C.c_uint64), ("host_bytes", C.c_uint64)]


class keep_profile(C.Structure):
    _fields_ = [("ms", C.c_double * 16), ("flops", C.c_double * 16), ("bytes", C.c_double * 16),
                ("launches", C.c_int64 * 16), ("kernels", C.c_int64 * 16)]


class keep_load_record(C.Structure):
    _fields_ = [("layer", C.c_int32), ("kind", C.c_int32), ("at_layer", C.c_int32), ("owner", keep_owner),
                ("bytes", C.c_uint64), ("batch_start_ms", C.c_double), ("batch_end_ms", C.c_double),
                ("compute_start_ms", C.c_double)]


LOAD_KINDS = {0: "urgent", 1: "ahead", 2: "preload"}

PROFILE_PHASES = ["qkv", "attn", "wo", "mlp_in", "mlp_out", "summary", "select", "cached_kv", "compact",
                  "embed", "logits", "loader", "comm", "xchg", "refresh", "attn_decode"]


class keep_timeline_event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("owner", keep_owner), ("bytes", C.c_uint64),
                ("start_ms", C.c_double), ("end_ms", C.c_double)]


class keep_plan_result(C.Structure):
    _fields_ = [("plan", C.POINTER(C.c_uint8)), ("orders", C.POINTER(C.c_int32)),
                ("order_len", C.POINTER(C.c_int32)), ("hops", C.POINTER(C.c_int32)),
                ("summaries", C.POINTER(C.c_double)), ("final_hidden", C.POINTER(C.c_float)),
                ("last_logits", C.POINTER(C.c_double)), ("rows_per_layer", C.POINTER(C.c_int64)),
                ("layer_ms", C.POINTER(C.c_double)), ("ttft_ms", C.c_double)]


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


_lib = None


def load_library() -> C.CDLL:
    """Load the in-tree product library; raise loudly if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, u8p = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.POINTER(C.c_uint8)
    i32p, dp, fp = C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_float)
    sig = {
        "keep_last_error": (C.c_char_p, []),
        "keep_version": (C.c_char_p, []),
        "keep_ctx_create": (C.c_int, [C.POINTER(keep_config), C.POINTER(vp)]),
        "keep_ctx_destroy": (C.c_int, [vp]),
        "keep_ctx_synchronize": (C.c_int, [vp]),
        "keep_model_init": (C.c_int, [vp]),
        "keep_model_export": (C.c_int, [vp, fp, u64]),
        "keep_memory_put": (C.c_int, [vp, keep_owner, u64, i32, i64, fp, fp, i32]),
        "keep_memory_compute": (C.c_int, [vp, keep_owner, u64, i32, i32p, i32p, i32]),
        "keep_memory_compute_batch": (C.c_int, [vp, i32, C.POINTER(keep_owner), C.POINTER(C.c_uint64),
                                                i32p, i32p, i32p, i32]),
        "keep_load_memory": (C.c_int, [vp, keep_owner, i32, C.POINTER(keep_kv_view)]),
        "keep_memory_has_current": (C.c_int, [vp, keep_owner, u64, i32p]),
        "keep_invalidate": (C.c_int, [vp, keep_owner, u64, u64]),
        "keep_memory_stats_get": (C.c_int, [vp, C.POINTER(keep_memory_stats)]),
        "keep_memory_read": (C.c_int, [vp, keep_owner, i32, fp, fp]),
        "keep_prefill_begin": (C.c_int, [vp, C.POINTER(keep_layout), i32p, i32]),
        "keep_prefill_layer": (C.c_int, [vp, u8p, dp]),
        "keep_prefill_finish": (C.c_int, [vp, fp, fp]),
        "keep_importance_evaluation": (C.c_int, [vp, i32, dp, dp, i64, u8p, i32p, i32p, i32p]),
        "keep_ratio_schedule": (C.c_int, [i32, C.c_double, dp]),
        "keep_layer_budget": (i64, [C.c_double, i64]),
        "keep_plan_keep": (C.c_int, [vp, C.POINTER(keep_layout), i32p, i32, dp, i32,
                                     C.POINTER(keep_plan_result)]),
        "keep_plan_keep_batch": (C.c_int, [vp, C.POINTER(keep_layout), i32, i32p, i32, dp, i32,
                                           C.POINTER(keep_plan_result)]),
        "keep_selective_prefill_batch": (C.c_int, [vp, C.POINTER(keep_layout), i32, i32p, i32, u8p,
                                                   C.POINTER(keep_plan_result)]),
        "keep_ctx_trim": (C.c_int, [vp]),
        "keep_logits": (C.c_int, [vp, fp, dp]),
        "keep_divergence": (C.c_int, [vp, fp, fp, dp, dp]),
        "keep_debug_gemm_bf16": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
        "keep_set_rope": (C.c_int, [vp, C.c_double]),
        "keep_timeline_trace": (C.c_int, [vp, C.POINTER(keep_timeline_event), i32, i32p, dp]),
        "keep_debug_gemm_parity": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
        "keep_debug_exp_f64": (C.c_int, [vp, vp, i64]),
        "keep_memory_residency": (C.c_int, [vp, u64, C.POINTER(C.c_uint64)]),
        "keep_load_memory_async": (C.c_int, [vp, keep_owner, i32, C.POINTER(keep_kv_view), C.POINTER(vp)]),
        "keep_load_wait": (C.c_int, [vp]),
        "keep_comm_unique_id": (C.c_int, [C.c_char_p]),
        "keep_loader_trace": (C.c_int, [vp, C.POINTER(keep_load_record), i32, i32p]),
        "keep_shard_heads": (C.c_int, [i32, i32, i32, i32, i32p, i32p, i32p, i32p]),
        "keep_shard_rows": (C.c_int, [i64, i32, i32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "keep_loopback_create": (C.c_int, [i32, C.POINTER(vp)]),
        "keep_loopback_destroy": (C.c_int, [vp]),
        "keep_profile_enable": (C.c_int, [vp, i32]),
        "keep_profile_read": (C.c_int, [vp, C.POINTER(keep_profile), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> List[str]:
    """Function names declared by the C-ABI headers (include/keep_b200.h,
    include/keep_episode.h)."""
    import glob
    import re
    src = ""
    for h in sorted(glob.glob(os.path.join(os.path.dirname(HEADER), "*.h"))):
        with open(h) as f:
            src += f.read()
    return sorted(set(re.findall(r"\b(keep_[a-z_]+)\s*\(", src)))


def _check(rc: int):
    if rc != OK:
        raise KeepError(rc, load_library().keep_last_error().decode())


def ratio_schedule(num_layers: int, r_avg: float) -> np.ndarray:
    """recompute.hpp:33-70 (host function of the library)."""
    r = np.empty(num_layers, np.float64)
    _check(load_library().keep_ratio_schedule(num_layers, r_avg, _p(r, C.c_double)))
    return r


def layer_budget(ratio: float, num_segments: int) -> int:
    """recompute.hpp:73-77."""
    return int(load_library().keep_layer_budget(ratio, num_segments))


@dataclass
class Layout:
    """Segments in layout order plus retrieval units (prefill.hpp:41-69).

    units: [(begin, end, owner_kind, owner_id)]; empty = one dynamic segment
    owner s<position> per segment (Layout::of)."""
    seg_len: np.ndarray
    tokens: np.ndarray
    units: list = field(default_factory=list)

    @property
    def S(self) -> int:
        return int(len(self.seg_len))

    def c_struct(self) -> keep_layout:
        self._keep = [np.ascontiguousarray(self.seg_len, np.int32), np.ascontiguousarray(self.tokens, np.int32)]
        lay = keep_layout()
        lay.num_segments = self.S
        lay.seg_len = _p(self._keep[0], C.c_int32)
        lay.tokens = _p(self._keep[1], C.c_int32)
        lay.num_units = len(self.units)
        if self.units:
            ub = np.array([u[0] for u in self.units], np.int32)
            ue = np.array([u[1] for u in self.units], np.int32)
            owners = (keep_owner * len(self.units))(*[keep_owner(int(u[2]), int(u[3])) for u in self.units])
            self._keep += [ub, ue, owners]
            lay.unit_begin = _p(ub, C.c_int32)
            lay.unit_end = _p(ue, C.c_int32)
            lay.unit_owner = C.cast(owners, C.POINTER(keep_owner))
        return lay

    def owners(self) -> List[Tuple[int, int, int, int]]:
        """(owner_kind, owner_id, begin, end) of every unit."""
        if self.units:
            return [(int(u[2]), int(u[3]), int(u[0]), int(u[1])) for u in self.units]
        return [(SEGMENT, i, i, i + 1) for i in range(self.S)]


def shard_heads(num_heads: int, model_dim: int, world: int, rank: int) -> Tuple[int, int, int, int]:
    """(h0, hn, c0, cn): the heads and model columns a rank owns (keep_shard_heads)."""
    v = [C.c_int32() for _ in range(4)]
    _check(load_library().keep_shard_heads(num_heads, model_dim, world, rank, *[C.byref(x) for x in v]))
    return tuple(int(x.value) for x in v)


def shard_rows(n: int, world: int, rank: int) -> Tuple[int, int]:
    """(r0, m): a rank's Wo + MLP block of n compact rows (keep_shard_rows)."""
    r0, m = C.c_int64(), C.c_int64()
    _check(load_library().keep_shard_rows(n, world, rank, C.byref(r0), C.byref(m)))
    return int(r0.value), int(m.value)


def comm_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0 makes it, every rank receives it)."""
    buf = C.create_string_buffer(128)
    _check(load_library().keep_comm_unique_id(buf))
    return buf.raw


class LoopbackGroup:
    """G logical ranks on one GPU in one process (one host thread per rank):
    the test double for the sharded collectives (comm.cu)."""

    def __init__(self, world: int):
        self.world = world
        self._h = C.c_void_p()
        _check(load_library().keep_loopback_create(world, C.byref(self._h)))

    def close(self):
        if self._h:
            load_library().keep_loopback_destroy(self._h)
            self._h = C.c_void_p()


class Context:
    """One B200 context: model weights, memory tier and a prefill cursor.

    KV-head sharding: world > 1 with rank in [0, world) and either nccl_id
    (bytes from comm_unique_id(), shared by all ranks) or a LoopbackGroup."""

    def __init__(self, L: int, H: int, d: int, mlp: int, V: int, seed: int,
                 numerics: int = PARITY, device: int = 0, world: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, loopback: Optional[LoopbackGroup] = None, max_hops: int = 0):
        self.lib = load_library()
        cfg = keep_config(L, H, d, mlp, V, numerics, seed, device, world, rank, max_hops)
        self._id = None
        if nccl_id is not None:
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(self._id, C.c_void_p)
        if loopback is not None:
            cfg.loopback = loopback._h
        self.world, self.rank = world, rank
        self.dl = d // world
        self._h = C.c_void_p()
        _check(self.lib.keep_ctx_create(C.byref(cfg), C.byref(self._h)))
        self.L, self.H, self.d, self.mlp, self.V, self.seed = L, H, d, mlp, V, seed
        self.numerics = numerics
        self._T = 0
        self._S = 0

    def close(self):
        if self._h:
            self.lib.keep_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- model ------------------------------------------------------------
    def trim(self):
        """Release the grow-only workspaces (keep_ctx_trim)."""
        _check(self.lib.keep_ctx_trim(self._h))

    def set_rope(self, theta: float):
        """Opt-in RoPE position re-shift hook (0 = off: the reference's NoPE)."""
        _check(self.lib.keep_set_rope(self._h, float(theta)))
        return self

    def model_init(self):
        _check(self.lib.keep_model_init(self._h))
        return self

    def export_weights(self) -> np.ndarray:
        n = 2 * self.V * self.d + self.L * (4 * self.d * self.d + 2 * self.d * self.mlp)
        w = np.empty(n, np.float32)
        _check(self.lib.keep_model_export(self._h, _p(w, C.c_float), n))
        return w

    def logits(self, row) -> np.ndarray:
        row = np.ascontiguousarray(row, np.float32)
        out = np.empty(self.V, np.float64)
        _check(self.lib.keep_logits(self._h, _p(row, C.c_float), _p(out, C.c_double)))
        return out

    def divergence(self, row_a, row_b):
        """divergence (prefill.hpp:501-531) on the device: (L2, symmetric KL)."""
        a = np.ascontiguousarray(row_a, np.float32)
        b = np.ascontiguousarray(row_b, np.float32)
        l2, kl = C.c_double(), C.c_double()
        _check(self.lib.keep_divergence(self._h, _p(a, C.c_float), _p(b, C.c_float), C.byref(l2), C.byref(kl)))
        return l2.value, kl.value

    # -- per-phase device timing --------------------------------------------
    def profile_enable(self, on=True):
        _check(self.lib.keep_profile_enable(self._h, int(bool(on))))

    def profile_read(self, reset=True) -> dict:
        pr = keep_profile()
        _check(self.lib.keep_profile_read(self._h, C.byref(pr), int(bool(reset))))
        return {name: {"ms": pr.ms[i], "flops": pr.flops[i], "bytes": pr.bytes[i],
                       "launches": int(pr.launches[i]), "kernels": int(pr.kernels[i])}
                for i, name in enumerate(PROFILE_PHASES)}

    # -- memory tier (load_memory) ----------------------------------------
    def memory_put(self, kind, oid, version, layer, keys, values, tier=TIER_DEVICE):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        _check(self.lib.keep_memory_put(self._h, keep_owner(kind, oid), version, layer, keys.shape[0],
                                        _p(keys, C.c_float), _p(values, C.c_float), tier))

    def memory_compute(self, kind, oid, version, member_lens, tokens, tier=TIER_DEVICE):
        ml = np.ascontiguousarray(member_lens, np.int32)
        tk = np.ascontiguousarray(tokens, np.int32)
        _check(self.lib.keep_memory_compute(self._h, keep_owner(kind, oid), version, len(ml),
                                            _p(ml, C.c_int32), _p(tk, C.c_int32), tier))

    def memory_compute_batch(self, owners: Sequence[Tuple[int, int]], versions, members: Sequence[Sequence[int]],
                             tokens, tier=TIER_DEVICE):
        n = len(owners)
        arr = (keep_owner * n)(*[keep_owner(k, i) for k, i in owners])
        ver = np.ascontiguousarray(versions, np.uint64)
        om = np.array([len(m) for m in members], np.int32)
        ml = np.array([x for m in members for x in m], np.int32)
        tk = np.ascontiguousarray(tokens, np.int32)
        _check(self.lib.keep_memory_compute_batch(self._h, n, C.cast(arr, C.POINTER(keep_owner)),
                                                  ver.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                  _p(om, C.c_int32), _p(ml, C.c_int32), _p(tk, C.c_int32), tier))

    def memory_compute_layout(self, layout: Layout, version=1, tier=TIER_DEVICE):
        """Canonical KV for every unit of a layout (compute_and_put)."""
        starts = np.concatenate([[0], np.cumsum(layout.seg_len)]).astype(np.int64)
        owners, members, toks = [], [], []
        for kind, oid, b, e in layout.owners():
            owners.append((kind, oid))
            members.append([int(x) for x in layout.seg_len[b:e]])
            toks.append(np.asarray(layout.tokens[starts[b]:starts[e]]))
        self.memory_compute_batch(owners, [version] * len(owners), members, np.concatenate(toks), tier)

    def memory_refresh(self, layout: Layout, owner_idx, version, tier=TIER_DEVICE):
        """compute_and_put for a subset of a layout's owners (indices into
        layout.owners()): the canonical-KV refresh of updated memory
        (harness.hpp:609-628), in place when the blocks already exist."""
        starts = np.concatenate([[0], np.cumsum(layout.seg_len)]).astype(np.int64)
        allo = layout._owners_cache if getattr(layout, "_owners_cache", None) else layout.owners()
        layout._owners_cache = allo
        owners, members, toks = [], [], []
        for u in owner_idx:
            kind, oid, b, e = allo[int(u)]
            owners.append((kind, oid))
            members.append([int(x) for x in layout.seg_len[b:e]])
            toks.append(np.asarray(layout.tokens[starts[b]:starts[e]]))
        if owners:
            self.memory_compute_batch(owners, [version] * len(owners), members, np.concatenate(toks), tier)

    def memory_residency(self, hbm_budget_bytes: int) -> int:
        """Keep the deepest layers of the pinned-host memory also in HBM (the
        capacity-bounded fast tier); returns the resident bytes."""
        out = C.c_uint64()
        _check(self.lib.keep_memory_residency(self._h, int(hbm_budget_bytes), C.byref(out)))
        return out.value

    def load_memory_async(self, kind, oid, layer):
        """load_memory without waiting: (view, completion event handle);
        call load_wait() (or wait on the event) before reading the view."""
        v = keep_kv_view()
        ev = C.c_void_p()
        _check(self.lib.keep_load_memory_async(self._h, keep_owner(kind, oid), layer, C.byref(v), C.byref(ev)))
        return v, ev.value

    def load_wait(self):
        _check(self.lib.keep_load_wait(self._h))

    def load_memory(self, kind, oid, layer) -> keep_kv_view:
        v = keep_kv_view()
        _check(self.lib.keep_load_memory(self._h, keep_owner(kind, oid), layer, C.byref(v)))
        return v

    def loader_trace(self) -> list:
        """The K10 load schedule of the last prefill (keep_loader_trace)."""
        n = C.c_int32()
        _check(self.lib.keep_loader_trace(self._h, None, 0, C.byref(n)))
        buf = (keep_load_record * max(n.value, 1))()
        _check(self.lib.keep_loader_trace(self._h, buf, n.value, C.byref(n)))
        return [{"layer": r.layer, "kind": LOAD_KINDS[r.kind], "at_layer": r.at_layer,
                 "owner": (r.owner.kind, r.owner.id), "bytes": int(r.bytes), "start_ms": r.batch_start_ms,
                 "end_ms": r.batch_end_ms, "compute_start_ms": r.compute_start_ms} for r in buf[: n.value]]

    def timeline_trace(self):
        """keep_timeline_trace: the realised timeline of the last plan_keep over
        pinned-host memory as reference Timeline events + the D2 attention fraction."""
        n, frac = C.c_int32(), C.c_double()
        _check(self.lib.keep_timeline_trace(self._h, None, 0, C.byref(n), C.byref(frac)))
        buf = (keep_timeline_event * max(n.value, 1))()
        _check(self.lib.keep_timeline_trace(self._h, buf, n.value, C.byref(n), C.byref(frac)))
        evs = [{"kind": e.kind, "layer": e.layer, "owner": (e.owner.kind, e.owner.id), "bytes": int(e.bytes),
                "start": e.start_ms, "end": e.end_ms} for e in buf[: n.value]]
        return evs, frac.value

    def has_current(self, kind, oid, version) -> bool:
        out = C.c_int32()
        _check(self.lib.keep_memory_has_current(self._h, keep_owner(kind, oid), version, C.byref(out)))
        return bool(out.value)

    def invalidate(self, kind, oid, new_version, tokens=0):
        _check(self.lib.keep_invalidate(self._h, keep_owner(kind, oid), new_version, tokens))

    def memory_stats(self) -> dict:
        s = keep_memory_stats()
        _check(self.lib.keep_memory_stats_get(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def memory_read(self, kind, oid, layer, tokens):
        """[tokens x d/world]: this rank's head columns of the block."""
        k = np.empty((tokens, self.dl), np.float32)
        v = np.empty((tokens, self.dl), np.float32)
        _check(self.lib.keep_memory_read(self._h, keep_owner(kind, oid), layer, _p(k, C.c_float), _p(v, C.c_float)))
        return k, v

    # -- prefill cursor (prefill_layer) -------------------------------------
    def prefill_begin(self, layout: Layout, query):
        q = np.ascontiguousarray(query if len(query) else np.zeros(1), np.int32)
        self._lay = layout.c_struct()
        _check(self.lib.keep_prefill_begin(self._h, C.byref(self._lay), _p(q, C.c_int32), len(query)))
        self._T = int(np.sum(layout.seg_len)) + len(query)
        self._S = layout.S

    def prefill_layer(self, active, summary=True):
        a = np.ascontiguousarray(active, np.uint8)
        S = self._S
        out = np.empty(S + S * S, np.float64) if summary else None
        _check(self.lib.keep_prefill_layer(self._h, _p(a, C.c_uint8), _p(out, C.c_double)))
        if out is None:
            return None
        return out[:S].copy(), out[S:].reshape(S, S).copy()

    def prefill_finish(self, kv=True):
        fh = np.empty((self._T, self.d), np.float32)
        kvb = np.empty((self.L, 2, self._T, self.dl), np.float32) if kv else None
        _check(self.lib.keep_prefill_finish(self._h, _p(fh, C.c_float), _p(kvb, C.c_float)))
        return fh, kvb

    def selective_prefill(self, layout: Layout, query, plan):
        """selective_prefill (prefill.hpp:478-497) through the cursor."""
        plan = np.asarray(plan, np.uint8)
        self.prefill_begin(layout, query)
        qts, sts = [], []
        for l in range(self.L):
            q_, s_ = self.prefill_layer(plan[l])
            qts.append(q_)
            sts.append(s_)
        fh, kv = self.prefill_finish()
        return {"final_hidden": fh, "kv": kv, "qts": np.array(qts), "sts": np.array(sts)}

    # -- selection ------------------------------------------------------------
    def importance_evaluation(self, qts, sts, budget, candidates=None):
        qts = np.ascontiguousarray(qts, np.float64)
        S = len(qts)
        sts = np.ascontiguousarray(sts, np.float64).reshape(S, S)
        cand = None if candidates is None else np.ascontiguousarray(candidates, np.uint8)
        order = np.empty(max(S, 1), np.int32)
        n, hops = C.c_int32(), C.c_int32()
        _check(self.lib.keep_importance_evaluation(self._h, S, _p(qts, C.c_double), _p(sts, C.c_double), budget,
                                                   _p(cand, C.c_uint8), _p(order, C.c_int32), C.byref(n),
                                                   C.byref(hops)))
        return [int(x) for x in order[: n.value]], hops.value

    def _schedule(self, sched) -> np.ndarray:
        # plan_keep reads sched[l + 1] for every layer (recompute.hpp:144:
        # ConfigError "schedule length != num_layers")
        sched = np.ascontiguousarray(sched, np.float64).ravel()
        if len(sched) != self.L:
            raise KeepError(1, f"schedule length {len(sched)} != num_layers {self.L}")
        return sched

    def plan_keep(self, layout: Layout, query, sched, multihop=True, summaries=False, final_hidden=True):
        L, S = self.L, layout.S
        T = int(np.sum(layout.seg_len)) + len(query)
        plan = np.empty((L, S), np.uint8)
        orders = np.full((L, S), -1, np.int32)
        olen = np.empty(L, np.int32)
        hops = np.empty(L, np.int32)
        summ = np.empty((L, S + S * S), np.float64) if summaries else None
        fh = np.empty((T, self.d), np.float32) if final_hidden else None
        logits = np.empty(self.V, np.float64)
        rows = np.empty(L, np.int64)
        lms = np.empty(L, np.float64)
        res = keep_plan_result(_p(plan, C.c_uint8), _p(orders, C.c_int32), _p(olen, C.c_int32),
                               _p(hops, C.c_int32), _p(summ, C.c_double), _p(fh, C.c_float),
                               _p(logits, C.c_double), _p(rows, C.c_int64), _p(lms, C.c_double), 0.0)
        q = np.ascontiguousarray(query if len(query) else np.zeros(1), np.int32)
        sched = self._schedule(sched)
        lay = layout.c_struct()
        _check(self.lib.keep_plan_keep(self._h, C.byref(lay), _p(q, C.c_int32), len(query),
                                       _p(sched, C.c_double), int(bool(multihop)), C.byref(res)))
        out = {"plan": plan, "hops": hops,
               "orders": [None if olen[l] < 0 else [int(x) for x in orders[l, : olen[l]]] for l in range(L)],
               "final_hidden": fh, "last_logits": logits, "rows_per_layer": rows, "layer_ms": lms,
               "ttft_ms": res.ttft_ms}
        if summaries:
            out["qts"] = summ[:, :S].copy()
            out["sts"] = summ[:, S:].reshape(L, S, S).copy()
        return out

    def plan_keep_batch(self, layout: Layout, queries, sched, multihop=True, final_hidden=False, summaries=False,
                        plans=None):
        """keep_plan_keep_batch: B planning queries (rows of `queries`, equal
        lengths) over one memory layout; one result dict per query, as
        plan_keep returns it (ttft_ms / layer_ms are the batch's)."""
        Q = np.ascontiguousarray(np.atleast_2d(queries), np.int32)
        B, qlen = Q.shape
        L, S = self.L, layout.S
        T = int(np.sum(layout.seg_len)) + qlen
        bufs, res = [], (keep_plan_result * B)()
        for b in range(B):
            f = {"plan": np.empty((L, S), np.uint8), "orders": np.full((L, S), -1, np.int32),
                 "olen": np.empty(L, np.int32), "hops": np.empty(L, np.int32),
                 "summ": np.empty((L, S + S * S), np.float64) if summaries else None,
                 "fh": np.empty((T, self.d), np.float32) if final_hidden else None,
                 "logits": np.empty(self.V, np.float64), "rows": np.empty(L, np.int64), "lms": np.empty(L, np.float64)}
            bufs.append(f)
            res[b] = keep_plan_result(_p(f["plan"], C.c_uint8), _p(f["orders"], C.c_int32), _p(f["olen"], C.c_int32),
                                      _p(f["hops"], C.c_int32), _p(f["summ"], C.c_double), _p(f["fh"], C.c_float),
                                      _p(f["logits"], C.c_double), _p(f["rows"], C.c_int64), _p(f["lms"], C.c_double),
                                      0.0)
        lay = layout.c_struct()
        if plans is not None:  # keep_selective_prefill_batch
            pl = np.ascontiguousarray(plans, np.uint8).reshape(B, L, S)
            _check(self.lib.keep_selective_prefill_batch(self._h, C.byref(lay), B, _p(Q, C.c_int32), qlen,
                                                         _p(pl, C.c_uint8), res))
        else:
            sched = self._schedule(sched)
            _check(self.lib.keep_plan_keep_batch(self._h, C.byref(lay), B, _p(Q, C.c_int32), qlen,
                                                 _p(sched, C.c_double), int(bool(multihop)), res))
        outs = []
        for b, f in enumerate(bufs):
            o = {"plan": f["plan"], "hops": f["hops"],
                 "orders": [None if f["olen"][l] < 0 else [int(x) for x in f["orders"][l, : f["olen"][l]]]
                            for l in range(L)],
                 "final_hidden": f["fh"], "last_logits": f["logits"], "rows_per_layer": f["rows"],
                 "layer_ms": f["lms"], "ttft_ms": res[b].ttft_ms}
            if summaries:
                o["qts"] = f["summ"][:, :S].copy()
                o["sts"] = f["summ"][:, S:].reshape(L, S, S).copy()
            outs.append(o)
        return outs
