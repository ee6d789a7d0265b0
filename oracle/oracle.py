"""ctypes binding of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Binds either implementation of oracle/keep_oracle.h:
  Oracle("ko")  -- oracle/libkeep_oracle.so, the plain-C restatement
  Oracle("kr")  -- oracle/_ref/libkeep_ref.so, the unmodified reference
                   headers behind a C shim (built only where /root/reference
                   exists; travels as a prebuilt artefact)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
this module, as the checker or the timed CPU baseline -- never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATHS = {
    "ko": os.path.join(HERE, "libkeep_oracle.so"),
    "kr": os.path.join(HERE, "_ref", "libkeep_ref.so"),
}

ERRORS = {1: "ConfigError", 2: "InputError", 3: "PlanError", 4: "CacheMissError",
          5: "TraceError", 9: "InternalError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


class keep_problem(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("num_heads", C.c_int32), ("model_dim", C.c_int32),
        ("mlp_dim", C.c_int32), ("vocab_size", C.c_int32), ("pad_", C.c_int32),
        ("seed", C.c_uint64),
        ("num_segments", C.c_int32), ("query_len", C.c_int32),
        ("seg_len", C.POINTER(C.c_int32)), ("tokens", C.POINTER(C.c_int32)),
        ("query", C.POINTER(C.c_int32)),
        ("num_units", C.c_int32), ("pad2_", C.c_int32),
        ("unit_begin", C.POINTER(C.c_int32)), ("unit_end", C.POINTER(C.c_int32)),
        ("unit_is_group", C.POINTER(C.c_int32)),
    ]


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class Problem:
    """Model config + layout + query (mirrors keep_problem)."""
    L: int
    H: int
    d: int
    mlp: int
    V: int
    seed: int
    seg_len: np.ndarray
    tokens: np.ndarray
    query: np.ndarray
    units: list = field(default_factory=list)  # [(begin, end, is_group)]

    @property
    def S(self) -> int:
        return int(len(self.seg_len))

    @property
    def Tm(self) -> int:
        return int(self.seg_len.sum())

    @property
    def T(self) -> int:
        return self.Tm + int(len(self.query))

    def c_struct(self) -> keep_problem:
        self._keep = [np.ascontiguousarray(self.seg_len, np.int32),
                      np.ascontiguousarray(self.tokens, np.int32),
                      np.ascontiguousarray(self.query if len(self.query) else np.zeros(1), np.int32)]
        ub = np.array([u[0] for u in self.units] or [0], np.int32)
        ue = np.array([u[1] for u in self.units] or [0], np.int32)
        ug = np.array([int(u[2]) for u in self.units] or [0], np.int32)
        self._keep += [ub, ue, ug]
        p = keep_problem()
        p.num_layers, p.num_heads, p.model_dim = self.L, self.H, self.d
        p.mlp_dim, p.vocab_size, p.seed = self.mlp, self.V, self.seed
        p.num_segments, p.query_len = self.S, int(len(self.query))
        p.seg_len = _ptr(self._keep[0], C.c_int32)
        p.tokens = _ptr(self._keep[1], C.c_int32)
        p.query = _ptr(self._keep[2], C.c_int32)
        p.num_units = len(self.units)
        p.unit_begin, p.unit_end, p.unit_is_group = (_ptr(ub, C.c_int32), _ptr(ue, C.c_int32),
                                                     _ptr(ug, C.c_int32))
        return p


def build() -> None:
    """Build the restatement (and the reference shim where the tree exists)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True)


def available(prefix: str) -> bool:
    return os.path.exists(LIB_PATHS[prefix])


class kr_timeline_event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("owner_kind", C.c_int32), ("owner_id", C.c_uint32),
                ("bytes", C.c_uint64), ("start", C.c_double), ("end", C.c_double)]


class Oracle:
    def __init__(self, prefix: str = "ko"):
        path = LIB_PATHS[prefix]
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.prefix = prefix
        self.lib = lib = C.CDLL(path)
        P = prefix + "_"
        f = lambda n: getattr(lib, P + n)  # noqa: E731
        dp, fp, u8p, i32p = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                             C.POINTER(C.c_uint8), C.POINTER(C.c_int32))
        pp = C.POINTER(keep_problem)
        f("weight_count").restype = C.c_uint64
        f("weight_count").argtypes = [C.c_int] * 5
        f("model_init").argtypes = [C.c_int] * 5 + [C.c_uint64, fp]
        f("make_instance_layout").argtypes = [C.c_uint64] + [C.c_int] * 5 + [i32p] * 3
        f("ratio_schedule").argtypes = [C.c_int, C.c_double, dp]
        f("layer_budget").restype = C.c_int64
        f("layer_budget").argtypes = [C.c_double, C.c_int64]
        f("converge").argtypes = [C.c_int, dp, dp, C.c_int64, u8p, i32p, i32p, i32p]
        f("canonical_kv").argtypes = [pp, fp, fp]
        f("full_prefill").argtypes = [pp, fp, fp, fp, dp]
        f("selective_prefill").argtypes = [pp, fp, fp, u8p, fp, fp, dp]
        f("plan_keep").argtypes = [pp, fp, fp, dp, C.c_int, u8p, i32p, i32p, i32p, dp, fp, fp]
        f("divergence").argtypes = [pp, fp, fp, fp, dp, dp]
        f("logits").argtypes = [pp, fp, fp, dp]
        f("last_error").restype = C.c_char_p
        if prefix == "ko":
            lib.ko_set_max_hops.argtypes = [C.c_int]
        self._f = f

    def set_max_hops(self, max_hops: int):
        """restatement only (ko): cap converge at max_hops hops, 0 = uncapped."""
        if self.prefix != "ko":
            raise OracleError(1, "the hop cap exists only in the restatement (the reference has none)")
        self.lib.ko_set_max_hops(int(max_hops))

    def validate_timeline(self, plan, seg_len, query_tokens, units, slow_bytes, attention_fraction, events):
        """The reference's validate_timeline (pipeline_sim.hpp:340-428) over a
        realised timeline (kr only).  units: [(begin, end, is_group, owner_id)];
        slow_bytes: [n_units x L]; events: dicts {kind, layer, owner (kind, id),
        bytes, start, end}.  Returns the violation codes (empty = valid)."""
        if self.prefix != "kr":
            raise OracleError(1, "validate_timeline is the reference's own checker (kr)")
        plan = np.ascontiguousarray(plan, np.uint8)
        L, S = plan.shape
        sl = np.ascontiguousarray(seg_len, np.int32)
        ub = np.array([u[0] for u in units], np.int32)
        ue = np.array([u[1] for u in units], np.int32)
        ug = np.array([int(u[2]) for u in units], np.int32)
        uo = np.array([u[3] for u in units], np.uint32)
        sb = np.ascontiguousarray(slow_bytes, np.uint64).reshape(len(units), L)
        ev = (kr_timeline_event * max(len(events), 1))()
        for i, e in enumerate(events):
            ev[i] = kr_timeline_event(e["kind"], e["layer"], e.get("owner", (0, 0))[0], e.get("owner", (0, 0))[1],
                                      e.get("bytes", 0), e["start"], e["end"])
        buf = C.create_string_buffer(256)
        f = self.lib.kr_validate_timeline
        f.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.c_int, C.c_int,
                      C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_uint32),
                      C.POINTER(C.c_uint64), C.c_double, C.POINTER(kr_timeline_event), C.c_int, C.c_char_p, C.c_int]
        self._check(f(L, S, _ptr(plan, C.c_uint8), _ptr(sl, C.c_int32), int(query_tokens), len(units),
                      _ptr(ub, C.c_int32), _ptr(ue, C.c_int32), _ptr(ug, C.c_int32), _ptr(uo, C.c_uint32),
                      _ptr(sb, C.c_uint64), float(attention_fraction), ev, len(events), buf, 256))
        txt = buf.value.decode()
        return txt.split() if txt else []

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self._f("last_error")().decode())

    # -- model / instance -------------------------------------------------
    def weight_count(self, L, H, d, mlp, V) -> int:
        return int(self._f("weight_count")(L, H, d, mlp, V))

    def model_init(self, L, H, d, mlp, V, seed) -> np.ndarray:
        w = np.empty(self.weight_count(L, H, d, mlp, V), np.float32)
        self._check(self._f("model_init")(L, H, d, mlp, V, seed, _ptr(w, C.c_float)))
        return w

    def make_instance(self, seed, S, L=4, H=4, d=32, mlp=64, V=128, lo=8, hi=12, qlen=8) -> Problem:
        """testutil::make_instance (tests/test_util.hpp:19-40) minus the cache."""
        seg_len = np.empty(S, np.int32)
        tokens = np.empty(S * hi, np.int32)
        query = np.empty(max(qlen, 1), np.int32)
        self._check(self._f("make_instance_layout")(seed, S, V, lo, hi, qlen, _ptr(seg_len, C.c_int32),
                                                    _ptr(tokens, C.c_int32), _ptr(query, C.c_int32)))
        return Problem(L, H, d, mlp, V, seed, seg_len, tokens[: int(seg_len.sum())].copy(), query[:qlen].copy())

    # -- schedule / selector ----------------------------------------------
    def ratio_schedule(self, L, r_avg) -> np.ndarray:
        r = np.empty(L, np.float64)
        self._check(self._f("ratio_schedule")(L, r_avg, _ptr(r, C.c_double)))
        return r

    def layer_budget(self, ratio, S) -> int:
        return int(self._f("layer_budget")(ratio, S))

    def converge(self, qts, sts, budget, candidates=None):
        qts = np.ascontiguousarray(qts, np.float64)
        S = len(qts)
        sts = np.ascontiguousarray(sts, np.float64).reshape(S, S)
        cand = None if candidates is None else np.ascontiguousarray(candidates, np.uint8)
        order = np.empty(max(S, 1), np.int32)
        n, hops = C.c_int32(), C.c_int32()
        self._check(self._f("converge")(S, _ptr(qts, C.c_double), _ptr(sts, C.c_double), budget,
                                        _ptr(cand, C.c_uint8), _ptr(order, C.c_int32),
                                        C.byref(n), C.byref(hops)))
        return [int(x) for x in order[: n.value]], hops.value

    # -- prefill ------------------------------------------------------------
    def canonical_kv(self, p: Problem, w) -> np.ndarray:
        out = np.empty(p.L * 2 * p.Tm * p.d, np.float32)
        ps = p.c_struct()
        self._check(self._f("canonical_kv")(C.byref(ps), _ptr(w, C.c_float), _ptr(out, C.c_float)))
        return out.reshape(p.L, 2, p.Tm, p.d)

    def _outs(self, p: Problem, kv: bool):
        fh = np.empty((p.T, p.d), np.float32)
        kvb = np.empty((p.L, 2, p.T, p.d), np.float32) if kv else None
        sm = np.empty((p.L, p.S + p.S * p.S), np.float64)
        return fh, kvb, sm

    @staticmethod
    def _split(p: Problem, sm):
        return sm[:, : p.S].copy(), sm[:, p.S:].reshape(p.L, p.S, p.S).copy()

    def full_prefill(self, p: Problem, w, kv=True):
        fh, kvb, sm = self._outs(p, kv)
        ps = p.c_struct()
        self._check(self._f("full_prefill")(C.byref(ps), _ptr(w, C.c_float), _ptr(fh, C.c_float),
                                            _ptr(kvb, C.c_float), _ptr(sm, C.c_double)))
        qts, sts = self._split(p, sm)
        return {"final_hidden": fh, "kv": kvb, "qts": qts, "sts": sts}

    def selective_prefill(self, p: Problem, w, plan, cached=None, kv=True):
        fh, kvb, sm = self._outs(p, kv)
        plan = np.ascontiguousarray(plan, np.uint8)
        ps = p.c_struct()
        cp = None if cached is None else np.ascontiguousarray(cached, np.float32)
        self._check(self._f("selective_prefill")(C.byref(ps), _ptr(w, C.c_float), _ptr(cp, C.c_float),
                                                 _ptr(plan, C.c_uint8), _ptr(fh, C.c_float),
                                                 _ptr(kvb, C.c_float), _ptr(sm, C.c_double)))
        qts, sts = self._split(p, sm)
        return {"final_hidden": fh, "kv": kvb, "qts": qts, "sts": sts}

    def plan_keep(self, p: Problem, w, sched, multihop=True, cached=None, kv=False):
        L, S = p.L, p.S
        plan = np.empty((L, S), np.uint8)
        orders = np.full((L, S), -1, np.int32)
        olen = np.empty(L, np.int32)
        hops = np.empty(L, np.int32)
        fh, kvb, sm = self._outs(p, kv)
        sched = np.ascontiguousarray(sched, np.float64)
        ps = p.c_struct()
        cp = None if cached is None else np.ascontiguousarray(cached, np.float32)
        self._check(self._f("plan_keep")(C.byref(ps), _ptr(w, C.c_float), _ptr(cp, C.c_float),
                                         _ptr(sched, C.c_double), int(bool(multihop)),
                                         _ptr(plan, C.c_uint8), _ptr(orders, C.c_int32),
                                         _ptr(olen, C.c_int32), _ptr(hops, C.c_int32),
                                         _ptr(sm, C.c_double), _ptr(fh, C.c_float), _ptr(kvb, C.c_float)))
        qts, sts = self._split(p, sm)
        order_list = [None if olen[l] < 0 else [int(x) for x in orders[l, : olen[l]]] for l in range(L)]
        return {"plan": plan, "orders": order_list, "hops": hops.copy(), "qts": qts, "sts": sts,
                "final_hidden": fh, "kv": kvb}

    def logits(self, p: Problem, w, row) -> np.ndarray:
        out = np.empty(p.V, np.float64)
        ps = p.c_struct()
        row = np.ascontiguousarray(row, np.float32)
        self._check(self._f("logits")(C.byref(ps), _ptr(w, C.c_float), _ptr(row, C.c_float),
                                      _ptr(out, C.c_double)))
        return out

    def divergence(self, p: Problem, w, row_a, row_b):
        l2, kl = C.c_double(), C.c_double()
        ps = p.c_struct()
        a = np.ascontiguousarray(row_a, np.float32)
        b = np.ascontiguousarray(row_b, np.float32)
        self._check(self._f("divergence")(C.byref(ps), _ptr(w, C.c_float), _ptr(a, C.c_float),
                                          _ptr(b, C.c_float), C.byref(l2), C.byref(kl)))
        return l2.value, kl.value
