"""Generate the golden vectors in tests/golden/ from the UNMODIFIED reference.

Runs only where /root/reference exists (this build container): it builds
oracle/_ref/libkeep_ref.so (the reference headers behind a C shim) and records
the reference's outputs for the known-answer cases its own tests pin
(SURVEY.md section 8(c)).  The committed JSON is what the CPU and GPU parity
tests read on any machine.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, OracleError, build  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# acceptance.cpp:32-34
ACCEPT_SEEDS = [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 22, 23]

MASK64 = (1 << 64) - 1


class PyRng:
    """keep::Rng (prng.hpp:34-82) -- used only to regenerate the reference
    tests' random *inputs* (test_recompute.cpp:224-247); expected outputs come
    from the reference shim."""

    def __init__(self, seed: int):
        self.s = seed & MASK64
        self.next_u64()
        self.next_u64()

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def next_below(self, n: int) -> int:
        return self.next_u64() % n

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def instance_case(kr: Oracle, seed, S, L=4, H=4, d=32, mlp=64, V=128, lo=8, hi=12, qlen=8,
                  r_avg=0.5, units=None, multihop=True, sched=None):
    p = kr.make_instance(seed, S, L, H, d, mlp, V, lo, hi, qlen)
    if units:
        p.units = units
    w = kr.model_init(L, H, d, mlp, V, seed)
    r = np.asarray(sched, np.float64) if sched is not None else kr.ratio_schedule(L, r_avg)
    res = kr.plan_keep(p, w, r, multihop=multihop, kv=True)
    full = kr.full_prefill(p, w)
    l2, kl = kr.divergence(p, w, res["final_hidden"][-1], full["final_hidden"][-1])
    canon = kr.canonical_kv(p, w)
    return {
        "seed": seed, "S": S, "L": L, "H": H, "d": d, "mlp": mlp, "V": V, "lo": lo, "hi": hi,
        "qlen": qlen, "r_avg": r_avg, "units": units or [], "multihop": multihop,
        "sched": [float(x) for x in r],
        "seg_len": [int(x) for x in p.seg_len], "tokens_sha": sha(p.tokens),
        "query": [int(x) for x in p.query],
        "plan": res["plan"].astype(int).tolist(), "orders": res["orders"],
        "hops": [int(x) for x in res["hops"]],
        "qts": res["qts"].tolist(), "sts": res["sts"].tolist(),
        "final_hidden_sha": sha(res["final_hidden"]), "kv_sha": sha(res["kv"]),
        "canonical_kv_sha": sha(canon),
        "last_row": [float(x) for x in res["final_hidden"][-1]],
        "full_last_row": [float(x) for x in full["final_hidden"][-1]],
        "full_final_hidden_sha": sha(full["final_hidden"]),
        "div_l2": l2, "div_kl": kl,
    }


def main():
    build()
    kr = Oracle("kr")
    g = {"generator": "tests/golden/make_golden.py over oracle/_ref (unmodified reference)"}

    # -- weights (model.hpp:54-73, 88-94) --------------------------------------
    wcases = []
    for cfg in [(4, 4, 32, 64, 128, 2), (2, 8, 64, 128, 256, 7), (1, 2, 8, 8, 32, 11)]:
        w = kr.model_init(*cfg)
        wcases.append({"cfg": list(cfg), "sha": sha(w), "count": int(w.size),
                       "head": [float(x) for x in w[:16]], "tail": [float(x) for x in w[-16:]]})
    g["weights"] = wcases

    # -- ratio schedule / budgets (recompute.hpp:33-77; test_recompute.cpp:127-163)
    sched = []
    for L, ra in [(1, 0.3), (1, 1.0), (4, 1.0), (4, 0.55), (4, 0.5), (4, 0.2), (4, 1.2), (5, 0.2),
                  (28, 0.15), (48, 0.5), (48, 0.15), (64, 0.15), (8, 0.15)]:
        try:
            r = kr.ratio_schedule(L, ra)
            sched.append({"L": L, "r_avg": ra, "r": [float(x) for x in r]})
        except OracleError as e:
            sched.append({"L": L, "r_avg": ra, "error": e.kind})
    g["ratio_schedule"] = sched
    budgets = []
    for ratio, S in [(1.0, 8), (0.5, 8), (0.54368901, 8), (0.1, 3), (0.0, 5), (0.3333333333, 3),
                     (0.15, 1638), (0.9664, 1638), (1e-12, 7)]:
        budgets.append({"ratio": ratio, "S": S, "budget": kr.layer_budget(ratio, S)})
    g["layer_budget"] = budgets

    # -- converge known answers (test_recompute.cpp:110-247, acceptance.cpp:150-167)
    conv = []
    chain_q = [0.05, 0.10, 0.15, 0.70]
    chain_a = [[0, 0, 0, 0], [0.80, 0, 0, 0], [0, 0, 0, 0], [0.10, 0.75, 0.10, 0]]
    for name, q, a, b in [("hand_trace", chain_q, chain_a, 3), ("budget_one", chain_q, chain_a, 1),
                          ("zero_propagation", [0, 0, 0.4, 0], [[0] * 4] * 4, 3)]:
        order, hops = kr.converge(q, a, b)
        conv.append({"name": name, "qts": q, "sts": a, "budget": b, "order": order, "hops": hops})
    rng = PyRng(31337)
    for trial in range(200):
        S = 2 + rng.next_below(7)
        q = [0.0 if rng.next_below(4) == 0 else rng.next_double() for _ in range(S)]
        a = [[0.0] * S for _ in range(S)]
        for i in range(S):
            for j in range(i):
                a[i][j] = 0.0 if rng.next_below(3) == 0 else rng.next_double() / S
        b = 1 + rng.next_below(S)
        order, hops = kr.converge(q, a, b)
        conv.append({"name": f"random_{trial}", "qts": q, "sts": a, "budget": b, "order": order,
                     "hops": hops})
    # candidate-restricted walks and exact ties (lowest position wins)
    rng = PyRng(4242)
    for trial in range(60):
        S = 3 + rng.next_below(14)
        q = [0.0 if rng.next_below(3) == 0 else float(rng.next_below(4)) / 8 for _ in range(S)]
        a = [[0.0] * S for _ in range(S)]
        for i in range(S):
            for j in range(i):
                a[i][j] = 0.0 if rng.next_below(2) == 0 else float(rng.next_below(3)) / 16
        cand = [int(rng.next_below(3) != 0) for _ in range(S)]
        b = 1 + rng.next_below(S)
        lib_order, hops = kr.converge(q, a, b, cand)
        conv.append({"name": f"ties_cand_{trial}", "qts": q, "sts": a, "budget": b,
                     "candidates": cand, "order": lib_order, "hops": hops})
    g["converge"] = conv

    # -- per-instance plans, summaries, hidden states ---------------------------
    inst = []
    for s in ACCEPT_SEEDS:
        inst.append(instance_case(kr, s, 8, r_avg=0.5))
        inst.append(instance_case(kr, s, 8, r_avg=1.0))
    inst.append(instance_case(kr, 2, 8, r_avg=0.5, units=[[0, 4, 0], [4, 8, 0]]))  # witness
    for s in [60, 61, 62]:  # test_recompute.cpp:270-282
        inst.append(instance_case(kr, s, 6, r_avg=0.5))
    inst.append(instance_case(kr, 52, 4, sched=[1.0, 0.5, 0.25, 0.25]))
    # static groups: joint canonical KV sliced per member (harness.hpp:512-532, 659-677)
    inst.append(instance_case(kr, 31, 9, r_avg=0.5, units=[[0, 3, 1], [3, 4, 0], [4, 7, 1], [7, 9, 0]]))
    inst.append(instance_case(kr, 32, 6, r_avg=0.5, units=[[0, 6, 1]]))
    # single-hop ablation (recompute.hpp:166-176)
    for s in [2, 5, 9]:
        inst.append(instance_case(kr, s, 8, r_avg=0.5, multihop=False))
    # deeper / wider instances (longer walks, depth ties)
    inst.append(instance_case(kr, 101, 16, L=8, H=4, d=64, mlp=128, V=256, r_avg=0.3))
    inst.append(instance_case(kr, 102, 24, L=6, H=8, d=64, mlp=96, V=200, lo=3, hi=9, r_avg=0.5))
    inst.append(instance_case(kr, 103, 12, L=16, H=4, d=32, mlp=64, V=128, r_avg=0.25))
    inst.append(instance_case(kr, 104, 5, L=3, H=2, d=8, mlp=8, V=32, lo=2, hi=4, qlen=3, r_avg=0.5))
    inst.append(instance_case(kr, 105, 10, L=4, H=4, d=32, mlp=64, V=128, lo=1, hi=1, qlen=1, r_avg=0.5))
    g["instances"] = inst

    path = os.path.join(OUT, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print(f"wrote {path}: {len(inst)} instances, {len(conv)} converge cases,"
          f" {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
