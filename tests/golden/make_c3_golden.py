"""C3-width golden from the UNMODIFIED reference (oracle/_ref): the benchmark's
own memory and query at Qwen2.5-14B width, on the first two layers.

BASELINE.json configs[2] / SURVEY.md 8 "C3": L=48, H=40, d=5120, mlp=13824,
V=152064, the 16,280-token synthetic memory of bench.workload (S=1,638
segments, half of them in static groups of 8) and an 8-token query.  A full
48-layer reference run needs ~118 GB of RAM and days of one core, but the
reference's weights are counter-based per tensor name (model.hpp:54-73,
88-94), so a 2-layer model has exactly the 48-layer model's layers 0 and 1.
Running plan_keep (recompute.hpp:140-180) on it with r[0..1] of the 48-layer
ratio_schedule reproduces the 48-layer run's layer-0 summary, its layer-0 walk
(converge at budget layer_budget(r[1], S), ~847 hops) and the layer-1 plan.

Only the vocabulary is compacted: the embedding rows of the tokens that occur
(and the matching unembedding columns) are gathered from the full V=152064
Model::init, and the tokens are renumbered.  Rows of `embed` do not depend on
V (element e = row*d + col of the named stream), so every hidden state, KV row
and summary is unchanged (checked at toy width by --selfcheck).

The cached KV of every owner (segment_prefill per dynamic segment, one joint
full_prefill per static group: harness.hpp:512-532) is computed by the
reference in worker processes, one contiguous block of owners each: owners
are independent, so the split changes nothing.  The plan_keep call itself is
one single-threaded reference run (~2-3 h on one core).

    python tests/golden/make_c3_golden.py            # writes tests/golden/c3_width_golden.npz
    python tests/golden/make_c3_golden.py --selfcheck  # toy-width check of the method
"""
from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Problem, build  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

C3 = dict(L48=48, H=40, d=5120, mlp=13824, V=152064, S=1638, r_avg=0.5, seed=20250807)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def layout_of(S, V, seed):
    from paper_2602_23592_b200.synth import group_units, make_instance_layout
    inst = make_instance_layout(seed, S, V)
    units = [(u[0], u[1], 1 if u[2] == 1 else 0) for u in group_units(S, 8, 0.5)]
    return inst, units


def compact(w, L, d, mlp, V, tokens_all):
    """Gather the embedding rows / unembedding columns of the used tokens."""
    vocab = np.unique(tokens_all)
    Vc = len(vocab)
    emb = w[: V * d].reshape(V, d)[vocab]
    une = w[V * d: 2 * V * d].reshape(d, V)[:, vocab]
    rest = w[2 * V * d:]
    wc = np.concatenate([emb.ravel(), une.ravel(), rest])
    remap = {int(t): i for i, t in enumerate(vocab)}
    return wc, Vc, remap


_G = {}


def _canon_worker(args):
    (b, e) = args
    g = _G
    kr = Oracle("kr")
    seg_len = g["seg_len"][b:e]
    t0 = int(np.sum(g["seg_len"][:b]))
    t1 = t0 + int(np.sum(seg_len))
    units = [(ub - b, ue - b, ig) for (ub, ue, ig) in g["units"] if ub >= b and ue <= e]
    p = Problem(g["L"], g["H"], g["d"], g["mlp"], g["Vc"], g["seed"], seg_len, g["tokens"][t0:t1],
                np.zeros(0, np.int32), units)
    return b, e, kr.canonical_kv(p, g["w"])


def canonical_parallel(w, L, H, d, mlp, Vc, seed, seg_len, tokens, units, nproc):
    """Canonical KV [L][2][Tm][d] of all owners, computed by the reference in
    nproc workers over contiguous owner blocks (unit boundaries respected)."""
    S = len(seg_len)
    # cut points at unit boundaries, balanced by tokens
    bounds = sorted({u[0] for u in units} | {S})
    cuts = [0]
    tot = int(np.sum(seg_len))
    csum = np.concatenate([[0], np.cumsum(seg_len)])
    for k in range(1, nproc):
        target = tot * k / nproc
        best = min(bounds, key=lambda x: abs(csum[x] - target))
        if best > cuts[-1] and best < S:
            cuts.append(best)
    cuts.append(S)
    blocks = [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
    _G.update(dict(w=w, L=L, H=H, d=d, mlp=mlp, Vc=Vc, seed=seed, seg_len=np.asarray(seg_len, np.int32),
                   tokens=np.asarray(tokens, np.int32), units=units))
    Tm = tot
    out = np.empty((L, 2, Tm, d), np.float32)
    ctx = mp.get_context("fork")
    with ctx.Pool(len(blocks)) as pool:
        for b, e, kv in pool.imap_unordered(_canon_worker, blocks):
            r0, r1 = int(csum[b]), int(csum[e])
            out[:, :, r0:r1, :] = kv
            print(f"  canonical KV of segments [{b}, {e}) done ({time.strftime('%H:%M:%S')})", flush=True)
    return out


def walk_margins(qts, sts, order, budget):
    """Per hop of the reference walk: the chosen score and the runner-up's
    (relative gap), recomputed from the summary (recompute.hpp:94-126)."""
    S = len(qts)
    chosen = np.zeros(S, bool)
    colsum = np.zeros(S, np.float64)
    gaps = []
    for h, pick in enumerate(order):
        if h == 0:
            score = qts.copy()
        else:
            score = colsum / h
        score = np.where(chosen, -np.inf, score)
        best = score[pick]
        rest = np.delete(score, pick)
        second = np.max(rest) if len(rest) else -np.inf
        gaps.append(float((best - second) / abs(best)) if best != 0 else 0.0)
        chosen[pick] = True
        colsum += sts[pick]
    return np.array(gaps)


def run(cfg, L, nproc, out_path, selfcheck=False):
    build()
    kr = Oracle("kr")
    H, d, mlp, V, S, seed = cfg["H"], cfg["d"], cfg["mlp"], cfg["V"], cfg["S"], cfg["seed"]
    inst, units = layout_of(S, V, seed)
    r_full = kr.ratio_schedule(cfg["L48"], cfg["r_avg"])
    sched = np.ascontiguousarray(r_full[:L])
    t0 = time.time()
    w = kr.model_init(L, H, d, mlp, V, seed)
    print(f"Model::init {time.time() - t0:.1f}s", flush=True)
    wc, Vc, remap = compact(w, L, d, mlp, V, np.concatenate([inst.tokens, inst.query]))
    del w
    tok = np.array([remap[int(t)] for t in inst.tokens], np.int32)
    qry = np.array([remap[int(t)] for t in inst.query], np.int32)
    t0 = time.time()
    cached = canonical_parallel(wc, L, H, d, mlp, Vc, seed, inst.seg_len, tok, units, nproc)
    print(f"canonical KV {time.time() - t0:.1f}s", flush=True)
    p = Problem(L, H, d, mlp, Vc, seed, inst.seg_len, tok, qry, units)
    if selfcheck:
        # the method against a direct run: full vocabulary, canonical KV inside the shim
        ps = Problem(L, H, d, mlp, V, seed, inst.seg_len, inst.tokens, inst.query, units)
        wf = kr.model_init(L, H, d, mlp, V, seed)
        direct = kr.plan_keep(ps, wf, sched, kv=True)
        via = kr.plan_keep(p, wc, sched, cached=cached, kv=True)
        for k in ("plan", "hops", "qts", "sts", "final_hidden", "kv"):
            assert np.array_equal(direct[k], via[k]), k
        assert direct["orders"] == via["orders"]
        assert np.array_equal(kr.canonical_kv(ps, wf), cached)
        print("selfcheck ok: compact vocabulary + parallel canonical KV == direct reference run")
        return
    t0 = time.time()
    res = kr.plan_keep(p, wc, sched, cached=cached, kv=False)
    secs = time.time() - t0
    print(f"plan_keep {secs:.1f}s", flush=True)
    order0 = np.array(res["orders"][0] if res["orders"][0] is not None else [], np.int32)
    budget0 = kr.layer_budget(float(sched[1]), S)
    gaps = walk_margins(res["qts"][0], res["sts"][0], order0.tolist(), budget0)
    meta = {
        "generator": "tests/golden/make_c3_golden.py over oracle/_ref (unmodified reference headers)",
        "config": dict(cfg, L=L), "sched": [float(x) for x in sched], "budget_layer1": int(budget0),
        "S": S, "Tm": int(np.sum(inst.seg_len)), "T": int(np.sum(inst.seg_len)) + len(inst.query),
        "units": [list(u) for u in units], "compact_vocab": int(Vc), "plan_keep_seconds": secs,
        "orders_none": [o is None for o in res["orders"]],
        "hops": [int(x) for x in res["hops"]],
        "sts_sha": [sha(res["sts"][l]) for l in range(L)], "qts_sha": [sha(res["qts"][l]) for l in range(L)],
        "final_hidden_sha": sha(res["final_hidden"]), "cached_kv_sha": sha(cached),
        "walk0_min_rel_gap": float(np.min(gaps)) if len(gaps) else None,
        "walk0_gaps_below_1e-6": int(np.sum(gaps < 1e-6)), "walk0_gaps_below_1e-9": int(np.sum(gaps < 1e-9)),
    }
    np.savez_compressed(
        out_path, meta=np.frombuffer(json.dumps(meta).encode(), np.uint8),
        plan=res["plan"], order0=order0, hops=res["hops"], qts=res["qts"],
        sts0_rows=res["sts"][0][order0[:16]] if len(order0) else np.zeros((0, S)),
        sts0_rowsum=res["sts"][0].sum(axis=1), sts1_rowsum=res["sts"][1].sum(axis=1) if L > 1 else np.zeros(S),
        walk0_gaps=gaps, final_query_rows=res["final_hidden"][-len(inst.query):],
        final_rows_sample=res["final_hidden"][:: max(1, p.T // 64)],
        cached_rows_sample=cached[:, :, :: max(1, p.Tm // 32), :],
    )
    print(f"wrote {out_path}")
    print(json.dumps(meta)[:2000])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--selfcheck", action="store_true")
    ap.add_argument("--nproc", type=int, default=6)
    ap.add_argument("--out", default=os.path.join(OUT, "c3_width_golden.npz"))
    a = ap.parse_args()
    if a.selfcheck:
        run(dict(C3, H=4, d=32, mlp=64, V=300, S=40, L48=48), 2, 3, None, selfcheck=True)
        return
    run(C3, 2, a.nproc, a.out)


if __name__ == "__main__":
    main()
