#!/usr/bin/env python
"""KEEP per-layer memory prefill benchmark (TTFT + recomputed tokens/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full KEEP prefill (plan_keep: every layer's scoring, multi-hop
selection, gathered recompute, merged-KV assembly, plus the first-token
logits) over a 16K-token synthetic memory on Qwen2.5-14B dimensions
(BASELINE.json configs[2], SURVEY.md 8 "C3").  Prints one JSON line.

The headline runs the PARITY numerics -- the reference's own arithmetic
(fp32 storage, fp64-grade accumulation: Ozaki int8 tensor-core projections and
fp64 DMMA attention), whose plans, walk orders and hop counts are the
reference's (tests/test_gpu_parity.py, tests/test_gpu_c3_golden.py).  The bf16
FAST mode runs beside it on the same inputs (`other_mode`), with its
`selection_parity` against the headline (plans / walk orders / hops per layer
and the PARITY walk's decision margins).

  value    recomputed tokens/s = sum_l N_act(l) / TTFT, device-timed (CUDA
           events) with the memory KV resident in HBM.
  e2e      the same metric through the C ABI call with host buffers (token
           ids H2D, logits/plan D2H inside the timed region), host wall clock.
  updates  configs[2]'s "frequent dynamic-group updates": 35% of the dynamic
           owners refreshed in place inside the TTFT before each query.
The CPU baseline is the reference's own path (oracle/_ref, the unmodified
headers) timed on a bounded one-layer full-width sample on one host core and
extrapolated op-for-op to the same realised plan (the reference is
single-threaded; a full C3 run takes days).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: model dims, memory size in segments (8-12 tokens each), ratio
    "c1": dict(L=4, H=4, d=32, mlp=64, V=128, S=16, r_avg=0.5, desc="reference CPU default (example-config.json)"),
    "c2": dict(L=28, H=28, d=3584, mlp=18944, V=152064, S=410, r_avg=0.15,
               desc="Qwen2.5-7B dims, 4K-token memory, r_avg 0.15"),
    "c3": dict(L=48, H=40, d=5120, mlp=13824, V=152064, S=1638, r_avg=0.5,
               desc="Qwen2.5-14B dims, 16K-token memory, r_avg 0.5 (reference default, harness.hpp:57)"),
    "c4": dict(L=64, H=40, d=5120, mlp=27648, V=152064, S=3276, r_avg=0.15,
               desc="Qwen2.5-32B dims, 32K-token memory, r_avg 0.15 (BASELINE configs[3], here on one GPU)"),
    "c5": dict(L=64, H=40, d=5120, mlp=27648, V=152064, S=13107, r_avg=0.15,
               desc="Qwen2.5-32B dims, 128K-token memory bank in pinned host DRAM, batch of 16 planning queries "
                    "(BASELINE configs[4])"),
}
METRIC = "memory-prefill TTFT (ms) and recomputed tokens/s, 16K-token memory, 1/2/4/8 B200"
UNIT = "recomputed tokens/s"



def _finite(o):
    """Strict JSON: non-finite floats become null."""
    if isinstance(o, float) and not math.isfinite(o):
        return None
    if isinstance(o, dict):
        return {k: _finite(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [_finite(v) for v in o]
    return o

def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6], float(parts[6])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        sm = [r[0] for r in rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(r[3] for r in rows)}


DETAIL = {}  # per kernel: the captured ncu launches behind `traffic`


def ncu_traffic():
    """Per-launch DRAM traffic (read + write bytes) of the kernels captured by
    the committed `ncu --set full` summaries (profiles/, tools/ncu_summary.py),
    averaged over the captured launches of each kernel."""
    import csv
    import glob
    out = {}
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu*full*.csv")))
    if not files:
        return out
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc, detail = {}, {}
    for fn in files:
        with open(fn) as f:
            rows = list(csv.DictReader(f))
        for r in rows:
            name = r["kernel"].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            tot = 0.0
            for k, v in r.items():
                if k.startswith("dram__bytes_read.sum [") or k.startswith("dram__bytes_write.sum ["):
                    if v:
                        tot += float(v) * scale.get(k.split("[")[1].rstrip("]"), 1.0)
            if not math.isfinite(tot):  # a launch ncu could not measure (replay limits)
                continue
            acc.setdefault(name, []).append(tot)
            det = detail.setdefault(name, {"launches": 0, "ms": 0.0, "dram_pct": 0.0})
            det["launches"] += 1
            for k, v in r.items():
                if v and k.startswith("gpu__time_duration.sum ["):
                    det["ms"] += float(v) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(k.split("[")[1].rstrip("]"), 1.0)
                if v and k.startswith("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):
                    det["dram_pct"] += float(v)
    for k, det in detail.items():
        n = max(det["launches"], 1)
        DETAIL[k] = {"captured_launches": det["launches"], "mean_ms": det["ms"] / n,
                     "mean_dram_pct_of_peak": det["dram_pct"] / n,
                     "mean_dram_bytes": sum(acc[k]) / len(acc[k]) if acc.get(k) else None}
    return {k: sum(v) / len(v) for k, v in acc.items() if v}


def numerics_for(args, cfg):
    """PARITY (the reference's arithmetic; bit-exact selections) is the
    headline; FAST (bf16 tensor cores) needs model / MLP widths in multiples
    of 64 and reports its selection agreement beside it."""
    import paper_2602_23592_b200 as kb
    if args.numerics == "exact":
        return kb.PARITY_EXACT
    if args.numerics == "parity" or cfg["d"] % 64 or cfg["mlp"] % 64:
        return kb.PARITY
    return kb.FAST


def workload(cfg, seed):
    import paper_2602_23592_b200 as kb
    from paper_2602_23592_b200.synth import group_units, make_instance_layout
    inst = make_instance_layout(seed, cfg["S"], cfg["V"])
    # static/dynamic memory layout: half the memory in static groups of 8
    # segments (joint KV), half dynamic per-segment owners
    units = group_units(cfg["S"], 8, 0.5)
    return kb.Layout(inst.seg_len, inst.tokens, units), inst.query


def attention_pairs(layout, qlen, plan):
    """sum over computed rows of visible keys (t + 1), per layer."""
    seg_len = np.asarray(layout.seg_len, np.int64)
    starts = np.concatenate([[0], np.cumsum(seg_len)])
    Tm = int(starts[-1])
    out = []
    for l in range(plan.shape[0]):
        act = plan[l].astype(bool)
        b, e = starts[:-1][act], starts[1:][act]
        s = float(np.sum((e * (e + 1) - b * (b + 1)) // 2))  # sum_{t=b}^{e-1} (t+1)
        s += float(sum(Tm + k + 1 for k in range(qlen)))
        out.append(s)
    return np.array(out)


# ------------------------------------------------------------------ CPU arm --
PLAN_FIXTURE = os.path.join(ROOT, "tests", "golden", "{}_realized_plan.json")


def host_cpu():
    """Model name and logical core count of this host (stated beside the CPU baseline)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def plan_from_fixture(name, S, L):
    """The realised plan of the workload as the GPU arm's PARITY run produced
    it (tests/golden/c3_realized_plan.json, written by tools/c3_parity.py):
    runs of layers sharing one segment set.  None if the fixture is absent."""
    try:
        with open(PLAN_FIXTURE.format(name)) as f:
            fx = json.load(f)
    except OSError:
        return None
    if fx.get("config") != name or fx.get("S") != S or fx.get("L") != L:
        return None
    plan = np.zeros((L, S), np.uint8)
    for l0, l1, segs in fx["runs"]:
        plan[l0:l1, segs] = 1
    return plan


_W_CACHE = {}


def cpu_sample(cfg, seed=7, sample_segments=2):
    """Time the reference's own path (plan_keep: PrefillCursor::step +
    converge, recompute.hpp:140-180) for ONE layer at the workload's full width
    on a small layout, on one host core (the reference is single-threaded).
    Weights come from the reference's Model::init (model.hpp:54-73); the
    layer's tensors are the same named streams as the workload model's.
    Returns the measured fp64-accumulate MAC rate and what was sampled."""
    from oracle.oracle import Oracle, available, Problem
    kind = "reference" if available("kr") else "port"
    orc = Oracle("kr" if kind == "reference" else "ko")
    L1, H, d, mlp = 1, cfg["H"], cfg["d"], cfg["mlp"]
    V = 1024  # the vocabulary only feeds the embedding gather in a step
    key = (kind, L1, H, d, mlp, V, seed)
    if key not in _W_CACHE:
        _W_CACHE[key] = orc.model_init(L1, H, d, mlp, V, seed)
    w = _W_CACHE[key]
    from paper_2602_23592_b200.synth import make_instance_layout
    inst = make_instance_layout(seed, sample_segments, V)
    p = Problem(L1, H, d, mlp, V, seed, inst.seg_len, inst.tokens, inst.query)
    T = p.T
    cached = np.zeros((L1, 2, p.Tm, d), np.float32)
    t0 = time.perf_counter()
    orc.plan_keep(p, w, np.ones(1), cached=cached)
    dt = time.perf_counter() - t0
    macs = T * (4.0 * d * d + 2.0 * d * mlp) + 2.0 * d * T * (T + 1) / 2.0
    return {"kind": kind, "seconds": dt, "macs": macs, "rate": macs / dt, "rows": T,
            "sample": f"reference plan_keep (oracle/_ref: the unmodified headers, -O2) for one layer at full width "
                      f"(d={d}, H={H}, mlp={mlp}; Model::init weights) over {T} rows ({sample_segments} segments + "
                      f"{len(inst.query)}-token query), V reduced to {V}; 1 host core; extrapolated op-for-op to the "
                      f"workload's realised plan"}


def cpu_extrapolate(sample, cfg, rows_per_layer, pairs_per_layer):
    d, mlp = cfg["d"], cfg["mlp"]
    macs = float(np.sum(rows_per_layer)) * (4.0 * d * d + 2.0 * d * mlp) + 2.0 * d * float(np.sum(pairs_per_layer))
    ttft_s = macs / sample["rate"]
    return {"ttft_s": ttft_s, "tokens_per_s": float(np.sum(rows_per_layer)) / ttft_s}


def workload_config(args, cfg, layout, query, world, numerics_name):
    """The config object both arms print (identical: same workload, metric, plan)."""
    return {"workload": args.config, "desc": cfg["desc"], "L": cfg["L"], "H": cfg["H"], "d": cfg["d"],
            "mlp": cfg["mlp"], "V": cfg["V"], "S": layout.S, "T": int(np.sum(layout.seg_len)) + len(query),
            "units": {"static_groups_of_8": sum(1 for u in layout.units if u[2] == 1),
                      "dynamic_segments": sum(1 for u in layout.units if u[2] == 0)},
            "r_avg": cfg["r_avg"], "seed": args.seed, "query_len": len(query),
            "parallelism": f"KV-head sharded x{world} (NCCL)" if world > 1 else "1 GPU",
            "memory_kv": ("pinned-host canonical KV, layer-balanced K10 loader" if args.memory == "host" else
                          "HBM-resident canonical KV (static groups joint, dynamic per segment)"),
            "l2": "inputs larger than L2 (fp32 weights {:.1f} GB + memory KV {:.1f} GB read per step)".format(
                4e-9 * cfg["L"] * (4 * cfg["d"] ** 2 + 2 * cfg["d"] * cfg["mlp"]),
                8e-9 * cfg["L"] * cfg["d"] * int(np.sum(layout.seg_len)))}


def run_reference(args, cfg):
    """The reference's own CPU implementation of the path (oracle/_ref, the
    unmodified headers) on this host: the same workload and realised plan as
    the GPU arm.  Only oracle/ and the pure-Python synthetic generator are
    touched -- the product library is never loaded."""
    from oracle.oracle import Oracle, available
    orc = Oracle("kr" if available("kr") else "ko")
    layout, query = workload(cfg, args.seed)
    r = orc.ratio_schedule(cfg["L"], cfg["r_avg"])
    plan = plan_from_fixture(args.config, layout.S, cfg["L"])
    plan_model = f"realised plan of the GPU PARITY run (tests/golden/{args.config}_realized_plan.json)"
    if plan is None:  # no fixture for this config: every budget fully realised (an upper bound)
        plan = np.zeros((cfg["L"], layout.S), np.uint8)
        for l in range(cfg["L"]):
            b = layout.S if l == 0 else min(layout.S, orc.layer_budget(float(r[l]), layout.S))
            plan[l, :b] = 1
        plan_model = "budgets fully realised (no plan fixture for this config)"
    seg_len = np.asarray(layout.seg_len)
    rows = plan.astype(np.int64) @ seg_len + len(query)
    pairs = attention_pairs(layout, len(query), plan)
    for _ in range(args.warmup):
        cpu_sample(cfg)
    vals = []
    t0 = time.perf_counter()
    s = None
    for _ in range(args.steps):
        s = cpu_sample(cfg)
        vals.append(cpu_extrapolate(s, cfg, rows, pairs))
    wall = time.perf_counter() - t0
    v = float(np.median([x["tokens_per_s"] for x in vals]))
    ttft = float(np.median([x["ttft_s"] for x in vals])) * 1e3
    conf = workload_config(args, cfg, layout, query, 1, "reference")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / max(args.steps, 1) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32-store/f64-acc",
            "data": "synthetic", "ttft_ms": ttft, "config": conf,
            "plan_model": plan_model, "recomputed_tokens_per_step": float(np.sum(rows)),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": s["kind"], "sample": s["sample"],
                             "host_cpu": host_cpu(), "ttft_ms_extrapolated": ttft},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(_finite(line)), flush=True)


# -------------------------------------------------- selection parity (FAST) --
def walk_margins(qts, sts, order, cand):
    """Per hop of a converge walk (recompute.hpp:94-126): relative gap between
    the chosen score and the best other allowed candidate (inf: no rival)."""
    S = len(qts)
    allowed = np.asarray(cand, bool).copy()
    colsum = np.zeros(S, np.float64)
    gaps = []
    for h, pick in enumerate(order):
        score = qts if h == 0 else colsum / h
        ok = allowed & (score > 0)
        ok[pick] = False
        best = score[pick]
        second = float(np.max(score[ok])) if ok.any() else -np.inf
        gaps.append(float((best - second) / abs(best)) if best != 0 and np.isfinite(second) else float("inf"))
        allowed[pick] = False
        colsum += sts[pick]
    return np.array(gaps)


def selection_parity(ref, other, summaries):
    """Compare another numerics mode's plan_keep with the headline (PARITY)
    one on the same inputs: plans, walk orders and hops per layer, and the
    PARITY walk's decision margins (bf16 can only flip near-ties)."""
    L = ref["plan"].shape[0]
    plans_eq = [bool(np.array_equal(ref["plan"][l], other["plan"][l])) for l in range(L)]
    orders_eq = [ref["orders"][l] == other["orders"][l] for l in range(L)]
    walks = [l for l in range(L) if ref["orders"][l] is not None]
    per_walk = []
    for l in walks:
        cand = ref["plan"][l].astype(bool)
        g = walk_margins(summaries["qts"][l], summaries["sts"][l], ref["orders"][l], cand)
        o, f = ref["orders"][l], other["orders"][l] or []
        first = next((i for i in range(min(len(o), len(f))) if o[i] != f[i]), None)
        if first is None and len(o) != len(f):
            first = min(len(o), len(f))
        per_walk.append({"layer": l, "hops": len(o), "orders_equal": o == f, "first_differing_hop": first,
                         "margin_at_first_difference": (float(g[first]) if first is not None and first < len(g)
                                                        else None),
                         "min_rel_margin": float(np.min(g)) if len(g) else None,
                         "decisions_below_1e-6": int(np.sum(g < 1e-6)), "decisions_below_1e-3": int(np.sum(g < 1e-3))})
    return {"layers": L, "plans_equal": int(sum(plans_eq)), "orders_equal": int(sum(orders_eq)),
            "hops_equal": bool(np.array_equal(ref["hops"], other["hops"])),
            "plan_layers_differing": [l for l in range(L) if not plans_eq[l]],
            "order_layers_differing": [l for l in range(L) if not orders_eq[l]],
            "walks": per_walk}


# ------------------------------------------------------------------ GPU arm --
def gpu_context(args, cfg, numerics, world, dev):
    import paper_2602_23592_b200 as kb
    L, H, d, mlp, V = cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"]
    if world > 1:
        # KV-head sharding: one context per rank over the library's own NCCL
        # communicator (torch.distributed only carries its unique id)
        from paper_2602_23592_b200.dist import sharded_context
        return sharded_context(L, H, d, mlp, V, args.seed, numerics, device=dev)
    return kb.Context(L, H, d, mlp, V, args.seed, numerics, device=dev)


def run_ours(args, cfg, rank, world, dist):
    import torch

    import paper_2602_23592_b200 as kb
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    numerics = numerics_for(args, cfg)
    parity = numerics == kb.PARITY
    L, H, d, mlp, V = cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"]
    layout, query = workload(cfg, args.seed)
    r = kb.ratio_schedule(L, cfg["r_avg"])
    t0 = time.perf_counter()
    ctx = gpu_context(args, cfg, numerics, world, dev)
    ctx.model_init()
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    host_mem = args.memory == "host"
    tier = kb.TIER_HOST if host_mem else kb.TIER_DEVICE
    ctx.memory_compute_layout(layout, version=1, tier=tier)
    resident = 0
    if host_mem and args.hbm_budget_gb > 0:
        # the capacity-bounded fast tier: the deepest layers also in HBM
        resident = ctx.memory_residency(int(args.hbm_budget_gb * 1e9))
    t_mem = time.perf_counter() - t0

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        return ctx.plan_keep(layout, query, r, final_hidden=False)

    for _ in range(args.warmup):
        step()
    ctx.profile_read(reset=True)
    barrier()
    steps = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            steps.append(step())
    barrier()
    ttft = np.array([s["ttft_ms"] for s in steps])
    tokens = float(np.sum(steps[-1]["rows_per_layer"]))
    total_ms = float(np.sum(ttft))
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # one prefill per step for the whole job (heads split across the ranks)
    value = tokens * args.steps / (total_ms / 1e3)

    # per-phase device times (roofline, phase shares) from separate profiled
    # steps: the per-phase events are a measurement artefact kept out of the
    # timed steps above
    n_prof = 1 if parity else max(1, min(args.steps, 3))
    ctx.profile_enable(True)
    for _ in range(n_prof):
        step()
    ctx.profile_enable(False)
    prof = ctx.profile_read(reset=True)

    # e2e: the C-ABI call with host buffers (token ids in, plan / walk orders /
    # logits out), host wall clock
    n_e2e = max(1, min(args.steps, 3 if parity else args.steps))
    e2e_s = []
    for _ in range(n_e2e):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = step()
        e2e_s.append(time.perf_counter() - t0)
    e2e_mean = float(np.mean(e2e_s))
    if dist is not None:
        t = torch.tensor([e2e_mean], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_mean = float(t.item())
    e2e_val = tokens / e2e_mean
    h2d = 4 * (len(layout.tokens) + len(query) + layout.S + 3 * len(layout.units) + L)
    d2h = 8 * V + L * layout.S * (1 + 4) + 4 * 2 * L + 8 * 2 * L

    # configs[2] "with frequent dynamic-group updates": before each query a
    # fraction of the dynamic owners was updated and is refreshed in place
    # inside the TTFT (harness.hpp:609-628; 0.35 as test_harness.cpp:266-268)
    updates = None
    if args.updates > 0 and world == 1:
        owners_all = layout.owners()
        dyn = [i for i, o in enumerate(owners_all) if o[0] == kb.SEGMENT]
        owner_tokens = [int(np.sum(layout.seg_len[o[2]:o[3]])) for o in owners_all]
        upd_rng = np.random.default_rng(args.seed + 1)
        version = 1
        u_ttft, u_tok, u_ref = [], [], []
        for i in range(1 + args.update_steps):
            version += 1
            pick = [u for u in dyn if upd_rng.random() < args.updates]
            ctx.profile_read(reset=True)
            ctx.profile_enable(True)
            ctx.memory_refresh(layout, pick, version, tier=tier)
            ctx.profile_enable(False)
            ref_ms = ctx.profile_read(reset=True)["refresh"]["ms"]
            res_u = step()
            if i == 0:
                continue  # (first: warm-up of the refresh workspace)
            u_ttft.append(res_u["ttft_ms"] + ref_ms)
            u_ref.append(ref_ms)
            u_tok.append(float(np.sum(res_u["rows_per_layer"])) + L * float(sum(owner_tokens[u] for u in pick)))
        updates = {"fraction_of_dynamic_owners": args.updates, "steps": args.update_steps,
                   "ttft_ms": float(np.mean(u_ttft)), "refresh_ms_per_step": float(np.mean(u_ref)),
                   "recomputed_tokens_per_step": float(np.mean(u_tok)),
                   "value": float(np.mean(u_tok)) / (float(np.mean(u_ttft)) / 1e3), "unit": UNIT,
                   "note": "the refreshed owners' canonical KV (all layers) is recomputed in place before the query; "
                           "its device time is part of the TTFT and its rows of the recomputed tokens"}

    pk, src = peaks()
    extra = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_peaks_int8_fp64.json")) as f:
            extra = json.load(f)
    except OSError:
        pass
    gemm_phases = ["qkv", "wo", "mlp_in", "mlp_out"]
    g_ms = sum(prof[p]["ms"] for p in gemm_phases)
    g_fl = sum(prof[p]["flops"] for p in gemm_phases)
    g_by = sum(prof[p]["bytes"] for p in gemm_phases)
    g_n = sum(prof[p]["launches"] for p in gemm_phases)
    a_ms, a_fl = prof["attn"]["ms"], prof["attn"]["flops"]
    phase_ms = {k: round(v["ms"] / n_prof, 3) for k, v in prof.items() if v["ms"] > 0}
    traffic = ncu_traffic()
    if parity:
        moduli = int(os.environ.get("KEEP_OZ_MODULI", "14"))
        i8_peak = extra.get("int8_tops_sustained") or 2 * pk["bf16_tflops_sustained"]
        g_ach = g_fl * moduli / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
        gemm_roof = {"kernel": "gemm_oz_kernel (Ozaki-II int8 tcgen05 kind::i8, CRT residues, Garner + fp64 Horner epilogue)", "bound": "tensor",
                     "achieved": g_ach, "peak": i8_peak, "unit": "TOP/s (int8)", "frac": g_ach / i8_peak,
                     "traffic": traffic.get("gemm_oz_kernel"), "traffic_launches": DETAIL.get("gemm_oz_kernel"),
                     "peak_source": "measured int8 sustained (profiles/r02_peaks_int8_fp64.json: cuBLASLt "
                                    "torch._int_mm 8192^3)" if extra else "2 x measured bf16 sustained",
                     "algorithmic": f"2*M*N*K per projection x {moduli} moduli (one exact int8 GEMM per CRT residue); "
                                    f"phase includes the residue splits and the few-row DFMA weight stream",
                     "fp64_equivalent_tflops": g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0,
                     "per_launch_ms": g_ms / max(g_n, 1)}
        fp64_peak = extra.get("fp64_dmma_tflops") or 37.0
        a_ach = a_fl / (a_ms / 1e3) / 1e12 if a_ms > 0 else 0.0
        attn_roof = {"kernel": "attn_dmma16_flash_kernel (K5 flash pass, mma.m16n8k16.f64) + attn_dmma_ws_kernel "
                               "(summary layers: context pass with the bins fused as E.Z, one pass when the "
                               "Cauchy-Schwarz bound admits it)", "bound": "tensor",
                     "achieved": a_ach, "peak": fp64_peak, "unit": "TFLOP/s (fp64)", "frac": a_ach / fp64_peak,
                     "traffic": traffic.get("attn_dmma16_flash_kernel"),
                     "traffic_launches": DETAIL.get("attn_dmma16_flash_kernel"),
                     "peak_source": "measured fp64 DMMA (tools/micro/fp64_peak.cu)",
                     "note": "algorithmic FLOPs 4*d*sum(t+1) (QK^T + PV once) over the whole attention phase; "
                             "a summary layer outside the one-pass bound adds a max pass (Q.K^T once more); "
                             "traffic = ncu DRAM bytes of one C3 "
                             "layer-1 flash launch (profiles/r02_ncu_dmma16_full.csv)"}
        roofs = [gemm_roof, attn_roof]
    else:
        tensor_peak = pk["bf16_tflops_sustained"]
        g_ach = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
        a_ach = a_fl / (a_ms / 1e3) / 1e12 if a_ms > 0 else 0.0
        gemm_roof = {"kernel": "gemm_tc_kernel (tcgen05 bf16, fused epilogues)", "bound": "tensor", "achieved": g_ach,
                     "peak": tensor_peak, "unit": "TFLOP/s", "frac": g_ach / tensor_peak,
                     "traffic": traffic.get("gemm_tc_kernel"), "peak_source": src + " (bf16 sustained)",
                     "per_launch_ms": g_ms / max(g_n, 1), "algorithmic_bytes_per_launch": g_by / max(g_n, 1),
                     "traffic_launches": DETAIL.get("gemm_tc_kernel")}
        attn_roof = {"kernel": "attn_tc2_kernel STATS + CTX / FLASH (K5, tcgen05, summary bins on the tensor core)",
                     "bound": "tensor", "achieved": a_ach, "peak": tensor_peak, "unit": "TFLOP/s",
                     "frac": a_ach / tensor_peak, "traffic": traffic.get("attn_tc2_kernel"), "peak_source": src,
                     "note": "algorithmic FLOPs 4*d*sum(t+1) (QK^T + PV once)"}
        roofs = [gemm_roof, attn_roof]
        d_ms, d_by, d_n = prof["attn_decode"]["ms"], prof["attn_decode"]["bytes"], prof["attn_decode"]["launches"]
        if d_ms > 0:
            d_ach = d_by / (d_ms / 1e3) / 1e9
            roofs.append({"kernel": "attn_decode_kernel (K5d, split-K flash decoding, TMA stages)", "bound": "hbm",
                          "achieved": d_ach, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": d_ach / pk["hbm_gbs"],
                          "traffic": traffic.get("attn_decode_kernel"), "peak_source": src,
                          "per_launch_ms": d_ms / max(d_n, 1), "algorithmic_bytes_per_launch": d_by / max(d_n, 1)})
    roof = gemm_roof if g_ms >= a_ms else attn_roof
    launches = int(sum(v["kernels"] for v in prof.values())) // n_prof
    loader_info = None
    if host_mem:
        tr = ctx.loader_trace()
        h2d_kv = float(sum(x["bytes"] for x in tr))
        ms = prof["loader"]["ms"] / n_prof
        h2d += h2d_kv  # the memory KV crosses PCIe inside every step
        loader_info = {"h2d_bytes_per_step": h2d_kv, "copy_ms_per_step": ms,
                       "hbm_resident_bytes": resident, "hbm_budget_gb": args.hbm_budget_gb,
                       "h2d_gbs": h2d_kv / (ms * 1e6) if ms > 0 else None,
                       "items": len(tr), "preloads": sum(1 for x in tr if x["kind"] == "preload"),
                       "urgent": sum(1 for x in tr if x["kind"] == "urgent")}

    # selections of the other numerics modes on the same inputs (SURVEY.md
    # 0.1(2): a bf16 mode must report its agreement and the decision margins;
    # PARITY_EXACT -- bit-exact projections, reference-order scores -- is the
    # arbiter of the tensor-core PARITY mode)
    sel, other_mode, exact_mode = None, None, None
    if world == 1 and not args.no_compare and parity and cfg["d"] % 64 == 0 and cfg["mlp"] % 64 == 0:
        head = ctx.plan_keep(layout, query, r, final_hidden=True, summaries=True)
        summ = {"qts": head.pop("qts"), "sts": head.pop("sts")}
        hq = head["final_hidden"][-len(query):].astype(np.float64)
        ctx.close()
        ctx = None
        torch.cuda.synchronize()

        def run_mode(mode, n):
            c2 = kb.Context(L, H, d, mlp, V, args.seed, mode, device=dev)
            c2.model_init()
            c2.memory_compute_layout(layout, version=1, tier=tier)
            c2.plan_keep(layout, query, r, final_hidden=False)
            outs = [c2.plan_keep(layout, query, r, final_hidden=True) for _ in range(n)]
            c2.close()
            torch.cuda.synchronize()
            return outs

        def hidden_rel(o):
            oq = o["final_hidden"][-len(query):].astype(np.float64)
            return float(np.max(np.abs(oq - hq)) / max(float(np.max(np.abs(oq))), 1e-300))

        o_steps = run_mode(kb.FAST, 3)
        ores = o_steps[-1]
        o_ttft = float(np.median([x["ttft_ms"] for x in o_steps]))
        sel = selection_parity(head, ores, summ)
        other_mode = {"numerics": "fast (bf16 tcgen05)", "ttft_ms": o_ttft,
                      "value": float(np.sum(ores["rows_per_layer"])) / (o_ttft / 1e3), "unit": UNIT,
                      "plan_segments_per_layer": [int(x) for x in ores["plan"].sum(1)],
                      "selections_identical_to_parity": (sel["plans_equal"] == L and sel["orders_equal"] == L
                                                         and sel["hops_equal"]),
                      "query_rows_rel_diff_vs_parity": hidden_rel(ores),
                      "logits_top1_equal": bool(np.argmax(ores["last_logits"]) == np.argmax(head["last_logits"]))}
        if not args.no_exact:
            e_res = run_mode(kb.PARITY_EXACT, 1)[-1]
            se = selection_parity(e_res, head, summ)
            exact_mode = {"numerics": "parity_exact (DFMA projections bit-exact with vec_mat, scalar fp64 attention "
                                      "in the reference's dimension order)", "ttft_ms": e_res["ttft_ms"],
                          "plans_equal": se["plans_equal"], "orders_equal": se["orders_equal"],
                          "hops_equal": se["hops_equal"], "layers": L,
                          "selections_identical": (se["plans_equal"] == L and se["orders_equal"] == L
                                                   and se["hops_equal"]),
                          "query_rows_rel_diff": hidden_rel(e_res),
                          "logits_top1_equal": bool(np.argmax(e_res["last_logits"]) == np.argmax(head["last_logits"])),
                          "note": "without norms the reference's deep layers are one-hot (|logit| ~ 1e18, fp64 ulp "
                                  "~ 1e2): any re-ordered fp64 sum can move a deep attention pick, so the final hidden "
                                  "state of the tensor-core mode may differ while every selection stays identical"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        s = cpu_sample(cfg)
        plan = steps[-1]["plan"]
        ex = cpu_extrapolate(s, cfg, steps[-1]["rows_per_layer"], attention_pairs(layout, len(query), plan))
        cpu = {"value": ex["tokens_per_s"], "unit": UNIT, "cores": 1, "kind": s["kind"], "sample": s["sample"],
               "host_cpu": host_cpu(), "ttft_ms_extrapolated": ex["ttft_s"] * 1e3, "sample_seconds": s["seconds"]}

    if rank == 0:
        plan = steps[-1]["plan"]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32-store/f64-acc" if parity else "bf16", "data": "synthetic",
            "numerics": ("parity: fp32 storage, fp64-grade accumulation (Ozaki int8 tcgen05 projections, "
                         "fp64 DMMA attention) -- the reference's arithmetic (tensor.hpp:31-47)" if parity else
                         "fast: bf16 tcgen05, fp32 accumulation (selections NOT guaranteed bit-exact)"),
            "ttft_ms": float(np.median(ttft)), "ttft_ms_min": float(np.min(ttft)),
            "config": workload_config(args, cfg, layout, query, world, "parity" if parity else "fast"),
            "recomputed_tokens_per_step": tokens,
            "plan_segments_per_layer": [int(x) for x in plan.sum(1)],
            "rows_per_layer": [int(x) for x in steps[-1]["rows_per_layer"]],
            "hops_per_layer": [int(x) for x in steps[-1]["hops"]],
            "phase_ms_per_step": phase_ms,
            "setup_s": {"model_init": t_init, "canonical_kv_refresh": t_mem},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ttft_ms": e2e_mean * 1e3, "steps": n_e2e},
            "gpu_launches": launches,
            "updates": updates,
            "selection_parity": sel,
            "other_mode": other_mode,
            "exact_mode": exact_mode,
            "loader": loader_info,
            "roofline": roof,
            "roofline_kernels": roofs,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(_finite(line)), flush=True)
    if ctx is not None:
        ctx.close()


def run_batch(args, cfg):
    """--batch B: B concurrent planning queries over one memory layout through
    keep_plan_keep_batch (BASELINE configs[4]'s batch of 16; here with the
    memory KV in HBM), against the same B queries one plan_keep at a time."""
    import torch

    import paper_2602_23592_b200 as kb
    torch.cuda.set_device(0)
    numerics = numerics_for(args, cfg)
    L, H, d, mlp, V = cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"]
    layout, query = workload(cfg, args.seed)
    r = kb.ratio_schedule(L, cfg["r_avg"])
    B = args.batch
    rng = np.random.default_rng(args.seed + 17)
    Q = rng.integers(0, V, size=(B, len(query))).astype(np.int32)
    Q[0] = query
    ctx = kb.Context(L, H, d, mlp, V, args.seed, numerics)
    ctx.model_init()
    host_mem = args.memory == "host"
    resident = 0
    if host_mem and args.hbm_budget_gb > 0:
        # the fast tier: the deepest layers of the new pinned-host memory are
        # computed straight into HBM (they never occupy host DRAM)
        ctx.memory_residency(int(args.hbm_budget_gb * 1e9))
    t0 = time.perf_counter()
    ctx.memory_compute_layout(layout, tier=kb.TIER_HOST if host_mem else kb.TIER_DEVICE)
    t_mem = time.perf_counter() - t0
    mem_st = ctx.memory_stats()
    mem_st["hbm_free_after_memory_bytes"] = int(torch.cuda.mem_get_info()[0])
    print(f"# memory KV: host {mem_st['host_bytes'] / 1e9:.1f} GB, device {mem_st['device_bytes'] / 1e9:.1f} GB, "
          f"HBM free {mem_st['hbm_free_after_memory_bytes'] / 1e9:.1f} GB, setup {t_mem:.1f} s", file=sys.stderr, flush=True)
    sb = args.sub_batch if args.sub_batch > 0 else B

    def batch_step():
        # B queries as ceil(B / sb) sub-batches of one plan_keep_batch each
        outs, ms = [], 0.0
        for q0 in range(0, B, sb):
            o = ctx.plan_keep_batch(layout, Q[q0:q0 + sb], r)
            ms += o[0]["ttft_ms"]
            outs += o
        for o in outs:
            o["batch_ms"] = ms
        return outs

    for _ in range(args.warmup):
        batch_step()
    torch.cuda.synchronize()
    res = []
    dev = torch.cuda.current_device()
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            res.append(batch_step())
    torch.cuda.synchronize()
    # per-phase times from one separate profiled batch (kept out of the timed steps)
    ctx.profile_read(reset=True)
    ctx.profile_enable(True)
    batch_step()
    ctx.profile_enable(False)
    prof = ctx.profile_read(reset=True)
    n_prof = 1
    batch_ms = np.array([x[0]["batch_ms"] for x in res])
    tokens = float(sum(np.sum(o["rows_per_layer"]) for o in res[-1]))
    value = tokens / (float(np.mean(batch_ms)) / 1e3)
    # e2e: host query ids in, host plans + logits out, wall clock
    e2e = []
    for _ in range(max(1, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        batch_step()
        e2e.append(time.perf_counter() - t0)
    st_b = ctx.memory_stats()["bytes_loaded_slow"]
    batch_step()
    h2d_batch = ctx.memory_stats()["bytes_loaded_slow"] - st_b
    # the same queries one at a time (the batch workspace released first)
    seq_ms, same = None, None
    if not args.no_sequential:
        ctx.trim()
        for b in range(min(B, 2)):
            ctx.plan_keep(layout, Q[b], r, final_hidden=False)
        seq = [ctx.plan_keep(layout, Q[b], r, final_hidden=False) for b in range(B)]
        seq_ms = float(sum(x["ttft_ms"] for x in seq))
        same = [bool(np.array_equal(res[-1][b]["plan"], seq[b]["plan"])) for b in range(B)]
    line = {
        "metric": METRIC + " -- batched planning queries", "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(batch_ms)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16" if numerics == kb.FAST else "f32-store/f64-acc", "data": "synthetic",
        "config": {"workload": args.config + f"-batch{B}" + ("-hostmem" if host_mem else ""), "desc": cfg["desc"],
                   "S": layout.S, "batch": B, "query_len": len(query),
                   "memory": "pinned host DRAM, one staged layer sheet per layer for the batch" if host_mem else "hbm",
                   "l2": "inputs > L2 ({:.1f} GB memory KV)".format(4e-9 * L * d * int(np.sum(layout.seg_len)))},
        "batch": {"batch_ttft_ms": float(np.median(batch_ms)), "sequential_ttft_ms_sum": seq_ms,
                  "speedup_vs_sequential": seq_ms / float(np.median(batch_ms)) if seq_ms else None,
                  "plans_equal_to_sequential": same, "sub_batch": sb,
                  "memory": {"host_bytes": mem_st["host_bytes"], "device_bytes": mem_st["device_bytes"],
                             "hbm_free_after_memory_bytes": mem_st["hbm_free_after_memory_bytes"],
                             "hbm_budget_gb": args.hbm_budget_gb, "canonical_kv_setup_s": t_mem},
                  "plan_segments_per_layer_q0": [int(x) for x in res[-1][0]["plan"].sum(axis=1)],
                  "recomputed_tokens_per_batch": tokens, "h2d_memory_bytes_per_batch": int(h2d_batch)},
        "phase_ms_per_step": {k: round(v["ms"] / n_prof, 3) for k, v in prof.items() if v["ms"] > 0},
        "e2e": {"value": tokens / float(np.mean(e2e)), "unit": UNIT,
                "h2d_bytes_per_step": int(4 * Q.size + 8 * L + h2d_batch),
                "d2h_bytes_per_step": int(B * (8 * V + L * layout.S * 5 + 8 * 2 * L)),
                "ttft_ms": float(np.mean(e2e)) * 1e3},
        "gpu_launches": int(sum(v["kernels"] for v in prof.values()) / n_prof),
        "clocks": clk.summary(),
    }
    print(json.dumps(_finite(line)), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--numerics", choices=["fast", "parity", "exact"], default="parity",
                    help="parity (default): the reference's fp32-store / fp64-accumulate arithmetic on the tensor "
                         "cores; exact: bit-exact projections + reference-order scores (scalar fp64); fast: bf16")
    ap.add_argument("--r-avg", type=float, default=None)
    ap.add_argument("--seed", type=int, default=20250807)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="(kept for compatibility; no-op)")
    ap.add_argument("--no-compare", action="store_true",
                    help="skip the other numerics modes' runs (selection_parity / other_mode / exact_mode blocks)")
    ap.add_argument("--no-exact", action="store_true", help="skip the PARITY_EXACT comparison (~40 s at C3)")
    ap.add_argument("--updates", type=float, default=0.35,
                    help="fraction of dynamic owners updated (refreshed inside the TTFT) before each query of the "
                         "updates block (configs[2]: frequent dynamic-group updates; 0 disables the block)")
    ap.add_argument("--update-steps", type=int, default=2)
    ap.add_argument("--memory", choices=["hbm", "host"], default="hbm",
                    help="memory KV resident in HBM (C2-C4) or pinned host DRAM with the K10 loader (C5-style)")
    ap.add_argument("--hbm-budget-gb", type=float, default=0.0,
                    help="--memory host: keep the deepest layers of the memory KV also in HBM up to this budget "
                         "(the capacity-bounded fast tier; keep_memory_residency)")
    ap.add_argument("--sub-batch", type=int, default=0,
                    help="--batch: run the B queries as sub-batches of this many (HBM for larger memories)")
    ap.add_argument("--no-sequential", action="store_true",
                    help="--batch: skip the one-query-at-a-time comparison")
    ap.add_argument("--batch", type=int, default=1,
                    help="B > 1: B concurrent planning queries through keep_plan_keep_batch (one GPU)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.r_avg is not None:
        cfg["r_avg"] = args.r_avg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg)
        return
    if args.batch > 1:
        if rank == 0:
            run_batch(args, cfg)
        return
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    run_ours(args, cfg, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
