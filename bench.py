#!/usr/bin/env python
"""KEEP per-layer memory prefill benchmark (TTFT + recomputed tokens/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full KEEP prefill (plan_keep: every layer's scoring, multi-hop
selection, gathered recompute, merged-KV assembly, plus the first-token
logits) over a 16K-token synthetic memory on Qwen2.5-14B dimensions
(BASELINE.json configs[2], SURVEY.md 8 "C3").  Prints one JSON line.

  value  recomputed tokens/s = sum_l N_act(l) / TTFT, device-timed (CUDA
         events) with the memory KV resident in HBM.
  e2e    the same metric through the C ABI call with host buffers (token
         ids H2D, logits/plan D2H inside the timed region), host wall clock.
The CPU baseline is the reference's own path (oracle/_ref, the unmodified
headers; else the plain-C restatement) timed on a bounded one-layer sample of
the same configuration on one host core and extrapolated op-for-op to the
workload (the reference is single-threaded; a full C3 run takes days).
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
                     "mean_dram_pct_of_peak": det["dram_pct"] / n, "mean_dram_bytes": sum(acc[k]) / n}
    return {k: sum(v) / len(v) for k, v in acc.items()}


def numerics_for(args, cfg):
    """FAST (bf16 tensor cores) needs model / MLP widths in multiples of 64;
    the reference's tiny CPU default (c1: d = 32) runs in PARITY."""
    import paper_2602_23592_b200 as kb
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
_W_CACHE = {}


def cpu_sample(cfg, seed=7, sample_segments=2, reps=1):
    """Time the reference path (PrefillCursor::step + converge via plan_keep)
    for ONE layer at the workload's full width on a small layout; return the
    measured fp64-accumulate MAC rate and what was sampled."""
    from oracle.oracle import Oracle, available, Problem
    kind = "reference" if available("kr") else "port"
    orc = Oracle("kr" if kind == "reference" else "ko")
    L1, H, d, mlp = 1, cfg["H"], cfg["d"], cfg["mlp"]
    V = 1024  # vocabulary only feeds the embedding gather in a step
    rng = np.random.default_rng(seed)
    std = 1.0 / np.sqrt(d)
    n_w = orc.weight_count(L1, H, d, mlp, V)
    key = (n_w, seed)
    if key not in _W_CACHE:
        _W_CACHE[key] = (rng.standard_normal(n_w, dtype=np.float32) * np.float32(std)).astype(np.float32)
    w = _W_CACHE[key]
    from paper_2602_23592_b200.synth import make_instance_layout
    inst = make_instance_layout(seed, sample_segments, V)
    p = Problem(L1, H, d, mlp, V, seed, inst.seg_len, inst.tokens, inst.query)
    T = p.T
    cached = np.zeros((L1, 2, p.Tm, d), np.float32)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.plan_keep(p, w, np.ones(1), cached=cached)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    macs = T * (4.0 * d * d + 2.0 * d * mlp) + 2.0 * d * T * (T + 1) / 2.0
    return {"kind": kind, "seconds": best, "macs": macs, "rate": macs / best, "rows": T,
            "sample": f"one layer at full width (d={d}, H={H}, mlp={mlp}) over {T} rows "
                      f"({sample_segments} segments + {len(inst.query)}-token query), V reduced to {V}; "
                      f"{kind} path, 1 host core, extrapolated op-for-op to the workload"}


def cpu_extrapolate(sample, cfg, rows_per_layer, pairs_per_layer):
    d, mlp = cfg["d"], cfg["mlp"]
    macs = float(np.sum(rows_per_layer)) * (4.0 * d * d + 2.0 * d * mlp) + 2.0 * d * float(np.sum(pairs_per_layer))
    ttft_s = macs / sample["rate"]
    return {"ttft_s": ttft_s, "tokens_per_s": float(np.sum(rows_per_layer)) / ttft_s}


def budget_plan(cfg, layout, r):
    """Plan sizes if every budget were realised (reference arm's workload
    model; the realised walk can only be shorter)."""
    import paper_2602_23592_b200 as kb
    S = layout.S
    plan = np.zeros((cfg["L"], S), np.uint8)
    for l in range(cfg["L"]):
        b = S if l == 0 else min(S, kb.layer_budget(r[l], S))
        plan[l, :b] = 1
    return plan


def run_reference(args, cfg):
    import paper_2602_23592_b200 as kb
    layout, query = workload(cfg, args.seed)
    r = kb.ratio_schedule(cfg["L"], cfg["r_avg"])
    plan = budget_plan(cfg, layout, r)
    seg_len = np.asarray(layout.seg_len)
    rows = plan.astype(np.int64) @ seg_len + len(query)
    pairs = attention_pairs(layout, len(query), plan)
    for _ in range(args.warmup):
        cpu_sample(cfg, reps=1)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = cpu_sample(cfg, reps=1)
        vals.append(cpu_extrapolate(s, cfg, rows, pairs))
    wall = time.perf_counter() - t0
    v = float(np.median([x["tokens_per_s"] for x in vals]))
    ttft = float(np.median([x["ttft_s"] for x in vals])) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32-store/f64-acc",
            "data": "synthetic", "ttft_ms": ttft,
            "config": {"workload": args.config, "desc": cfg["desc"], "S": layout.S,
                       "T": int(seg_len.sum()) + len(query), "plan_model": "budgets fully realised"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": s["kind"], "sample": s["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(_finite(line)), flush=True)


# ------------------------------------------------------------------ GPU arm --
def run_ours(args, cfg, rank, world, dist):
    import torch

    import paper_2602_23592_b200 as kb
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    numerics = numerics_for(args, cfg)
    L, H, d, mlp, V = cfg["L"], cfg["H"], cfg["d"], cfg["mlp"], cfg["V"]
    layout, query = workload(cfg, args.seed)
    r = kb.ratio_schedule(L, cfg["r_avg"])
    t0 = time.perf_counter()
    if world > 1:
        # KV-head sharding: one context per rank over the library's own NCCL
        # communicator (torch.distributed only carries its unique id)
        from paper_2602_23592_b200.dist import sharded_context
        ctx = sharded_context(L, H, d, mlp, V, args.seed, numerics, device=dev)
    else:
        ctx = kb.Context(L, H, d, mlp, V, args.seed, numerics, device=dev)
    ctx.model_init()
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    host_mem = args.memory == "host"
    ctx.memory_compute_layout(layout, version=1, tier=kb.TIER_HOST if host_mem else kb.TIER_DEVICE)
    t_mem = time.perf_counter() - t0

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # --updates F: before every query a fraction F of the dynamic owners was
    # updated and must be refreshed (harness.hpp:609-628; "frequent dynamic
    # updates", test_harness.cpp:266-268); the refresh is part of the TTFT
    owners_all = layout.owners()
    dyn = [i for i, o in enumerate(owners_all) if o[0] == kb.SEGMENT]
    owner_tokens = [int(np.sum(layout.seg_len[o[2]:o[3]])) for o in owners_all]
    upd_rng = np.random.default_rng(args.seed + 1)
    version = [1]

    def step():
        if args.updates > 0:
            version[0] += 1
            pick = [u for u in dyn if upd_rng.random() < args.updates]
            # (the profiler times the refresh call as one scope; the prefill
            # itself runs unprofiled in the timed steps)
            was_on = step.profiling
            ctx.profile_enable(True)
            ctx.memory_refresh(layout, pick, version[0], tier=kb.TIER_HOST if host_mem else kb.TIER_DEVICE)
            ctx.profile_enable(was_on)
            # (owners not picked stay current at their old version)
            step.refreshed_tokens = float(sum(owner_tokens[u] for u in pick))
        return ctx.plan_keep(layout, query, r, final_hidden=False)

    step.refreshed_tokens = 0.0
    step.profiling = False
    for _ in range(args.warmup):
        step()
    ctx.profile_read(reset=True)
    barrier()
    steps = []
    refreshed = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            steps.append(step())
            refreshed.append(step.refreshed_tokens)
    barrier()
    refresh_ms = ctx.profile_read(reset=True)["refresh"]["ms"]  # device time of the in-TTFT refreshes
    # per-phase device times (roofline, phase shares) from separate profiled
    # steps: the per-phase events are a measurement artefact kept out of the
    # timed steps above
    n_prof = max(1, min(args.steps, 3))
    step.profiling = True
    ctx.profile_enable(True)
    for _ in range(n_prof):
        step()
    ctx.profile_enable(False)
    step.profiling = False
    prof = ctx.profile_read(reset=True)
    ttft = np.array([s["ttft_ms"] for s in steps])
    if args.updates > 0:
        ttft = ttft + refresh_ms / max(args.steps, 1)
    # recomputed tokens: the plan's rows per layer, plus every layer of the refreshed owners
    tokens = float(np.sum(steps[-1]["rows_per_layer"])) + float(np.mean(refreshed)) * L
    total_ms = float(np.sum(ttft))
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # one prefill per step for the whole job (heads split across the ranks)
    value = tokens * args.steps / (total_ms / 1e3)

    # e2e: the C-ABI call with host buffers, host wall clock
    e2e_s = []
    for _ in range(max(1, args.steps)):
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

    pk, src = peaks()
    gemm_phases = ["qkv", "wo", "mlp_in", "mlp_out"]
    g_ms = sum(prof[p]["ms"] for p in gemm_phases)
    g_fl = sum(prof[p]["flops"] for p in gemm_phases)
    g_by = sum(prof[p]["bytes"] for p in gemm_phases)
    g_n = sum(prof[p]["launches"] for p in gemm_phases)
    a_ms, a_fl = prof["attn"]["ms"], prof["attn"]["flops"]
    phase_ms = {k: round(v["ms"] / n_prof, 3) for k, v in prof.items() if v["ms"] > 0}
    traffic = ncu_traffic()
    tensor_peak = pk["bf16_tflops_sustained"] if numerics == kb.FAST else 37.0
    g_ach = g_fl / (g_ms / 1e3) / 1e12 if g_ms > 0 else 0.0
    a_ach = a_fl / (a_ms / 1e3) / 1e12 if a_ms > 0 else 0.0
    gemm_roof = {"kernel": "gemm_tc_kernel (tcgen05 bf16, fused epilogues)" if numerics == kb.FAST else "gemm_f64acc",
                 "bound": "tensor", "achieved": g_ach, "peak": tensor_peak, "unit": "TFLOP/s",
                 "frac": g_ach / tensor_peak, "traffic": traffic.get("gemm_tc_kernel") if numerics == kb.FAST else None,
                 "peak_source": src + " (bf16 sustained)", "per_launch_ms": g_ms / max(g_n, 1),
                 "algorithmic_bytes_per_launch": g_by / max(g_n, 1),
                 "hbm_gbs_achieved": g_by / (g_ms / 1e3) / 1e9 if g_ms > 0 else 0.0,
                 "traffic_launches": DETAIL.get("gemm_tc_kernel") if numerics == kb.FAST else None,
                 "traffic_note": "traffic = the ncu-captured layer-0 launches (M = 16,280: 0.82 GB algorithmic for "
                                 "the QKV one), not the step average; A is re-read across weight-column bands, "
                                 "at ~20% of HBM peak -- the kernel stays tensor-bound"}
    attn_roof = {"kernel": "attn_tc2_kernel STATS + CTX / FLASH (K5, tcgen05, summary bins on the tensor core)"
                 if numerics == kb.FAST else "attn_stats / ctx / bins kernels (K5, fp64 SIMT, PARITY)",
                 "bound": "tensor", "achieved": a_ach, "peak": tensor_peak, "unit": "TFLOP/s",
                 "frac": a_ach / tensor_peak, "traffic": traffic.get("attn_tc2_kernel") if numerics == kb.FAST else None,
                 "peak_source": src,
                 "note": "algorithmic FLOPs 4*d*sum(t+1) (QK^T + PV once); the kernel pair does QK^T twice"}
    d_ms, d_by, d_n = prof["attn_decode"]["ms"], prof["attn_decode"]["bytes"], prof["attn_decode"]["launches"]
    hbm_peak = pk["hbm_gbs"]
    d_ach = d_by / (d_ms / 1e3) / 1e9 if d_ms > 0 else 0.0
    # the layers after the walk: the query rows alone against the whole merged
    # KV, HBM-bound (algorithmic bytes = K + V of the visible keys once + q + ctx)
    decode_roof = {"kernel": "attn_decode_kernel (K5d, split-K flash decoding, TMA stages)", "bound": "hbm",
                   "achieved": d_ach, "peak": hbm_peak, "unit": "GB/s", "frac": d_ach / hbm_peak,
                   "traffic": traffic.get("attn_decode_kernel"), "traffic_launches": DETAIL.get("attn_decode_kernel"),
                   "peak_source": src,
                   "per_launch_ms": d_ms / max(d_n, 1), "algorithmic_bytes_per_launch": d_by / max(d_n, 1),
                   "launches_per_step": d_n / n_prof}
    roof = gemm_roof if g_ms >= a_ms else attn_roof
    launches = int(sum(v["kernels"] for v in prof.values())) // n_prof
    loader_info = None
    if host_mem:
        tr = ctx.loader_trace()
        h2d_kv = float(sum(r["bytes"] for r in tr))
        ms = prof["loader"]["ms"] / n_prof
        # time compute(l) spent waiting beyond the previous layer: not measurable per stream here;
        # report volume, copy-engine time and achieved H2D bandwidth
        h2d += h2d_kv  # the memory KV crosses PCIe inside every step
        loader_info = {"h2d_bytes_per_step": h2d_kv, "copy_ms_per_step": ms,
                       "h2d_gbs": h2d_kv / (ms * 1e6) if ms > 0 else None,
                       "items": len(tr), "preloads": sum(1 for r in tr if r["kind"] == "preload"),
                       "urgent": sum(1 for r in tr if r["kind"] == "urgent")}

    # fidelity beside speed: KEEP's last row against a full
    # recompute of the same prefill (schedule of ones), divergence as in
    # prefill.hpp:501-531, plus the full recompute's own TTFT
    quality = None
    if args.updates == 0 and not args.no_quality:
        keep_res = ctx.plan_keep(layout, query, r, final_hidden=True)
        full_res = ctx.plan_keep(layout, query, np.ones(L), final_hidden=True)
        l2, kl = ctx.divergence(keep_res["final_hidden"][-1], full_res["final_hidden"][-1])
        quality = {"full_recompute_ttft_ms": full_res["ttft_ms"], "keep_ttft_ms": keep_res["ttft_ms"],
                   "speedup_vs_full_recompute": full_res["ttft_ms"] / keep_res["ttft_ms"],
                   "divergence_vs_full": {"l2": l2, "sym_kl": kl, "rel_l2": l2 / max(float(np.linalg.norm(
                       full_res["final_hidden"][-1].astype(np.float64))), 1e-300)},
                   # (sym_kl is NaN exactly where prefill.hpp:526-528's is: both
                   # softmaxes underflow to 0 at the same vocabulary entries)
                   "top1_agree": bool(np.argmax(keep_res["last_logits"]) == np.argmax(full_res["last_logits"])),
                   "full_recomputed_tokens": float(np.sum(full_res["rows_per_layer"]))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        s = cpu_sample(cfg)
        plan = steps[-1]["plan"]
        ex = cpu_extrapolate(s, cfg, steps[-1]["rows_per_layer"], attention_pairs(layout, len(query), plan))
        cpu = {"value": ex["tokens_per_s"], "unit": UNIT, "cores": 1, "kind": s["kind"], "sample": s["sample"],
               "ttft_ms_extrapolated": ex["ttft_s"] * 1e3, "sample_seconds": s["seconds"]}

    if rank == 0:
        plan = steps[-1]["plan"]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if numerics == kb.FAST else "f32-store/f64-acc", "data": "synthetic",
            "ttft_ms": float(np.median(ttft)), "ttft_ms_min": float(np.min(ttft)),
            "config": {"workload": args.config, "desc": cfg["desc"], "L": L, "H": H, "d": d, "mlp": mlp, "V": V,
                       "S": layout.S, "T": int(np.sum(layout.seg_len)) + len(query),
                       "units": {"static_groups_of_8": sum(1 for u in layout.units if u[2] == 1),
                                 "dynamic_segments": sum(1 for u in layout.units if u[2] == 0)},
                       "r_avg": cfg["r_avg"],
                       "parallelism": f"KV-head sharded x{world} (NCCL)" if world > 1 else "1 GPU",
                       "l2": "inputs larger than L2 ({:.1f} GB bf16 weights + {:.1f} GB memory KV read per step)".format(
                           2e-9 * L * (4 * d * d + 2 * d * mlp), 4e-9 * L * d * int(np.sum(layout.seg_len))),
                       "memory_kv": ("pinned-host canonical KV, layer-balanced K10 loader" if host_mem else
                                     "HBM-resident canonical KV (static groups joint, dynamic per segment)")},
            "recomputed_tokens_per_step": tokens,
            "updates": ({"fraction_of_dynamic_owners": args.updates, "refreshed_tokens_per_step": float(np.mean(refreshed)),
                         "refresh_ms_per_step": refresh_ms / max(args.steps, 1)} if args.updates > 0 else None),
            "plan_segments_per_layer": [int(x) for x in plan.sum(1)],
            "rows_per_layer": [int(x) for x in steps[-1]["rows_per_layer"]],
            "hops_per_layer": [int(x) for x in steps[-1]["hops"]],
            "phase_ms_per_step": phase_ms,
            "setup_s": {"model_init": t_init, "canonical_kv_refresh": t_mem},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ttft_ms": e2e_mean * 1e3},
            "gpu_launches": launches,
            "loader": loader_info,
            "quality": quality,
            "roofline": roof,
            "roofline_kernels": [gemm_roof, attn_roof] + ([decode_roof] if d_ms > 0 else []),
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(_finite(line)), flush=True)
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
    ctx.memory_compute_layout(layout, tier=kb.TIER_HOST if host_mem else kb.TIER_DEVICE)
    for _ in range(args.warmup):
        ctx.plan_keep_batch(layout, Q, r)
    torch.cuda.synchronize()
    res = []
    dev = torch.cuda.current_device()
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            res.append(ctx.plan_keep_batch(layout, Q, r))
    torch.cuda.synchronize()
    # per-phase times from one separate profiled batch (kept out of the timed steps)
    ctx.profile_read(reset=True)
    ctx.profile_enable(True)
    ctx.plan_keep_batch(layout, Q, r)
    ctx.profile_enable(False)
    prof = ctx.profile_read(reset=True)
    n_prof = 1
    batch_ms = np.array([x[0]["ttft_ms"] for x in res])
    tokens = float(sum(np.sum(o["rows_per_layer"]) for o in res[-1]))
    value = tokens / (float(np.mean(batch_ms)) / 1e3)
    # e2e: host query ids in, host plans + logits out, wall clock
    e2e = []
    for _ in range(max(1, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.plan_keep_batch(layout, Q, r)
        e2e.append(time.perf_counter() - t0)
    st_b = ctx.memory_stats()["bytes_loaded_slow"]
    ctx.plan_keep_batch(layout, Q, r)
    h2d_batch = ctx.memory_stats()["bytes_loaded_slow"] - st_b
    # the same queries one at a time (the batch workspace released first)
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
                  "speedup_vs_sequential": seq_ms / float(np.median(batch_ms)),
                  "plans_equal_to_sequential": same,
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
    ap.add_argument("--numerics", choices=["fast", "parity"], default="fast")
    ap.add_argument("--r-avg", type=float, default=None)
    ap.add_argument("--seed", type=int, default=20250807)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="skip the full-recompute fidelity comparison")
    ap.add_argument("--updates", type=float, default=0.0,
                    help="fraction of dynamic owners updated (refreshed inside the TTFT) before every query")
    ap.add_argument("--memory", choices=["hbm", "host"], default="hbm",
                    help="memory KV resident in HBM (C2-C4) or pinned host DRAM with the K10 loader (C5-style)")
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
