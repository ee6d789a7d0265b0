// loader.cu -- K10: layer-balanced loading of memory KV from pinned host DRAM
// into the merged KV of the prefill.
//
// The reference only simulates this (pipeline_sim.hpp); here it is real:
//   items      (layer l, owner) for every host-tier owner with a member
//              outside plan[l] -- the reference's workload items
//              (derive_workload, pipeline_sim.hpp:103-154); a block is
//              copied whole (group blocks are atomic), its recomputed rows
//              are overwritten afterwards by the QKV scatter of compute(l).
//   schedule   simulate_balanced (261-338) made online:
//                before compute(l): any item of layer l not yet loaded
//                  (owners the selection after layer l-1 just dropped);
//                  compute(l) waits on the copy stream (D1, 366-375);
//                behind compute(l): items of layer l+1 whose owner already
//                  has a member out at l (monotone plans keep it out), then
//                  pre-loads of owners whose members ALL left the plan by l
//                  (preload_eligible_from, 169-187) for layers >= l+2 in
//                  ascending (layer, owner) order while they fit the
//                  estimated compute window of layer l (the idle-window fill,
//                  314-333).
//   engine     cudaMemcpyAsync on the context's copy stream, one call per
//              run of adjacent blocks (merged below): copy engines, no SM time.
// Every batch is bracketed by timing events so the realised timeline can be
// checked against the reference's validate_timeline rules (D1, P, S).
#include <algorithm>
#include <climits>
#include <cstring>

#include "engine.hpp"

namespace keep_b200 {

namespace {

enum { KIND_URGENT = 0, KIND_AHEAD = 1, KIND_PRELOAD = 2 };

// HBM-resident owners: the in-stream copy kernel (K4) by default; measured
// at C3 it beats copy-engine D2D batches (4.6 vs 6.6 ms and no HBM contention
// with the GEMMs).  KEEP_D2D_LOADER=1 routes them through this loader too.
bool cached_kernel() {
    static const bool v = [] {
        const char* e = std::getenv("KEEP_D2D_LOADER");
        return !(e && *e == '1');
    }();
    return v;
}

const uint8_t* host_keys(const Context& c, const Payload& pl, int l) {
    const int64_t sheet = pl.arena->rows * c.dl * c.elem;
    return static_cast<const uint8_t*>(pl.arena->buf.p) + (int64_t(l) * 2) * sheet + pl.row0 * c.dl * c.elem;
}

cudaEvent_t take_event(Loader& ld) {
    if (!ld.pool.empty()) {
        cudaEvent_t e = ld.pool.back();
        ld.pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    KEEP_CUDA(cudaEventCreate(&e));
    return e;
}

bool block_ok(const Context& c, const Loader::Unit& u, int l) {
    auto cv = c.current_version.find(u.key);
    return u.pl && l < int(u.pl->present.size()) && u.pl->present[l] && cv != c.current_version.end() &&
           u.pl->layer_version[l] == cv->second;
}

// a missing / stale block is an error only when its layer is computed
// (prefill.hpp:340-350); early (ahead / pre-load) items just skip it
void check_block(Context& c, const Loader::Unit& u, int l) {
    if (block_ok(c, u, l)) return;
    c.stats.cache_misses++;
    raise(KEEP_ERR_CACHE_MISS, std::string("missing cached KV for owner ") +
                                   (u.key.kind == KEEP_OWNER_SEGMENT ? "s" : "g") + std::to_string(u.key.id) +
                                   " layer " + std::to_string(l));
}

// Issue one batch of (layer, unit) items on the copy stream.
void issue(Context& c, Pass& p, const std::vector<std::pair<int, int>>& items, int kind, int at_layer) {
    if (items.empty()) return;
    Loader& ld = c.loader;
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    dsts.reserve(2 * items.size());
    srcs.reserve(2 * items.size());
    sizes.reserve(2 * items.size());
    Loader::Batch bt;
    bt.kind = kind;
    bt.at_layer = at_layer;
    const int bi = int(ld.batches.size());
    for (auto [l, ui] : items) {
        const Loader::Unit& u = ld.units[ui];
        if (kind == KIND_URGENT) check_block(c, u, l);
        else if (!block_ok(c, u, l)) continue;
        const size_t blk = size_t(u.tokens) * c.dl * c.elem;
        const uint8_t* hk = host_keys(c, *u.pl, l);
        const uint8_t* hv = hk + u.pl->arena->rows * c.dl * c.elem;
        uint8_t* dk = static_cast<uint8_t*>(p.kdst[l]) + u.dst_row * c.dl * c.elem;
        uint8_t* dv = static_cast<uint8_t*>(p.vdst[l]) + u.dst_row * c.dl * c.elem;
        dsts.push_back(dk);
        srcs.push_back(const_cast<uint8_t*>(hk));
        sizes.push_back(blk);
        dsts.push_back(dv);
        srcs.push_back(const_cast<uint8_t*>(hv));
        sizes.push_back(blk);
        ld.loaded[size_t(l) * ld.units.size() + ui] = 1;
        ld.last_batch[l] = bi;
        ld.recs.push_back(Loader::Rec{l, ui, bi, 2 * blk});
        bt.bytes += 2 * blk;
        if (u.pl->arena->tier == KEEP_TIER_HOST) {
            bt.host = true;
            c.stats.bytes_loaded_slow += 2 * blk;
        }
    }
    if (dsts.empty()) return;
    // coalesce blocks that are adjacent in both the host arena and the merged
    // KV (consecutive owners of one refresh batch): fewer, larger DMA copies
    {
        std::vector<size_t> ord(dsts.size());
        for (size_t k = 0; k < ord.size(); ++k) ord[k] = k;
        std::sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return dsts[x] < dsts[y]; });
        std::vector<void*> d2, s2;
        std::vector<size_t> z2;
        for (size_t k : ord) {
            if (!d2.empty() && static_cast<uint8_t*>(d2.back()) + z2.back() == dsts[k] &&
                static_cast<uint8_t*>(s2.back()) + z2.back() == srcs[k]) {
                z2.back() += sizes[k];
                continue;
            }
            d2.push_back(dsts[k]);
            s2.push_back(srcs[k]);
            z2.push_back(sizes[k]);
        }
        dsts.swap(d2);
        srcs.swap(s2);
        sizes.swap(z2);
    }
    bt.a = take_event(ld);
    bt.b = take_event(ld);
    KEEP_CUDA(cudaEventRecord(bt.a, c.s_copy));
    {
        ProfScope ps(c.prof, KEEP_PROF_LOADER, c.s_copy, 0.0, double(bt.bytes), 0);
        for (size_t k = 0; k < dsts.size(); ++k)
            KEEP_CUDA(cudaMemcpyAsync(dsts[k], srcs[k], sizes[k], cudaMemcpyHostToDevice, c.s_copy));
    }
    KEEP_CUDA(cudaEventRecord(bt.b, c.s_copy));
    ld.batches.push_back(bt);
}

// bandwidth estimate from batches that have finished (non-blocking)
void update_bw(Loader& ld) {
    for (; ld.bw_seen < ld.batches.size(); ++ld.bw_seen) {
        const Loader::Batch& b = ld.batches[ld.bw_seen];
        if (cudaEventQuery(b.b) != cudaSuccess) {
            cudaGetLastError();
            break;
        }
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, b.a, b.b) == cudaSuccess && ms > 0.05f && b.bytes > (8u << 20)) {
            double& bw = b.host ? ld.bw_gbs : ld.bw_d2d_gbs;
            bw = 0.5 * bw + 0.5 * (double(b.bytes) / (ms * 1e6));
        }
        cudaGetLastError();
    }
}

}  // namespace

Loader::~Loader() {
    for (auto& b : batches) {
        if (b.a) cudaEventDestroy(b.a);
        if (b.b) cudaEventDestroy(b.b);
    }
    for (auto* v : {&comp_start, &comp_end, &attn_end, &eval_a, &eval_b})
        for (auto e : *v)
            if (e) cudaEventDestroy(e);
    for (auto e : pool) cudaEventDestroy(e);
    if (t0) cudaEventDestroy(t0);
}

bool loader_covers(const Context& c, int seg, int l) {
    const Loader& ld = c.loader;
    return ld.on && ld.seg_host[seg] && l < ld.seg_mirror_from[seg];
}

void loader_begin(Context& c, Pass& p) {
    Loader& ld = c.loader;
    for (auto& b : ld.batches) {
        ld.pool.push_back(b.a);
        ld.pool.push_back(b.b);
    }
    ld.batches.clear();
    ld.recs.clear();
    ld.units.clear();
    ld.bw_seen = 0;
    ld.L = c.L;
    // host-tier owners of the layout, one unit per contiguous owner run
    for (int i = 0; i < p.S;) {
        int j = i + 1;
        while (j < p.S && !(c.seg_owner[j] < c.seg_owner[i]) && !(c.seg_owner[i] < c.seg_owner[j])) ++j;
        auto it = c.store.find(c.seg_owner[i]);
        // pinned-host owners always; HBM owners only with KEEP_D2D_LOADER=1
        if (it != c.store.end() && (it->second.arena->tier == KEEP_TIER_HOST || !cached_kernel())) {
            Loader::Unit u;
            u.key = c.seg_owner[i];
            u.b = i;
            u.e = j;
            u.dst_row = p.seg_start[i] - c.seg_owner_row[i];
            u.tokens = it->second.tokens;
            u.pl = &it->second;
            int64_t members = 0;
            for (int k = i; k < j; ++k) members += p.seg_len[k];
            if (c.seg_owner_row[i] != 0 || members != u.tokens)
                raise(KEEP_ERR_INPUT, "host-tier owner block does not match its members in the layout");
            ld.units.push_back(u);
        }
        i = j;
    }
    ld.on = !ld.units.empty();
    ld.any_host = false;
    for (const auto& u : ld.units) ld.any_host |= u.pl->arena->tier == KEEP_TIER_HOST;
    ld.seg_host.assign(p.S, 0);
    ld.seg_mirror_from.assign(p.S, INT_MAX);
    for (const auto& u : ld.units)
        for (int k = u.b; k < u.e; ++k) {
            ld.seg_host[k] = 1;
            ld.seg_mirror_from[k] = std::min(u.pl->arena->mirror_from, c.L);
        }
    if (!ld.on) return;
    // (sort by owner so ascending (layer, owner) order = the reference's item order)
    std::sort(ld.units.begin(), ld.units.end(), [](const Loader::Unit& a, const Loader::Unit& b) { return a.key < b.key; });
    ld.loaded.assign(size_t(c.L) * ld.units.size(), 0);
    for (size_t ui = 0; ui < ld.units.size(); ++ui)  // HBM-resident layers: fast tier, nothing to load
        for (int l = std::min(ld.units[ui].pl->arena->mirror_from, c.L); l < c.L; ++l)
            ld.loaded[size_t(l) * ld.units.size() + ui] = 1;
    ld.out_from.assign(ld.units.size(), INT32_MAX);
    ld.last_batch.assign(c.L, -1);
    if (ld.comp_start.size() != size_t(c.L)) {
        for (auto* v : {&ld.comp_start, &ld.comp_end, &ld.attn_end, &ld.eval_a, &ld.eval_b}) {
            for (auto e : *v)
                if (e) cudaEventDestroy(e);
            v->assign(c.L, nullptr);
            for (auto& e : *v) KEEP_CUDA(cudaEventCreate(&e));
        }
    }
    ld.has_eval.assign(c.L, 0);
    if (!ld.t0) KEEP_CUDA(cudaEventCreate(&ld.t0));
    KEEP_CUDA(cudaEventRecord(ld.t0, c.s_main));
    // the copy stream starts after the prefill begins (timeline origin)
    KEEP_CUDA(cudaStreamWaitEvent(c.s_copy, ld.t0, 0));
}

void loader_before_layer(Context& c, Pass& p, int l, const uint8_t* active) {
    Loader& ld = c.loader;
    if (!ld.on) return;
    const size_t U = ld.units.size();
    std::vector<std::pair<int, int>> urgent;
    for (size_t ui = 0; ui < U; ++ui) {
        const auto& u = ld.units[ui];
        bool needed = false;
        for (int k = u.b; k < u.e && !needed; ++k) needed = !active[k];
        if (needed && !ld.loaded[size_t(l) * U + ui]) urgent.push_back({l, int(ui)});
    }
    issue(c, p, urgent, KIND_URGENT, l);
    if (ld.last_batch[l] >= 0) KEEP_CUDA(cudaStreamWaitEvent(c.s_main, ld.batches[ld.last_batch[l]].b, 0));
    KEEP_CUDA(cudaEventRecord(ld.comp_start[l], c.s_main));
}

void loader_after_layer(Context& c, Pass& p, int l, const uint8_t* active, double est_ms) {
    Loader& ld = c.loader;
    if (!ld.on) return;
    KEEP_CUDA(cudaEventRecord(ld.comp_end[l], c.s_main));
    if (l + 1 >= c.L) return;
    const size_t U = ld.units.size();
    update_bw(ld);
    std::vector<std::pair<int, int>> items;
    uint64_t ahead_bytes = 0;
    for (size_t ui = 0; ui < U; ++ui) {
        const auto& u = ld.units[ui];
        bool any_out = false, all_out = true;
        for (int k = u.b; k < u.e; ++k) {
            any_out |= !active[k];
            all_out &= !active[k];
        }
        if (all_out) ld.out_from[ui] = std::min(ld.out_from[ui], l);
        if (any_out && !ld.loaded[size_t(l + 1) * U + ui]) {
            items.push_back({l + 1, int(ui)});
            ahead_bytes += 2ull * u.tokens * c.dl * c.elem;
        }
    }
    // everything issued here starts with compute(l) at the earliest (the
    // reference's "loads for l+1 start with compute(l)", pipeline_sim.hpp:
    // 261-338): the host runs layers ahead of the device, and an early
    // pre-load would overlap a compute(k < l) whose plan still holds a member
    // (rule S)
    KEEP_CUDA(cudaStreamWaitEvent(c.s_copy, ld.comp_start[l], 0));
    // pre-loads into the idle window of compute(l)
    const double window = est_ms * 1e-3 * (ld.any_host ? ld.bw_gbs : ld.bw_d2d_gbs) * 1e9;
    double budget = window - double(ahead_bytes);
    for (int l2 = l + 2; l2 < c.L && budget > 0.0; ++l2)
        for (size_t ui = 0; ui < U && budget > 0.0; ++ui) {
            if (ld.out_from[ui] > l || ld.loaded[size_t(l2) * U + ui]) continue;
            const double b = 2.0 * ld.units[ui].tokens * c.dl * c.elem;
            if (b > budget) {
                budget = 0.0;  // an item that would overrun the window stops the fill
                break;
            }
            items.push_back({l2, int(ui)});
            budget -= b;
        }
    issue(c, p, items, KIND_AHEAD, l);
}

}  // namespace keep_b200

extern "C" int keep_loader_trace(void* ctx, keep_load_record* out, int32_t cap, int32_t* n_out) {
    using namespace keep_b200;
    try {
        Context& c = *static_cast<Context*>(ctx);
        KEEP_CUDA(cudaSetDevice(c.cfg.device));
        Loader& ld = c.loader;
        KEEP_CUDA(cudaStreamSynchronize(c.s_copy));
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
        int n = 0;
        for (const auto& r : ld.recs) {
            if (n >= cap) break;
            const Loader::Batch& b = ld.batches[r.batch];
            keep_load_record& o = out[n++];
            o.layer = r.layer;
            o.kind = (b.kind == 1 && r.layer >= b.at_layer + 2) ? 2 : b.kind;
            o.at_layer = b.at_layer;
            o.owner = keep_owner{ld.units[r.unit].key.kind, ld.units[r.unit].key.id};
            o.bytes = r.bytes;
            float ms = 0.f;
            KEEP_CUDA(cudaEventElapsedTime(&ms, ld.t0, b.a));
            o.batch_start_ms = ms;
            KEEP_CUDA(cudaEventElapsedTime(&ms, ld.t0, b.b));
            o.batch_end_ms = ms;
            KEEP_CUDA(cudaEventElapsedTime(&ms, ld.t0, ld.comp_start[r.layer]));
            o.compute_start_ms = ms;
        }
        *n_out = int32_t(ld.recs.size());
        return KEEP_OK;
    } catch (const KeepError& e) {
        set_last_error(e.what());
        return e.code;
    }
}

// The realised timeline of the last prefill over pinned-host owners, in the
// reference's Timeline vocabulary (pipeline_sim.hpp:69-92): loads (each copy
// batch's interval shared out to its items in byte proportion -- one copy
// engine moves them in order), compute(l) on the compute stream, and the walk
// (eval) of layer l on the selector stream.  attention_fraction out = the
// smallest (summary done - compute start) / compute span over the walked
// layers (bounded by the walk's own start), the D2 parameter of validate_timeline.
extern "C" int keep_timeline_trace(void* ctx, keep_timeline_event* out, int32_t cap, int32_t* n_out,
                                   double* attention_fraction) {
    using namespace keep_b200;
    try {
        Context& c = *static_cast<Context*>(ctx);
        KEEP_CUDA(cudaSetDevice(c.cfg.device));
        Loader& ld = c.loader;
        KEEP_CUDA(cudaStreamSynchronize(c.s_copy));
        KEEP_CUDA(cudaStreamSynchronize(c.s_sel));
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
        if (!ld.on) raise(KEEP_ERR_TRACE, "no loader trace: the last prefill had no pinned-host memory");
        auto at = [&](cudaEvent_t e) {
            float ms = 0.f;
            KEEP_CUDA(cudaEventElapsedTime(&ms, ld.t0, e));
            return double(ms);
        };
        std::vector<keep_timeline_event> ev;
        // loads: items of a batch in issue order, sub-intervals by bytes
        std::vector<uint64_t> done(ld.batches.size(), 0);
        for (const auto& r : ld.recs) {
            const Loader::Batch& b = ld.batches[r.batch];
            const double a = at(b.a), e = at(b.b);
            const double span = std::max(0.0, e - a);
            const double s0 = a + span * double(done[r.batch]) / double(std::max<uint64_t>(b.bytes, 1));
            done[r.batch] += r.bytes;
            const double s1 = a + span * double(done[r.batch]) / double(std::max<uint64_t>(b.bytes, 1));
            keep_timeline_event x{};
            x.kind = 0;
            x.layer = r.layer;
            x.owner = keep_owner{ld.units[r.unit].key.kind, ld.units[r.unit].key.id};
            x.bytes = r.bytes;
            x.start_ms = s0;
            x.end_ms = s1;
            ev.push_back(x);
        }
        double frac = 1.0;
        for (int l = 0; l < c.L; ++l) {
            keep_timeline_event x{};
            x.kind = 1;
            x.layer = l;
            x.start_ms = at(ld.comp_start[l]);
            x.end_ms = at(ld.comp_end[l]);
            ev.push_back(x);
            if (ld.has_eval[l]) {
                keep_timeline_event y{};
                y.kind = 2;
                y.layer = l;
                y.start_ms = at(ld.eval_a[l]);
                y.end_ms = at(ld.eval_b[l]);
                ev.push_back(y);
                const double span = x.end_ms - x.start_ms;
                // the walk starts once the summary exists (it waits on that
                // event): the earlier of the two timestamps bounds "attention done"
                if (span > 0.0) frac = std::min(frac, (std::min(at(ld.attn_end[l]), y.start_ms) - x.start_ms) / span);
            }
        }
        for (int i = 0; i < int(ev.size()) && i < cap; ++i) out[i] = ev[i];
        *n_out = int32_t(ev.size());
        if (attention_fraction) *attention_fraction = std::max(0.0, frac);
        return KEEP_OK;
    } catch (const KeepError& e) {
        set_last_error(e.what());
        return e.code;
    }
}
