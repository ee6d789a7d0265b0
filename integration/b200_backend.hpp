// b200_backend.hpp -- the adapter a reference maintainer adds beside the
// reference headers (include/keep/) to run KEEP's per-layer prefill on the
// B200 library (include/keep_b200.h).  Compiled against the UNMODIFIED
// reference headers by integration/Makefile and exercised by
// integration/demo.cpp (tests/test_gpu_integration.py).
//
//   reference                                   B200 (this adapter)
//   Model::init          model.hpp:54-73        B200Model        -> keep_model_init
//   compute_and_put      harness.hpp:512-532    b200_compute_and_put -> keep_memory_compute_batch
//   PrefillCursor::step  prefill.hpp:224-322    B200PrefillCursor::step -> keep_prefill_layer
//   converge             recompute.hpp:130-138  b200_converge    -> keep_importance_evaluation
//   plan_keep            recompute.hpp:140-180  b200_plan_keep (the reference loop over the two
//                                               above) or b200_plan_keep_device (keep_plan_keep:
//                                               the whole loop on the device)
#pragma once

#include <algorithm>
#include <stdexcept>
#include <vector>

#include "keep/errors.hpp"
#include "keep/memory_store.hpp"
#include "keep/prefill.hpp"
#include "keep/recompute.hpp"

extern "C" {
#include "keep_b200.h"
}

namespace keep {

inline void b200_check(int rc) {  // the ABI's codes are errors.hpp:8-26's exceptions
    if (rc == KEEP_OK) return;
    const char* m = keep_last_error();
    switch (rc) {
        case KEEP_ERR_CONFIG: throw ConfigError(m);
        case KEEP_ERR_INPUT: throw InputError(m);
        case KEEP_ERR_PLAN: throw PlanError(m);
        case KEEP_ERR_CACHE_MISS: throw CacheMissError(m);
        case KEEP_ERR_TRACE: throw TraceError(m);
        default: throw std::runtime_error(m);
    }
}

inline keep_owner to_owner(const OwnerRef& o) {
    return {o.kind == OwnerRef::Kind::Group ? KEEP_OWNER_GROUP : KEEP_OWNER_SEGMENT, o.id};
}

// Model::init (model.hpp:54-73): the same counter-based weights, generated on
// the device (bit-identical to the host Model).
class B200Model {
public:
    explicit B200Model(const ModelConfig& c, int numerics = KEEP_NUMERICS_PARITY, int device = 0) {
        keep_config kc{};
        kc.num_layers = c.num_layers;
        kc.num_heads = c.num_heads;
        kc.model_dim = c.model_dim;
        kc.mlp_dim = c.mlp_dim;
        kc.vocab_size = c.vocab_size;
        kc.numerics = numerics;
        kc.seed = c.seed;
        kc.device = device;
        kc.world_size = 1;
        b200_check(keep_ctx_create(&kc, &ctx_));
        b200_check(keep_model_init(ctx_));
    }
    ~B200Model() { keep_ctx_destroy(ctx_); }
    B200Model(const B200Model&) = delete;
    B200Model& operator=(const B200Model&) = delete;
    void* ctx() const { return ctx_; }

private:
    void* ctx_ = nullptr;
};

// A reference Layout plus the owner of each unit (OwnerRef, memory_store.hpp:61-88):
// static groups own one joint block, dynamic segments one block each.
struct B200Layout {
    std::vector<int32_t> seg_len, tokens, ub, ue;
    std::vector<keep_owner> owners;
    B200Layout(const Layout& layout, const std::vector<OwnerRef>& unit_owners) {
        if (unit_owners.size() != layout.units.size()) throw ConfigError("one owner per layout unit");
        for (const auto& s : layout.segments) {
            seg_len.push_back(int32_t(s.tokens.size()));
            tokens.insert(tokens.end(), s.tokens.begin(), s.tokens.end());
        }
        for (size_t u = 0; u < layout.units.size(); ++u) {
            ub.push_back(layout.units[u].first);
            ue.push_back(layout.units[u].second);
            owners.push_back(to_owner(unit_owners[u]));
        }
    }
    keep_layout c() const {
        return keep_layout{int32_t(seg_len.size()), int32_t(ub.size()), seg_len.data(), tokens.data(), ub.data(),
                           ue.data(), owners.data()};
    }
};

// compute_and_put (harness.hpp:512-532) for every unit of a layout: standalone
// KV per dynamic segment, one joint prefill per static group, on the device.
inline void b200_compute_and_put(const B200Model& m, const B200Layout& bl, uint64_t version) {
    std::vector<uint64_t> versions(bl.owners.size(), version);
    std::vector<int32_t> members;
    for (size_t u = 0; u < bl.owners.size(); ++u) members.push_back(bl.ue[u] - bl.ub[u]);
    b200_check(keep_memory_compute_batch(m.ctx(), int32_t(bl.owners.size()), bl.owners.data(), versions.data(),
                                         members.data(), bl.seg_len.data(), bl.tokens.data(), KEEP_TIER_DEVICE));
}

// PrefillCursor (prefill.hpp:174-337): step() returns the layer's summary.
class B200PrefillCursor {
public:
    B200PrefillCursor(const B200Model& m, const B200Layout& bl, const TokenSeq& query)
        : ctx_(m.ctx()), S_(bl.seg_len.size()) {
        const keep_layout kl = bl.c();
        std::vector<int32_t> q(query.begin(), query.end());
        b200_check(keep_prefill_begin(ctx_, &kl, q.data(), int32_t(q.size())));
        summary_.query_to_segment.assign(S_, 0.0);
        summary_.segment_to_segment.assign(S_, std::vector<double>(S_, 0.0));
    }
    const AttentionSummary& step(const std::vector<char>& active) {  // prefill.hpp:224
        std::vector<uint8_t> a(active.begin(), active.end());
        std::vector<double> raw(S_ + S_ * S_);
        b200_check(keep_prefill_layer(ctx_, a.data(), raw.data()));
        std::copy(raw.begin(), raw.begin() + S_, summary_.query_to_segment.begin());
        for (size_t i = 0; i < S_; ++i)
            std::copy(raw.begin() + S_ + i * S_, raw.begin() + S_ + (i + 1) * S_,
                      summary_.segment_to_segment[i].begin());
        summary_.layer = layer_++;
        return summary_;
    }
    std::vector<float> finish(int T, int d) {  // final_hidden (prefill.hpp:324-337)
        std::vector<float> fh(size_t(T) * d);
        b200_check(keep_prefill_finish(ctx_, fh.data(), nullptr));
        return fh;
    }

private:
    void* ctx_;
    size_t S_;
    int layer_ = 0;
    AttentionSummary summary_;
};

// converge (recompute.hpp:130-138) on the device selector.
inline ImportanceState b200_converge(void* ctx, const AttentionSummary& s, std::size_t budget,
                                     const std::vector<char>* candidates) {
    const int32_t S = int32_t(s.query_to_segment.size());
    std::vector<double> sts(size_t(S) * S);
    for (int i = 0; i < S; ++i)
        std::copy(s.segment_to_segment[i].begin(), s.segment_to_segment[i].end(), sts.begin() + size_t(i) * S);
    std::vector<uint8_t> cand;
    if (candidates) cand.assign(candidates->begin(), candidates->end());
    std::vector<int32_t> order(size_t(std::max(S, 1)));
    int32_t n = 0, hops = 0;
    b200_check(keep_importance_evaluation(ctx, S, s.query_to_segment.data(), sts.data(), int64_t(budget),
                                          candidates ? cand.data() : nullptr, order.data(), &n, &hops));
    ImportanceState st;
    st.relevant_order.assign(order.begin(), order.begin() + n);
    st.relevant.insert(st.relevant_order.begin(), st.relevant_order.end());
    st.hop = hops;
    return st;
}

// plan_keep (recompute.hpp:140-180): the reference's own loop, with the cursor
// and the selector on the B200.
inline RecomputePlan b200_plan_keep(const B200Model& m, const Layout& layout, const B200Layout& bl,
                                    const TokenSeq& query, const RatioSchedule& schedule, bool multihop = true) {
    const int L = schedule.num_layers();
    const int S = int(layout.num_segments());
    RecomputePlan plan;
    plan.layers.resize(L);
    std::vector<char> active(size_t(S), 1);
    B200PrefillCursor cursor(m, bl, query);
    for (int l = 0; l < L; ++l) {
        for (int i = 0; i < S; ++i)
            if (active[i]) plan.layers[l].insert(layout.segments[i].id);
        const AttentionSummary& summary = cursor.step(active);
        if (l + 1 >= L) break;
        const std::size_t budget = layer_budget(schedule.r[l + 1], S);
        std::size_t live = 0;
        for (char a : active) live += a;
        if (budget >= live) continue;
        std::vector<char> next(size_t(S), 0);
        if (multihop) {
            for (int i : b200_converge(m.ctx(), summary, budget, &active).relevant_order) next[i] = 1;
        } else {
            std::vector<int> order;
            for (int i = 0; i < S; ++i)
                if (active[i]) order.push_back(i);
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
                return summary.query_to_segment[a] > summary.query_to_segment[b];
            });
            for (std::size_t i = 0; i < budget && i < order.size(); ++i) next[order[i]] = 1;
        }
        active = std::move(next);
    }
    return plan;
}

// The whole loop as one device call (keep_plan_keep): selector overlap, no
// per-layer summary transfer.  The serving path.
inline RecomputePlan b200_plan_keep_device(const B200Model& m, const Layout& layout, const B200Layout& bl,
                                           const TokenSeq& query, const RatioSchedule& schedule,
                                           bool multihop = true) {
    const int L = schedule.num_layers();
    const int S = int(layout.num_segments());
    std::vector<uint8_t> pm(size_t(L) * S);
    keep_plan_result res{};
    res.plan = pm.data();
    const keep_layout kl = bl.c();
    std::vector<int32_t> q(query.begin(), query.end());
    b200_check(keep_plan_keep(m.ctx(), &kl, q.data(), int32_t(q.size()), schedule.r.data(), multihop ? 1 : 0, &res));
    RecomputePlan plan;
    plan.layers.resize(L);
    for (int l = 0; l < L; ++l)
        for (int i = 0; i < S; ++i)
            if (pm[size_t(l) * S + i]) plan.layers[l].insert(layout.segments[i].id);
    return plan;
}

}  // namespace keep
