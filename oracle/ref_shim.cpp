// ref_shim.cpp -- C wrapper over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see keep_oracle.h).  Compiled by oracle/Makefile
// against /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libkeep_ref.so.  Every kr_* entry point forwards to the
// reference's own functions; the only code here is marshalling between flat
// buffers and the reference's Mat / Layout / CachedKV types.

#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "keep/cache_manager.hpp"
#include "keep/pipeline_sim.hpp"
#include "keep/recompute.hpp"

#include "keep_oracle.h"

using namespace keep;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const InputError& e) {
        g_err = e.what();
        return 2;
    } catch (const PlanError& e) {
        g_err = e.what();
        return 3;
    } catch (const CacheMissError& e) {
        g_err = e.what();
        return 4;
    } catch (const TraceError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

ModelConfig cfg_of(const keep_problem* p) {
    ModelConfig c;
    c.num_layers = p->num_layers;
    c.num_heads = p->num_heads;
    c.model_dim = p->model_dim;
    c.mlp_dim = p->mlp_dim;
    c.vocab_size = p->vocab_size;
    c.seed = p->seed;
    return c;
}

void copy_in(Mat& m, int r, int c, const float*& src) {
    m = Mat(r, c);
    std::memcpy(m.a.data(), src, sizeof(float) * static_cast<size_t>(r) * c);
    src += static_cast<size_t>(r) * c;
}

void copy_out(const Mat& m, float*& dst) {
    std::memcpy(dst, m.a.data(), sizeof(float) * m.a.size());
    dst += m.a.size();
}

// Model from a weight buffer (same layout Model::init produces, see header).
Model model_from(const keep_problem* p, const float* w) {
    Model m;
    m.cfg = cfg_of(p);
    m.cfg.validate();
    const int d = m.cfg.model_dim, f = m.cfg.mlp_dim, V = m.cfg.vocab_size;
    copy_in(m.embedding, V, d, w);
    copy_in(m.unembed, d, V, w);
    m.layers.resize(m.cfg.num_layers);
    for (auto& lw : m.layers) {
        copy_in(lw.wq, d, d, w);
        copy_in(lw.wk, d, d, w);
        copy_in(lw.wv, d, d, w);
        copy_in(lw.wo, d, d, w);
        copy_in(lw.mlp_in, d, f, w);
        copy_in(lw.mlp_out, f, d, w);
    }
    return m;
}

Layout layout_from(const keep_problem* p) {
    std::vector<LayoutSegment> segs;
    const int32_t* t = p->tokens;
    for (int i = 0; i < p->num_segments; ++i) {
        LayoutSegment s;
        s.id = static_cast<SegmentId>(i);
        s.tokens.assign(t, t + p->seg_len[i]);
        t += p->seg_len[i];
        segs.push_back(std::move(s));
    }
    Layout l = Layout::of(std::move(segs));
    if (p->num_units > 0) {
        l.units.clear();
        for (int u = 0; u < p->num_units; ++u) l.units.emplace_back(p->unit_begin[u], p->unit_end[u]);
    }
    return l;
}

TokenSeq query_from(const keep_problem* p) {
    return TokenSeq(p->query, p->query + p->query_len);
}

// Canonical KV per segment: standalone segment_prefill for dynamic units, one
// joint full_prefill sliced per member for static groups (harness.hpp:512-532,
// 659-677).
CachedKV canonical_from_units(const Model& m, const Layout& layout, const keep_problem* p) {
    CachedKV cached;
    const int L = m.cfg.num_layers, d = m.cfg.model_dim;
    auto dyn = [&](int i) {
        cached[layout.segments[i].id] = segment_prefill(m, layout.segments[i].tokens);
    };
    if (p->num_units == 0) {
        for (int i = 0; i < static_cast<int>(layout.segments.size()); ++i) dyn(i);
        return cached;
    }
    for (int u = 0; u < p->num_units; ++u) {
        const int b = p->unit_begin[u], e = p->unit_end[u];
        if (!p->unit_is_group[u]) {
            for (int i = b; i < e; ++i) dyn(i);
            continue;
        }
        Layout members;
        for (int i = b; i < e; ++i) members.segments.push_back(layout.segments[i]);
        members.units.emplace_back(0, e - b);
        const auto kv = full_prefill(m, members, {}).kv;
        int off = 0;
        for (int i = b; i < e; ++i) {
            const int n = static_cast<int>(layout.segments[i].tokens.size());
            std::vector<LayerKV> per;
            for (int l = 0; l < L; ++l) {
                LayerKV s{Mat(n, d), Mat(n, d)};
                for (int r = 0; r < n; ++r) {
                    std::memcpy(s.keys.row_ptr(r), kv[l].keys.row_ptr(off + r), sizeof(float) * d);
                    std::memcpy(s.values.row_ptr(r), kv[l].values.row_ptr(off + r), sizeof(float) * d);
                }
                per.push_back(std::move(s));
            }
            cached[layout.segments[i].id] = std::move(per);
            off += n;
        }
    }
    return cached;
}

// Flat cached buffer (per layer keys[Tm*d], values[Tm*d]) <-> CachedKV.
CachedKV cached_from_flat(const Model& m, const Layout& layout, const float* flat) {
    CachedKV cached;
    const int L = m.cfg.num_layers, d = m.cfg.model_dim;
    const size_t Tm = layout.total_tokens();
    size_t row = 0;
    for (const auto& seg : layout.segments) {
        const int n = static_cast<int>(seg.tokens.size());
        std::vector<LayerKV> per;
        for (int l = 0; l < L; ++l) {
            const float* kb = flat + static_cast<size_t>(l) * 2 * Tm * d;
            const float* vb = kb + Tm * d;
            LayerKV s{Mat(n, d), Mat(n, d)};
            std::memcpy(s.keys.a.data(), kb + row * d, sizeof(float) * n * d);
            std::memcpy(s.values.a.data(), vb + row * d, sizeof(float) * n * d);
            per.push_back(std::move(s));
        }
        cached[seg.id] = std::move(per);
        row += n;
    }
    return cached;
}

void summaries_out(const std::vector<AttentionSummary>& attn, int S, double* out) {
    if (!out) return;
    for (const auto& a : attn) {
        for (int j = 0; j < S; ++j) *out++ = a.query_to_segment[j];
        for (int i = 0; i < S; ++i)
            for (int j = 0; j < S; ++j) *out++ = a.segment_to_segment[i][j];
    }
}

void result_out(const PrefillResult& r, float* final_hidden, float* kv, double* summaries, int S) {
    if (final_hidden) {
        float* fh = final_hidden;
        copy_out(r.final_hidden, fh);
    }
    if (kv) {
        float* o = kv;
        for (const auto& lk : r.kv) {
            copy_out(lk.keys, o);
            copy_out(lk.values, o);
        }
    }
    summaries_out(r.attn, S, summaries);
}

RecomputePlan plan_from_mask(const Layout& layout, const uint8_t* mask, int L) {
    RecomputePlan plan;
    plan.layers.resize(L);
    const int S = static_cast<int>(layout.segments.size());
    for (int l = 0; l < L; ++l)
        for (int i = 0; i < S; ++i)
            if (mask[l * S + i]) plan.layers[l].insert(layout.segments[i].id);
    return plan;
}

}  // namespace

extern "C" {

const char* kr_last_error(void) { return g_err.c_str(); }

uint64_t kr_weight_count(int L, int H, int d, int mlp, int V) {
    (void)H;
    return 2ull * V * d + static_cast<uint64_t>(L) * (4ull * d * d + 2ull * d * mlp);
}

int kr_model_init(int L, int H, int d, int mlp, int V, uint64_t seed, float* w) {
    return guard([&] {
        ModelConfig c{L, H, d, mlp, V, seed};
        const Model m = Model::init(c);
        float* o = w;
        copy_out(m.embedding, o);
        copy_out(m.unembed, o);
        for (const auto& lw : m.layers) {
            copy_out(lw.wq, o);
            copy_out(lw.wk, o);
            copy_out(lw.wv, o);
            copy_out(lw.wo, o);
            copy_out(lw.mlp_in, o);
            copy_out(lw.mlp_out, o);
        }
    });
}

// Layout part of testutil::make_instance (tests/test_util.hpp:19-40): the
// same Rng stream and draw order, without building the model.
int kr_make_instance_layout(uint64_t seed, int S, int V, int lo, int hi, int qlen,
                            int32_t* seg_len, int32_t* tokens, int32_t* query) {
    return guard([&] {
        Rng rng = Rng::stream(seed, "instance");
        int32_t* t = tokens;
        for (int i = 0; i < S; ++i) {
            const int n = lo + static_cast<int>(rng.next_below(hi - lo + 1));
            seg_len[i] = n;
            for (int k = 0; k < n; ++k) *t++ = static_cast<int32_t>(rng.next_below(V));
        }
        for (int k = 0; k < qlen; ++k) query[k] = static_cast<int32_t>(rng.next_below(V));
    });
}

int kr_ratio_schedule(int L, double r_avg, double* r_out) {
    return guard([&] {
        const auto s = ratio_schedule(L, r_avg);
        for (int l = 0; l < L; ++l) r_out[l] = s.r[l];
    });
}

int64_t kr_layer_budget(double ratio, int64_t S) {
    return static_cast<int64_t>(layer_budget(ratio, static_cast<std::size_t>(S)));
}

int kr_converge(int S, const double* qts, const double* sts, int64_t budget,
                const uint8_t* candidates, int32_t* order_out, int32_t* n_out, int32_t* hops_out) {
    return guard([&] {
        AttentionSummary a;
        a.query_to_segment.assign(qts, qts + S);
        a.segment_to_segment.resize(S);
        for (int i = 0; i < S; ++i) a.segment_to_segment[i].assign(sts + static_cast<size_t>(i) * S, sts + static_cast<size_t>(i + 1) * S);
        std::vector<char> cand;
        if (candidates) cand.assign(candidates, candidates + S);
        const auto st = converge(a, static_cast<std::size_t>(budget), candidates ? &cand : nullptr);
        *n_out = static_cast<int32_t>(st.relevant_order.size());
        for (size_t k = 0; k < st.relevant_order.size(); ++k) order_out[k] = st.relevant_order[k];
        *hops_out = st.hop;
    });
}

int kr_canonical_kv(const keep_problem* p, const float* w, float* kv_out) {
    return guard([&] {
        const Model m = model_from(p, w);
        const Layout layout = layout_from(p);
        const CachedKV cached = canonical_from_units(m, layout, p);
        const int L = m.cfg.num_layers, d = m.cfg.model_dim;
        const size_t Tm = layout.total_tokens();
        size_t row = 0;
        for (const auto& seg : layout.segments) {
            const auto& per = cached.at(seg.id);
            const size_t n = seg.tokens.size();
            for (int l = 0; l < L; ++l) {
                float* kb = kv_out + static_cast<size_t>(l) * 2 * Tm * d;
                float* vb = kb + Tm * d;
                std::memcpy(kb + row * d, per[l].keys.a.data(), sizeof(float) * n * d);
                std::memcpy(vb + row * d, per[l].values.a.data(), sizeof(float) * n * d);
            }
            row += n;
        }
    });
}

int kr_full_prefill(const keep_problem* p, const float* w, float* final_hidden, float* kv,
                    double* summaries) {
    return guard([&] {
        const Model m = model_from(p, w);
        const Layout layout = layout_from(p);
        const auto r = full_prefill(m, layout, query_from(p));
        result_out(r, final_hidden, kv, summaries, p->num_segments);
    });
}

int kr_selective_prefill(const keep_problem* p, const float* w, const float* cached_flat,
                         const uint8_t* plan_mask, float* final_hidden, float* kv,
                         double* summaries) {
    return guard([&] {
        const Model m = model_from(p, w);
        const Layout layout = layout_from(p);
        const CachedKV cached = cached_flat ? cached_from_flat(m, layout, cached_flat)
                                            : canonical_from_units(m, layout, p);
        const RecomputePlan plan = plan_from_mask(layout, plan_mask, m.cfg.num_layers);
        const auto r = selective_prefill(m, layout, cached, plan, query_from(p));
        result_out(r, final_hidden, kv, summaries, p->num_segments);
    });
}

// plan_keep (recompute.hpp:140-180).  The reference returns only the plan, so
// the per-layer walk is re-driven here through the reference's own
// PrefillCursor / layer_budget / converge to expose relevant_order and hop,
// and the result is cross-checked against the real plan_keep (code 9 on any
// mismatch).  The final hidden state / merged KV come from
// selective_prefill(plan), as run_strategy does (recompute.hpp:318).
int kr_plan_keep(const keep_problem* p, const float* w, const float* cached_flat,
                 const double* sched, int multihop, uint8_t* plan_out, int32_t* orders,
                 int32_t* order_len, int32_t* hops, double* summaries, float* final_hidden,
                 float* kv) {
    return guard([&] {
        const Model m = model_from(p, w);
        const Layout layout = layout_from(p);
        const TokenSeq query = query_from(p);
        const CachedKV cached = cached_flat ? cached_from_flat(m, layout, cached_flat)
                                            : canonical_from_units(m, layout, p);
        const int L = m.cfg.num_layers, S = p->num_segments;
        RatioSchedule rs;
        rs.r.assign(sched, sched + L);

        std::memset(plan_out, 0, static_cast<size_t>(L) * S);
        for (int l = 0; l < L; ++l) {
            order_len[l] = -1;
            hops[l] = 0;
        }
        std::vector<char> active(S, 1);
        PrefillCursor cursor(m, layout, &cached, query);
        std::vector<AttentionSummary> attn;
        for (int l = 0; l < L; ++l) {
            for (int i = 0; i < S; ++i) plan_out[l * S + i] = active[i] ? 1 : 0;
            const AttentionSummary& summary = cursor.step(active);
            attn.push_back(summary);
            if (l + 1 >= L) break;
            const std::size_t budget = layer_budget(rs.r[l + 1], S);
            std::size_t active_count = 0;
            for (char a : active) active_count += a;
            if (budget >= active_count) continue;
            std::vector<char> next(S, 0);
            if (multihop) {
                const ImportanceState st = converge(summary, budget, &active);
                for (int i : st.relevant_order) next[i] = 1;
                order_len[l] = static_cast<int32_t>(st.relevant_order.size());
                for (size_t k = 0; k < st.relevant_order.size(); ++k)
                    orders[static_cast<size_t>(l) * S + k] = st.relevant_order[k];
                hops[l] = st.hop;
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
        summaries_out(attn, S, summaries);

        const RecomputePlan ref = plan_keep(m, layout, cached, query, rs, multihop != 0);
        const RecomputePlan mine = plan_from_mask(layout, plan_out, L);
        if (ref.layers != mine.layers) throw std::runtime_error("shim plan differs from plan_keep");

        if (final_hidden || kv) {
            const auto r = selective_prefill(m, layout, cached, ref, query);
            result_out(r, final_hidden, kv, nullptr, S);
        }
    });
}

int kr_divergence(const keep_problem* p, const float* w, const float* row_a, const float* row_b,
                  double* l2, double* sym_kl) {
    return guard([&] {
        const Model m = model_from(p, w);
        Mat a(1, m.cfg.model_dim), b(1, m.cfg.model_dim);
        std::memcpy(a.a.data(), row_a, sizeof(float) * m.cfg.model_dim);
        std::memcpy(b.a.data(), row_b, sizeof(float) * m.cfg.model_dim);
        const Divergence dv = divergence(m, a, b);
        *l2 = dv.l2;
        *sym_kl = dv.sym_kl;
    });
}

int kr_logits(const keep_problem* p, const float* w, const float* row, double* out) {
    return guard([&] {
        const Model m = model_from(p, w);
        const auto lg = m.logits(row);
        std::memcpy(out, lg.data(), sizeof(double) * lg.size());
    });
}

// validate_timeline (pipeline_sim.hpp:340-428) on a realised GPU timeline:
// the workload is the reference's own derive_workload (103-154) over the plan
// and the load units; the timeline's events are the device's.  codes_out gets
// the violation codes (D1 D2 R P S), space separated ("" = valid).
int kr_validate_timeline(int L, int S, const uint8_t* plan, const int32_t* seg_len, int query_tokens, int n_units,
                         const int32_t* unit_begin, const int32_t* unit_end, const int32_t* unit_is_group,
                         const uint32_t* unit_owner_id, const uint64_t* slow_bytes, double attention_fraction,
                         const kr_timeline_event* ev, int n_ev, char* codes_out, int cap) {
    return guard([&] {
        RecomputePlan rp;
        rp.layers.resize(L);
        for (int l = 0; l < L; ++l)
            for (int i = 0; i < S; ++i)
                if (plan[size_t(l) * S + i]) rp.layers[l].insert(SegmentId(i));
        std::vector<LayoutSegment> segs;
        for (int i = 0; i < S; ++i) {
            LayoutSegment sg;
            sg.id = SegmentId(i);
            sg.tokens.assign(size_t(seg_len[i]), 0);
            segs.push_back(std::move(sg));
        }
        const Layout layout = Layout::of(std::move(segs));
        std::vector<LoadUnit> units;
        for (int u = 0; u < n_units; ++u) {
            LoadUnit lu;
            lu.owner = unit_is_group[u] ? OwnerRef::group(unit_owner_id[u]) : OwnerRef::segment(unit_owner_id[u]);
            for (int i = unit_begin[u]; i < unit_end[u]; ++i) lu.segments.push_back(SegmentId(i));
            lu.slow_bytes.assign(slow_bytes + size_t(u) * L, slow_bytes + size_t(u + 1) * L);
            units.push_back(std::move(lu));
        }
        CostModel cost;
        cost.attention_fraction = attention_fraction;
        const Workload w = derive_workload(rp, layout, units, size_t(query_tokens), cost, 1.0, true);
        Timeline tl;
        for (int i = 0; i < n_ev; ++i) {
            SimEvent e;
            e.kind = ev[i].kind == 0 ? SimKind::Load : (ev[i].kind == 1 ? SimKind::Compute : SimKind::Eval);
            e.resource = ev[i].kind == 0 ? SimResource::LoadEngine
                                         : (ev[i].kind == 1 ? SimResource::ComputeEngine : SimResource::EvalEngine);
            e.layer = ev[i].layer;
            e.owner = ev[i].owner_kind ? OwnerRef::group(ev[i].owner_id) : OwnerRef::segment(ev[i].owner_id);
            e.bytes = ev[i].bytes;
            e.start = ev[i].start;
            e.end = ev[i].end;
            tl.events.push_back(e);
            tl.makespan = std::max(tl.makespan, e.end);
        }
        const auto vio = validate_timeline(tl, rp, w);
        std::string codes;
        for (const auto& v : vio) codes += (codes.empty() ? "" : " ") + v.code;
        if (cap > 0) {
            std::strncpy(codes_out, codes.c_str(), size_t(cap - 1));
            codes_out[cap - 1] = 0;
        }
    });
}

}  // extern "C"
