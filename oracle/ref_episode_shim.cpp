// ref_episode_shim.cpp -- C wrapper over the UNMODIFIED reference episode
// harness (TEST INFRASTRUCTURE ONLY, see keep_oracle.h).
//
// Compiled by oracle/Makefile against /root/reference/proj/include (read in
// place) plus the nlohmann/json header the reference's serialize.hpp
// includes, into oracle/_ref/libkeep_ref_episode.so.  Text in, text out in the
// reference's own formats: EpisodeConfig JSON (config_from_json,
// harness.hpp:172-235), JSONL traces (trace_to_jsonl / trace_from_jsonl,
// 297-322), report_to_json (448-484) and compare_csv (828-871).

#include <cstring>
#include <exception>
#include <string>

#include "keep/harness.hpp"

using namespace keep;

namespace {

thread_local std::string g_err;
thread_local std::string g_out;

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

std::vector<std::string> split(const char* csv) {
    std::vector<std::string> out;
    std::string cur;
    for (const char* p = csv; p && *p; ++p) {
        if (*p == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *p;
        }
    }
    if (!cur.empty()) out.push_back(cur);
    return out;
}

}  // namespace

extern "C" {

const char* kre_last_error() { return g_err.c_str(); }
// result text of the last successful call on this thread
const char* kre_output() { return g_out.c_str(); }

int kre_generate(const char* config_json) {
    return guard([&] { g_out = trace_to_jsonl(generate_episode(config_from_json(Json::parse(config_json)))); });
}

int kre_run_episode(const char* config_json, const char* trace_jsonl, const char* strategy) {
    return guard([&] {
        const EpisodeConfig cfg = config_from_json(Json::parse(config_json));
        g_out = report_to_json(run_episode(trace_from_jsonl(trace_jsonl), strategy, cfg)).dump();
    });
}

// ks / rs: comma-separated sweep points (empty: none)
int kre_compare_csv(const char* config_json, const char* trace_jsonl, const char* strategies, const char* ks,
                    const char* rs) {
    return guard([&] {
        const EpisodeConfig cfg = config_from_json(Json::parse(config_json));
        SweepSpec sw;
        for (const auto& k : split(ks)) sw.ks.push_back(std::stoi(k));
        for (const auto& r : split(rs)) sw.rs.push_back(std::stod(r));
        g_out = compare_csv(trace_from_jsonl(trace_jsonl), split(strategies), cfg, sw);
    });
}

// The MemoryStore alone over a trace, as run_episode drives it (updates,
// then advance_step, then retrievals): one JSON object per step with the
// invalidation records, transitions, the query embedding and its retrieval
// set, and the groups afterwards.
int kre_store_replay(const char* config_json, const char* trace_jsonl) {
    return guard([&] {
        const EpisodeConfig cfg = config_from_json(Json::parse(config_json));
        const auto trace = trace_from_jsonl(trace_jsonl);
        std::vector<MemorySegment> segs;
        std::map<std::int64_t, std::vector<const TraceEvent*>> steps;
        for (const auto& e : trace) {
            if (e.type == TraceEvent::Type::InitSegment) {
                MemorySegment s;
                s.id = e.id;
                s.category = e.category;
                s.tokens = e.tokens;
                s.embedding = e.embedding;
                segs.push_back(s);
            } else {
                steps[e.step].push_back(&e);
            }
        }
        std::vector<MemorySegment> sorted = segs;
        std::sort(sorted.begin(), sorted.end(), [](const auto& a, const auto& b) { return a.id < b.id; });
        std::vector<std::vector<double>> embs;
        for (const auto& s : sorted) embs.push_back(s.embedding);
        MemoryStore store(segs, detail::EpisodeRuntime::store_config(cfg));
        auto groups_json = [&] {
            Json g = Json::array();
            for (const auto& grp : store.groups())
                g.push_back(Json{{"members", grp.member_ids},
                                 {"state", grp.state == GroupState::Static ? "static" : "dynamic"},
                                 {"version", store.group_version(grp.id)}});
            return g;
        };
        std::string out = Json{{"initial_groups", groups_json()}}.dump() + "\n";
        for (const auto& [step, events] : steps) {
            Json js;
            js["step"] = step;
            Json recs = Json::array();
            for (const auto* e : events) {
                if (e->type != TraceEvent::Type::Update) continue;
                const auto r = store.apply_update(e->id, e->tokens, step);
                Json ents = Json::array();
                for (const auto& en : r.entries) ents.push_back(Json{en.owner.str(), en.tokens});
                recs.push_back(Json{{"entries", ents}, {"new_version", r.new_segment_versions.front().second}});
            }
            js["updates"] = recs;
            Json tr = Json::array();
            for (const auto& t : store.advance_step(step)) tr.push_back(Json{t.group, t.new_group_version});
            js["transitions"] = tr;
            Json qs = Json::array();
            for (const auto* e : events) {
                if (e->type != TraceEvent::Type::Query) continue;
                const auto q = derive_query(e->embedding_seed, embs, cfg.query_tokens, cfg.model.vocab_size);
                const auto rs = store.retrieve(q.embedding, e->k);
                Json units = Json::array();
                for (const auto& u : rs.units) units.push_back(Json{u.owner.str(), u.segments});
                qs.push_back(Json{{"embedding", q.embedding}, {"tokens", q.tokens}, {"k", e->k}, {"units", units}});
            }
            js["queries"] = qs;
            js["groups"] = groups_json();
            js["state_sound"] = store.state_sound();
            out += js.dump() + "\n";
        }
        g_out = out;
    });
}

}  // extern "C"
