// episode.cpp -- the memory control plane and episode replay (SURVEY.md
// 8(f4); include/keep_episode.h) over the B200 prefill engine.
//
// A client of the C ABI (keep_b200.h), as the reference's harness is a client
// of its cursor and cache manager:
//   * MemoryStore (memory_store.hpp:274-496): seeded k-means grouping, the
//     t-step static/dynamic state machine, invalidation records, retrieval;
//   * TierBook: CacheManager's block bookkeeping -- (owner, layer) keys,
//     versions, fast-tier capacity with LRU demotion, slow-load accounting
//     (cache_manager.hpp:60-228).  The payloads it books are the device
//     memory tier's blocks (keep_memory_compute_batch / keep_invalidate);
//   * the load/compute pipeline model that turns a plan into TTFT time units
//     (pipeline_sim.hpp:103-428);
//   * run_episode / compare_csv (harness.hpp:543-871).
// Plans, prefills, logits and divergences are computed on the GPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "keep_b200.h"
#include "keep_episode.h"

namespace keep_b200 {
void set_last_error(const std::string& msg);
}

namespace {

struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& m) { throw Err(code, m); }

void ck(int rc) {  // a nested keep_* call failed: carry its code and message
    if (rc != KEEP_OK) fail(rc, keep_last_error());
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return KEEP_OK;
    } catch (const Err& e) {
        keep_b200::set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        keep_b200::set_last_error("host out of memory");
        return KEEP_ERR_CUDA;
    } catch (const std::exception& e) {
        keep_b200::set_last_error(e.what());
        return KEEP_ERR_CUDA;
    }
}

using Tokens = std::vector<int32_t>;

// ----------------------------------------------------------------- Rng --
// Named splitmix64 streams, Irwin-Hall gaussians (prng.hpp:16-82).
uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t fnv(const std::string& s) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    return h;
}
struct Rng {
    uint64_t st;
    explicit Rng(uint64_t seed) : st(seed) {
        splitmix(st);
        splitmix(st);
    }
    static Rng stream(uint64_t seed, const std::string& name) { return Rng(seed ^ fnv(name)); }
    uint64_t u64() { return splitmix(st); }
    uint64_t below(uint64_t n) { return u64() % n; }
    double uniform() { return double(u64() >> 11) * 0x1.0p-53; }
    double gaussian() {
        double a = 0.0;
        for (int i = 0; i < 12; ++i) a += uniform();
        return a - 6.0;
    }
    std::vector<double> unit_vector(size_t dim) {
        std::vector<double> v(dim);
        double n2 = 0.0;
        do {
            n2 = 0.0;
            for (auto& x : v) {
                x = gaussian();
                n2 += x * x;
            }
        } while (n2 < 1e-12);
        const double inv = 1.0 / std::sqrt(n2);
        for (auto& x : v) x *= inv;
        return v;
    }
};

Tokens random_tokens(Rng& r, int n, int vocab) {
    Tokens t(static_cast<size_t>(n));
    for (auto& x : t) x = int32_t(r.below(uint64_t(vocab)));
    return t;
}

// --------------------------------------------------------------- owners --
struct Owner {  // OwnerRef (memory_store.hpp:61-88): segments order before groups
    int kind = KEEP_OWNER_SEGMENT;
    uint32_t id = 0;
    bool operator==(const Owner& o) const { return kind == o.kind && id == o.id; }
    bool operator<(const Owner& o) const { return kind != o.kind ? kind < o.kind : id < o.id; }
    keep_owner c() const { return keep_owner{kind, id}; }
    std::string str() const { return (kind == KEEP_OWNER_SEGMENT ? "s" : "g") + std::to_string(id); }
};

// ---------------------------------------------------------- MemoryStore --
struct Segment {
    uint32_t id = 0;
    std::string category;
    Tokens tokens;
    std::vector<double> emb;
    uint64_t version = 1;
    int64_t last_update_step = 0;
};
struct Group {
    uint32_t id = 0;
    std::vector<uint32_t> members;  // ascending
    bool is_static = false;
    int64_t last_change_step = 0;
};
struct Invalidation {
    std::vector<std::pair<Owner, uint64_t>> entries;  // owner, tokens
    std::vector<std::pair<uint32_t, uint64_t>> new_versions;
};
struct Transition {
    uint32_t group;
    std::vector<uint32_t> members;
    uint64_t version;
};
struct Unit {  // RetrievalUnit
    Owner owner;
    std::vector<uint32_t> segments;
};

double dot(const std::vector<double>& a, const std::vector<double>& b) {
    double acc = 0.0;
    for (size_t i = 0; i < a.size(); ++i) acc += a[i] * b[i];
    return acc;
}
double sqdist(const std::vector<double>& a, const std::vector<double>& b) {
    double acc = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

// Seeded k-means++ (memory_store.hpp:137-236): lowest center wins ties, an
// empty cluster is reseeded with the point farthest from its center.
std::vector<int> kmeans(const std::vector<std::vector<double>>& pts, int k, uint64_t seed) {
    const int n = int(pts.size());
    Rng rng = Rng::stream(seed, "kmeans");
    std::vector<std::vector<double>> ctr;
    ctr.push_back(pts[rng.below(uint64_t(n))]);
    std::vector<double> d2(static_cast<size_t>(n));
    while (int(ctr.size()) < k) {
        double total = 0.0;
        for (int i = 0; i < n; ++i) {
            double best = 1e300;
            for (const auto& c : ctr) best = std::min(best, sqdist(pts[i], c));
            d2[i] = best;
            total += best;
        }
        int pick = 0;
        if (total > 0.0) {
            const double target = rng.uniform() * total;
            double run = 0.0;
            for (int i = 0; i < n; ++i) {
                run += d2[i];
                if (run >= target) {
                    pick = i;
                    break;
                }
            }
        } else {
            pick = int(rng.below(uint64_t(n)));
        }
        ctr.push_back(pts[pick]);
    }
    std::vector<int> as(static_cast<size_t>(n), 0);
    for (int it = 0; it < 100; ++it) {
        bool changed = false;
        for (int i = 0; i < n; ++i) {
            int best = 0;
            double bd = sqdist(pts[i], ctr[0]);
            for (int c = 1; c < k; ++c) {
                const double d = sqdist(pts[i], ctr[c]);
                if (d < bd) {
                    bd = d;
                    best = c;
                }
            }
            if (as[i] != best) {
                as[i] = best;
                changed = true;
            }
        }
        for (int c = 0; c < k; ++c) {
            std::vector<double> mean(pts[0].size(), 0.0);
            int cnt = 0;
            for (int i = 0; i < n; ++i) {
                if (as[i] != c) continue;
                ++cnt;
                for (size_t j = 0; j < mean.size(); ++j) mean[j] += pts[i][j];
            }
            if (cnt == 0) {
                int far = 0;
                double fd = -1.0;
                for (int i = 0; i < n; ++i) {
                    const double d = sqdist(pts[i], ctr[as[i]]);
                    if (d > fd) {
                        fd = d;
                        far = i;
                    }
                }
                ctr[c] = pts[far];
                as[far] = c;
                changed = true;
            } else {
                for (auto& v : mean) v /= cnt;
                ctr[c] = std::move(mean);
            }
        }
        if (!changed) break;
    }
    return as;
}

struct StoreCfg {
    int t = 10, num_groups = 1;
    uint64_t seed = 0;
    bool fixed = false;  // GroupingMode::FixedBlocks
    void validate() const {
        if (t < 1) fail(KEEP_ERR_CONFIG, "stability window t must be >= 1");
        if (num_groups < 1) fail(KEEP_ERR_CONFIG, "num_groups must be >= 1");
    }
};

class Store {
public:
    Store(std::vector<Segment> segs, const StoreCfg& cfg) : cfg_(cfg) {
        cfg_.validate();
        for (auto& s : segs) {
            check_embedding(s.emb);
            if (!seg_.emplace(s.id, std::move(s)).second) fail(KEEP_ERR_CONFIG, "duplicate segment id");
        }
        cluster();
        gver_.assign(groups_.size(), 0);
        reindex();
    }

    const std::vector<Group>& groups() const { return groups_; }
    uint64_t group_version(uint32_t g) const { return gver_.at(g); }
    const Segment& segment(uint32_t id) const {
        auto it = seg_.find(id);
        if (it == seg_.end()) fail(KEEP_ERR_INPUT, "unknown segment " + std::to_string(id));
        return it->second;
    }
    uint64_t version(const Owner& o) const {
        return o.kind == KEEP_OWNER_SEGMENT ? segment(o.id).version : group_version(o.id);
    }

    // memory_store.hpp:309-341
    Invalidation apply_update(uint32_t id, Tokens toks, int64_t step) {
        auto it = seg_.find(id);
        if (it == seg_.end()) fail(KEEP_ERR_INPUT, "unknown segment " + std::to_string(id));
        if (step < cur_step_) fail(KEEP_ERR_INPUT, "update step moves backwards");
        Segment& s = it->second;
        Group& g = groups_[gidx(id)];
        Invalidation rec;
        if (cfg_.fixed) {  // positional: the segment and every later member of its block
            for (uint32_t m : g.members)
                if (m >= id) rec.entries.push_back({Owner{KEEP_OWNER_SEGMENT, m}, seg_.at(m).tokens.size()});
        } else if (g.is_static) {
            uint64_t tot = 0;
            for (uint32_t m : g.members) tot += seg_.at(m).tokens.size();
            rec.entries.push_back({Owner{KEEP_OWNER_GROUP, g.id}, tot});
        } else {
            rec.entries.push_back({Owner{KEEP_OWNER_SEGMENT, id}, s.tokens.size()});
        }
        s.tokens = std::move(toks);
        s.version += 1;
        s.last_update_step = step;
        g.is_static = false;
        g.last_change_step = step;
        cur_step_ = std::max(cur_step_, step);
        rec.new_versions.emplace_back(id, s.version);
        return rec;
    }

    // memory_store.hpp:343-367
    std::vector<Transition> advance_step(int64_t step) {
        if (step <= last_adv_) fail(KEEP_ERR_INPUT, "advance_step must strictly increase");
        last_adv_ = step;
        cur_step_ = std::max(cur_step_, step);
        std::vector<Transition> out;
        if (cfg_.fixed) return out;
        for (auto& g : groups_) {
            if (g.is_static) continue;
            int64_t newest = 0;
            for (uint32_t m : g.members) newest = std::max(newest, seg_.at(m).last_update_step);
            if (newest <= step - cfg_.t) {
                g.is_static = true;
                g.last_change_step = step;
                gver_[g.id] += 1;
                out.push_back({g.id, g.members, gver_[g.id]});
            }
        }
        return out;
    }

    // memory_store.hpp:372-418: static groups scored by their best member and
    // taken whole, dynamic segments individually, until k segments are covered
    std::vector<Unit> retrieve(const std::vector<double>& q, int k) const {
        if (k < 1) fail(KEEP_ERR_INPUT, "retrieval k must be >= 1");
        if (seg_.empty()) fail(KEEP_ERR_INPUT, "retrieve on empty store");
        struct Cand {
            double score;
            Unit u;
        };
        std::vector<Cand> cands;
        for (const auto& g : groups_) {
            if (g.is_static) {
                double best = -2.0;
                for (uint32_t m : g.members) best = std::max(best, dot(q, seg_.at(m).emb));
                cands.push_back({best, Unit{Owner{KEEP_OWNER_GROUP, g.id}, g.members}});
            } else {
                for (uint32_t m : g.members)
                    cands.push_back({dot(q, seg_.at(m).emb), Unit{Owner{KEEP_OWNER_SEGMENT, m}, {m}}});
            }
        }
        std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
            if (a.score != b.score) return a.score > b.score;
            return a.u.owner < b.u.owner;
        });
        std::vector<Unit> picked;
        size_t covered = 0;
        for (const auto& c : cands) {
            if (covered >= static_cast<size_t>(k)) break;
            picked.push_back(c.u);
            covered += c.u.segments.size();
        }
        std::sort(picked.begin(), picked.end(), [](const Unit& a, const Unit& b) {
            const bool ag = a.owner.kind == KEEP_OWNER_GROUP, bg = b.owner.kind == KEEP_OWNER_GROUP;
            if (ag != bg) return ag;
            return a.owner.id < b.owner.id;
        });
        return picked;
    }

    // memory_store.hpp:420-452
    void add_segment(Segment s, int64_t step) {
        check_embedding(s.emb);
        if (seg_.count(s.id)) fail(KEEP_ERR_CONFIG, "duplicate segment id");
        s.last_update_step = step;
        size_t bg = 0;
        if (cfg_.fixed) {
            bg = groups_.size() - 1;
        } else {
            double best = -2.0;
            for (size_t g = 0; g < groups_.size(); ++g) {
                std::vector<double> c(s.emb.size(), 0.0);
                for (uint32_t m : groups_[g].members)
                    for (size_t j = 0; j < c.size(); ++j) c[j] += seg_.at(m).emb[j];
                const double nrm = std::sqrt(std::max(1e-12, dot(c, c)));
                for (auto& v : c) v /= nrm;
                const double sc = dot(s.emb, c);
                if (sc > best) {
                    best = sc;
                    bg = g;
                }
            }
        }
        auto& g = groups_[bg];
        g.members.push_back(s.id);
        std::sort(g.members.begin(), g.members.end());
        g.is_static = false;
        g.last_change_step = step;
        seg_.emplace(s.id, std::move(s));
        cur_step_ = std::max(cur_step_, step);
        reindex();
    }

    // memory_store.hpp:456-468
    bool state_sound() const {
        if (cfg_.fixed) return true;
        for (const auto& g : groups_) {
            int64_t newest = 0;
            for (uint32_t m : g.members) newest = std::max(newest, seg_.at(m).last_update_step);
            if (g.is_static != (newest <= last_adv_ - cfg_.t)) return false;
        }
        return true;
    }

private:
    // cluster_segments (memory_store.hpp:240-272): canonical ids by smallest member
    void cluster() {
        if (seg_.empty()) fail(KEEP_ERR_CONFIG, "no segments to cluster");
        if (cfg_.num_groups > int(seg_.size())) fail(KEEP_ERR_CONFIG, "num_groups exceeds segment count");
        std::vector<std::vector<uint32_t>> mem(static_cast<size_t>(cfg_.num_groups));
        std::vector<const Segment*> by_id;
        for (const auto& [id, s] : seg_) by_id.push_back(&s);
        if (cfg_.fixed) {
            const size_t block = (by_id.size() + cfg_.num_groups - 1) / cfg_.num_groups;
            for (size_t i = 0; i < by_id.size(); ++i) mem[std::min(i / block, mem.size() - 1)].push_back(by_id[i]->id);
        } else {
            std::vector<std::vector<double>> pts;
            for (const auto* s : by_id) pts.push_back(s->emb);
            const auto as = kmeans(pts, cfg_.num_groups, cfg_.seed);
            for (size_t i = 0; i < by_id.size(); ++i) mem[as[i]].push_back(by_id[i]->id);
        }
        mem.erase(std::remove_if(mem.begin(), mem.end(), [](const auto& m) { return m.empty(); }), mem.end());
        std::sort(mem.begin(), mem.end(), [](const auto& a, const auto& b) { return a.front() < b.front(); });
        for (size_t g = 0; g < mem.size(); ++g) groups_.push_back(Group{uint32_t(g), std::move(mem[g]), false, 0});
    }
    void check_embedding(const std::vector<double>& e) const {
        if (e.empty()) fail(KEEP_ERR_CONFIG, "segment embedding is empty");
        if (std::abs(std::sqrt(dot(e, e)) - 1.0) > 1e-6) fail(KEEP_ERR_CONFIG, "segment embedding is not unit norm");
    }
    size_t gidx(uint32_t id) const {
        auto it = idx_.find(id);
        if (it == idx_.end()) fail(KEEP_ERR_INPUT, "unknown segment " + std::to_string(id));
        return it->second;
    }
    void reindex() {
        idx_.clear();
        for (size_t g = 0; g < groups_.size(); ++g)
            for (uint32_t m : groups_[g].members) idx_[m] = g;
    }

    StoreCfg cfg_;
    std::map<uint32_t, Segment> seg_;
    std::vector<Group> groups_;
    std::vector<uint64_t> gver_;
    std::map<uint32_t, size_t> idx_;
    int64_t cur_step_ = 0, last_adv_ = 0;
};

// ------------------------------------------------------------- TierBook --
// CacheManager's bookkeeping (cache_manager.hpp:60-228) for the device
// memory tier's blocks: which (owner, layer) blocks are current, which tier
// the cost model places them in, LRU order and the slow-load statistics.
struct TierCfg {
    uint64_t cap = 0, fast_bw = 0, slow_bw = 0;
    void validate() const {
        if (cap == 0 || fast_bw == 0 || slow_bw == 0) fail(KEEP_ERR_CONFIG, "tier parameters must be positive");
        if (slow_bw > fast_bw) fail(KEEP_ERR_CONFIG, "slow bandwidth must not exceed fast bandwidth");
    }
};
struct Stats {
    double reused = 0.0, recomputed = 0.0;
    uint64_t invalidated = 0, bytes_slow = 0, misses = 0;
};

class TierBook {
public:
    explicit TierBook(const TierCfg& c) : cfg_(c) { cfg_.validate(); }

    void put(const Owner& o, uint64_t version, int layer, uint64_t tokens, uint64_t bytes) {
        auto& cur = cur_[o];
        cur = std::max(cur, version);
        const Key key{o, layer};
        auto it = blocks_.find(key);
        if (it != blocks_.end()) {
            if (it->second.fast) used_ -= it->second.size;
            blocks_.erase(it);
        }
        Block b{version, tokens, bytes, false, ++touch_};
        if (bytes <= cfg_.cap) {
            make_room(bytes);
            b.fast = true;
            used_ += bytes;
        }
        blocks_.emplace(key, b);
    }
    // load (cache_manager.hpp:103-130): misses raise; slow hits promote
    double load(const Owner& o, int layer) {
        auto it = blocks_.find(Key{o, layer});
        if (it == blocks_.end() || !current(o, it->second)) {
            ++st_.misses;
            fail(KEEP_ERR_CACHE_MISS, (it == blocks_.end() ? "no block for " : "stale block for ") + o.str() +
                                          " layer " + std::to_string(layer));
        }
        Block& b = it->second;
        double cost = 0.0;
        if (!b.fast) {
            cost = double(b.size) / double(cfg_.slow_bw);
            st_.bytes_slow += b.size;
            if (b.size <= cfg_.cap) {
                make_room(b.size);
                b.fast = true;
                used_ += b.size;
            }
        }
        b.touch = ++touch_;
        return cost;
    }
    // peek_tier / peek_payload: 0 none, 1 fast, 2 slow
    int peek(const Owner& o, int layer) const {
        auto it = blocks_.find(Key{o, layer});
        if (it == blocks_.end() || !current(o, it->second)) return 0;
        return it->second.fast ? 1 : 2;
    }
    uint64_t bytes(const Owner& o, int layer) const { return blocks_.at(Key{o, layer}).size; }
    bool has_current(const Owner& o, uint64_t version, int L) const {
        auto cv = cur_.find(o);
        if (cv != cur_.end() && cv->second > version) return false;
        for (int l = 0; l < L; ++l) {
            auto it = blocks_.find(Key{o, l});
            if (it == blocks_.end() || it->second.version != version) return false;
        }
        return true;
    }
    void invalidate(const Invalidation& rec) {
        uint64_t dropped_tokens = 0;
        for (const auto& [o, toks] : rec.entries) {
            bool dropped = false;
            for (auto it = blocks_.begin(); it != blocks_.end();) {
                if (it->first.o == o) {
                    if (it->second.fast) used_ -= it->second.size;
                    it = blocks_.erase(it);
                    dropped = true;
                } else {
                    ++it;
                }
            }
            if (dropped) dropped_tokens += toks;
        }
        for (const auto& [s, v] : rec.new_versions) {
            auto& cur = cur_[Owner{KEEP_OWNER_SEGMENT, s}];
            cur = std::max(cur, v);
        }
        st_.invalidated += dropped_tokens;
    }
    void account(double reused, double recomputed) {
        st_.reused += reused;
        st_.recomputed += recomputed;
    }
    const Stats& stats() const { return st_; }

private:
    struct Key {
        Owner o;
        int layer;
        bool operator<(const Key& k) const { return !(o == k.o) ? o < k.o : layer < k.layer; }
    };
    struct Block {
        uint64_t version, tokens, size;
        bool fast;
        uint64_t touch;
    };
    bool current(const Owner& o, const Block& b) const {
        auto cv = cur_.find(o);
        return cv != cur_.end() && b.version == cv->second;
    }
    void make_room(uint64_t need) {  // LRU demotion to the slow tier
        while (used_ + need > cfg_.cap) {
            Block* lru = nullptr;
            for (auto& [k, b] : blocks_)
                if (b.fast && (lru == nullptr || b.touch < lru->touch)) lru = &b;
            if (lru == nullptr) break;
            lru->fast = false;
            used_ -= lru->size;
        }
    }
    TierCfg cfg_;
    std::map<Key, Block> blocks_;
    std::map<Owner, uint64_t> cur_;
    Stats st_;
    uint64_t used_ = 0, touch_ = 0;
};

// ----------------------------------------------------- pipeline model --
// derive_workload / simulate_{sequential,overlap,balanced} / validate_timeline
// (pipeline_sim.hpp:103-428).  Plans are per-layer masks over layout positions.
struct Cost {
    double compute = 1.0, eval = 0.0, attn_frac = 0.5;
    void validate() const {
        if (compute <= 0.0) fail(KEEP_ERR_CONFIG, "compute_tu_per_token_per_layer must be positive");
        if (eval < 0.0) fail(KEEP_ERR_CONFIG, "eval_tu_per_layer must be >= 0");
        if (attn_frac < 0.0 || attn_frac > 1.0) fail(KEEP_ERR_CONFIG, "attention_fraction must be in [0, 1]");
    }
};
using Plan = std::vector<std::vector<uint8_t>>;  // [L][S]

struct Item {
    int layer;
    Owner owner;
    uint64_t bytes;
    double tu;
};
struct Workload {
    int L = 0;
    std::vector<double> compute, eval;
    double attn_frac = 0.5;
    std::vector<Item> items;
    std::map<Owner, std::vector<int>> members;  // owner -> member positions (every unit of the layout)
};
enum Kind { LOAD, COMPUTE, EVAL };
struct Ev {
    Kind kind;
    int layer;
    Owner owner;
    uint64_t bytes;
    double start, end;
};
struct Timeline {
    std::vector<Ev> ev;
    double makespan = 0.0;
};
struct LoadUnit {
    Owner owner;
    std::vector<int> pos;           // member positions
    std::vector<uint64_t> slow;     // per layer
};

bool needed_at(const Plan& plan, int l, const std::vector<int>& pos) {
    for (int p : pos)
        if (!plan[l][p]) return true;
    return false;
}

Workload derive_workload(const Plan& plan, const std::vector<int64_t>& seg_tokens, const std::vector<LoadUnit>& units,
                         size_t qtok, const Cost& cost, double slow_bw, bool with_eval) {
    cost.validate();
    if (slow_bw <= 0.0) fail(KEEP_ERR_CONFIG, "slow bandwidth must be positive");
    const int L = int(plan.size());
    Workload w;
    w.L = L;
    w.attn_frac = cost.attn_frac;
    w.compute.assign(L, 0.0);
    w.eval.assign(L, 0.0);
    for (int l = 0; l < L; ++l) {
        size_t tok = qtok;
        for (size_t p = 0; p < plan[l].size(); ++p)
            if (plan[l][p]) tok += static_cast<size_t>(seg_tokens[p]);
        w.compute[l] = double(tok) * cost.compute;
        if (with_eval && l + 1 < L) w.eval[l] = cost.eval;
    }
    for (const auto& u : units) {
        if (u.owner.kind == KEEP_OWNER_GROUP) w.members[u.owner] = u.pos;
        for (int l = 0; l < L; ++l) {
            if (!needed_at(plan, l, u.pos)) continue;
            const uint64_t b = l < int(u.slow.size()) ? u.slow[l] : 0;
            if (b == 0) continue;
            w.items.push_back(Item{l, u.owner, b, double(b) / slow_bw});
        }
    }
    std::sort(w.items.begin(), w.items.end(), [](const Item& a, const Item& b) {
        return a.layer != b.layer ? a.layer < b.layer : a.owner < b.owner;
    });
    return w;
}

// members of an owner as layout positions; a segment owner is its own position
std::vector<int> members_of(const Workload& w, const Owner& o, const std::map<uint32_t, int>& pos_of) {
    if (o.kind == KEEP_OWNER_SEGMENT) {
        auto it = pos_of.find(o.id);
        return it == pos_of.end() ? std::vector<int>{} : std::vector<int>{it->second};
    }
    auto it = w.members.find(o);
    return it == w.members.end() ? std::vector<int>{} : it->second;
}

void emit(Timeline& tl, Kind k, int layer, double s, double e, const Owner& o = {}, uint64_t bytes = 0) {
    if (e <= s) return;
    tl.ev.push_back(Ev{k, layer, o, bytes, s, e});
    tl.makespan = std::max(tl.makespan, e);
}

int preload_from(const Workload& w, const Plan& plan, const Owner& o, const std::map<uint32_t, int>& pos_of) {
    const int L = int(plan.size());
    const auto mem = members_of(w, o, pos_of);
    if (mem.empty()) return std::numeric_limits<int>::max();
    int from = 0;
    for (int m : mem) {
        int first = std::numeric_limits<int>::max();
        for (int l = 0; l < L; ++l)
            if (!plan[l][m]) {
                first = l;
                break;
            }
        from = std::max(from, first);
        if (from == std::numeric_limits<int>::max()) break;
    }
    return from;
}

Timeline sim_sequential(const Workload& w) {
    Timeline tl;
    double t = 0.0;
    for (int l = 0; l < w.L; ++l) {
        for (const auto& it : w.items) {
            if (it.layer != l) continue;
            emit(tl, LOAD, l, t, t + it.tu, it.owner, it.bytes);
            t += it.tu;
        }
        if (l >= 1 && w.eval[l - 1] > 0.0) {
            emit(tl, EVAL, l - 1, t, t + w.eval[l - 1]);
            t += w.eval[l - 1];
        }
        emit(tl, COMPUTE, l, t, t + w.compute[l]);
        t += w.compute[l];
    }
    tl.makespan = std::max(tl.makespan, t);
    return tl;
}

// overlap (balanced = false) and balanced (pipeline_sim.hpp:214-338)
Timeline sim_overlap(const Workload& w, const Plan* plan, const std::map<uint32_t, int>& pos_of) {
    Timeline tl;
    const int L = w.L;
    struct Pend {
        Item item;
        int from;
        bool loaded;
    };
    std::vector<Pend> pend;
    for (const auto& it : w.items)
        pend.push_back({it, plan ? preload_from(w, *plan, it.owner, pos_of) : std::numeric_limits<int>::max(), false});
    std::vector<double> last_end(static_cast<size_t>(L), 0.0);
    double load_free = 0.0, eval_free = 0.0, prev_c = 0.0, prev_e = 0.0;
    for (auto& p : pend) {
        if (p.item.layer != 0) continue;
        emit(tl, LOAD, 0, load_free, load_free + p.item.tu, p.item.owner, p.item.bytes);
        load_free += p.item.tu;
        last_end[0] = load_free;
        p.loaded = true;
    }
    for (int l = 0; l < L; ++l) {
        const double cs = std::max({prev_c, prev_e, last_end[l]});
        const double ce = cs + w.compute[l];
        emit(tl, COMPUTE, l, cs, ce);
        prev_e = 0.0;
        if (w.eval[l] > 0.0) {
            const double attn_done = cs + w.attn_frac * w.compute[l];
            const double es = std::max(attn_done, eval_free);
            const double ee = es + w.eval[l];
            emit(tl, EVAL, l, es, ee);
            eval_free = ee;
            prev_e = ee;
        }
        if (l + 1 < L) {
            for (auto& p : pend) {
                if (p.loaded || p.item.layer != l + 1) continue;
                const double s = std::max(load_free, cs);
                emit(tl, LOAD, l + 1, s, s + p.item.tu, p.item.owner, p.item.bytes);
                load_free = s + p.item.tu;
                last_end[l + 1] = load_free;
                p.loaded = true;
            }
        }
        if (plan) {  // idle-window fill with eligible future items, ascending (layer, owner)
            while (true) {
                Pend* nx = nullptr;
                for (auto& p : pend) {
                    if (p.loaded || p.item.layer < l + 2 || p.from > l) continue;
                    nx = &p;
                    break;
                }
                if (!nx) break;
                const double s = std::max(load_free, cs);
                const double e = s + nx->item.tu;
                if (e > ce + 1e-12) break;
                emit(tl, LOAD, nx->item.layer, s, e, nx->item.owner, nx->item.bytes);
                load_free = e;
                nx->loaded = true;
            }
        }
        prev_c = ce;
    }
    tl.makespan = std::max(tl.makespan, prev_c);
    return tl;
}

// validate_timeline (pipeline_sim.hpp:340-428): first violation, or empty
std::string validate(const Timeline& tl, const Plan& plan, const Workload& w, const std::map<uint32_t, int>& pos_of) {
    constexpr double eps = 1e-9;
    for (Kind res : {LOAD, COMPUTE, EVAL}) {  // R
        std::vector<const Ev*> e;
        for (const auto& x : tl.ev)
            if (x.kind == res) e.push_back(&x);
        std::sort(e.begin(), e.end(), [](const Ev* a, const Ev* b) { return a->start < b->start; });
        for (size_t i = 0; i + 1 < e.size(); ++i)
            if (e[i + 1]->start < e[i]->end - eps) return "R overlapping events on one resource";
    }
    std::map<int, const Ev*> comp;
    for (const auto& x : tl.ev)
        if (x.kind == COMPUTE) comp[x.layer] = &x;
    for (const auto& [l, c] : comp)  // D1
        for (const auto& x : tl.ev) {
            if (x.kind == LOAD && x.layer == l && x.end > c->start + eps) return "D1 load ends after compute starts";
            if (x.kind == EVAL && x.layer == l - 1 && x.end > c->start + eps) return "D1 eval ends after compute";
        }
    for (const auto& x : tl.ev) {  // D2
        if (x.kind != EVAL) continue;
        auto it = comp.find(x.layer);
        if (it == comp.end()) continue;
        if (x.start < it->second->start + w.attn_frac * (it->second->end - it->second->start) - eps)
            return "D2 eval starts before attention completes";
    }
    {  // P
        std::map<std::pair<int, std::string>, uint64_t> got, want;
        for (const auto& x : tl.ev)
            if (x.kind == LOAD && x.bytes > 0) got[{x.layer, x.owner.str()}] += x.bytes;
        for (const auto& it : w.items)
            if (it.bytes > 0) want[{it.layer, it.owner.str()}] += it.bytes;
        if (got != want) return "P loaded bytes do not match workload items";
    }
    for (const auto& x : tl.ev) {  // S
        if (x.kind != LOAD) continue;
        for (const auto& [l, c] : comp) {
            if (x.start >= c->end - eps || x.end <= c->start + eps) continue;
            if (x.layer < l + 2) continue;
            for (int m : members_of(w, x.owner, pos_of))
                if (l < int(plan.size()) && plan[l][m]) return "S pre-load of an owner still planned";
        }
    }
    double mx = 0.0;
    for (const auto& x : tl.ev) mx = std::max(mx, x.end);
    if (tl.makespan + eps < mx) return "P makespan smaller than the last event end";
    return {};
}

// ----------------------------------------------------------- episode --
struct Category {
    std::string name;
    int count = 0, tokens = 8;
    double p = 0.0;
};
struct EpCfg {
    uint64_t seed = 0;
    int num_segments = 0, num_steps = 1, k = 1;
    double r_avg = 0.5;
    int qtok = 8, edim = 16, edge = 4;
    StoreCfg store;
    int L = 0, H = 0, d = 0, mlp = 0, V = 0;
    Cost cost;
    TierCfg tier;
    std::vector<Category> cats;
    bool multihop = true, balanced = true;
    int sched_override = KEEP_SCHEDULE_DEFAULT;

    static EpCfg from(const keep_episode_config* c) {
        if (!c) fail(KEEP_ERR_CONFIG, "null episode config");
        EpCfg e;
        e.seed = c->seed;
        e.num_segments = c->num_segments;
        e.num_steps = c->num_steps;
        e.k = c->retrieval_k;
        e.r_avg = c->r_avg;
        e.qtok = c->query_tokens;
        e.edim = c->embedding_dim;
        e.edge = c->fixed_pos_edge_tokens;
        e.store.t = c->store_t;
        e.store.num_groups = c->store_num_groups;
        e.store.seed = c->store_seed ? c->store_seed : c->seed;  // EpisodeRuntime::store_config
        e.store.fixed = c->grouping == KEEP_GROUPING_FIXED;
        e.L = c->num_layers;
        e.H = c->num_heads;
        e.d = c->model_dim;
        e.mlp = c->mlp_dim;
        e.V = c->vocab_size;
        e.cost = Cost{c->compute_tu_per_token_per_layer, c->eval_tu_per_layer, c->attention_fraction};
        e.tier = TierCfg{c->fast_capacity_bytes, c->fast_bandwidth_bytes_per_tu, c->slow_to_fast_bandwidth_bytes_per_tu};
        for (int i = 0; i < c->n_categories; ++i) {
            const keep_category& k = c->categories[i];
            e.cats.push_back(Category{k.name ? k.name : "", k.count, k.tokens_per_segment, k.update_prob_per_step});
        }
        e.multihop = c->multihop != 0;
        e.balanced = c->balanced_loading != 0;
        e.sched_override = c->schedule_override;
        return e;
    }
    // EpisodeConfig::validate (harness.hpp:68-104)
    void validate() const {
        if (num_steps < 1) fail(KEEP_ERR_CONFIG, "num_steps must be >= 1");
        if (k < 1) fail(KEEP_ERR_CONFIG, "retrieval_k must be >= 1");
        if (qtok < 1) fail(KEEP_ERR_CONFIG, "query_tokens must be >= 1");
        if (edim < 1) fail(KEEP_ERR_CONFIG, "embedding_dim must be >= 1");
        if (edge < 0) fail(KEEP_ERR_CONFIG, "fixed_pos_edge_tokens must be >= 0");
        if (L < 1 || H < 1 || d < 1 || mlp < 1 || V < 1) fail(KEEP_ERR_CONFIG, "model dimensions must be positive");
        if (d % H) fail(KEEP_ERR_CONFIG, "model_dim not divisible by num_heads");
        store.validate();
        cost.validate();
        tier.validate();
        int total = 0;
        for (const auto& c : cats) {
            if (c.count < 0) fail(KEEP_ERR_CONFIG, "category count must be >= 0");
            if (c.tokens < 1) fail(KEEP_ERR_CONFIG, "tokens_per_segment must be >= 1");
            if (c.p < 0.0 || c.p > 1.0) fail(KEEP_ERR_CONFIG, "update probability must be in [0, 1]");
            total += c.count;
        }
        if (total != num_segments) fail(KEEP_ERR_CONFIG, "category counts must sum to num_segments");
        if (L > 1) {
            const double lo = 1.0 / L;
            if (r_avg < lo - 1e-9 || r_avg > 1.0 + 1e-9) fail(KEEP_ERR_CONFIG, "r_avg outside [1/L, 1]");
        }
    }
};

struct Event {
    int type = KEEP_EVENT_INIT_SEGMENT;
    int64_t step = 0;
    uint32_t id = 0;
    std::string category;
    Tokens tokens;
    std::vector<double> emb;
    uint64_t eseed = 0;
    int k = 0;
};
struct Trace {
    std::vector<Event> ev;
};

// generate_episode (harness.hpp:362-413)
Trace generate(const EpCfg& c) {
    c.validate();
    Trace tr;
    Rng seg_rng = Rng::stream(c.seed, "segments");
    uint32_t next = 0;
    std::vector<double> prob;
    std::vector<int> ntok;
    for (const auto& cat : c.cats) {
        Rng cr = Rng::stream(c.seed, "centroid." + cat.name);
        const auto centroid = cr.unit_vector(static_cast<size_t>(c.edim));
        for (int i = 0; i < cat.count; ++i) {
            Event e;
            e.type = KEEP_EVENT_INIT_SEGMENT;
            e.id = next++;
            e.category = cat.name;
            e.tokens = random_tokens(seg_rng, cat.tokens, c.V);
            std::vector<double> emb = centroid;
            for (auto& x : emb) x += 0.35 * seg_rng.gaussian();
            double n = 0.0;
            for (double x : emb) n += x * x;
            n = std::sqrt(std::max(n, 1e-12));
            for (auto& x : emb) x /= n;
            e.emb = std::move(emb);
            prob.push_back(cat.p);
            ntok.push_back(cat.tokens);
            tr.ev.push_back(std::move(e));
        }
    }
    Rng upd = Rng::stream(c.seed, "updates");
    Rng qry = Rng::stream(c.seed, "queries");
    for (int step = 1; step <= c.num_steps; ++step) {
        for (uint32_t id = 0; id < next; ++id) {
            if (upd.uniform() < prob[id]) {
                Event e;
                e.type = KEEP_EVENT_UPDATE;
                e.step = step;
                e.id = id;
                e.tokens = random_tokens(upd, ntok[id], c.V);
                tr.ev.push_back(std::move(e));
            }
        }
        Event q;
        q.type = KEEP_EVENT_QUERY;
        q.step = step;
        q.eseed = qry.u64();
        q.k = c.k;
        tr.ev.push_back(std::move(q));
    }
    return tr;
}

// derive_query (harness.hpp:341-360)
void derive_query(uint64_t eseed, const std::vector<std::vector<double>>& embs, int qtok, int V,
                  std::vector<double>& emb, Tokens& toks) {
    Rng r(eseed);
    const size_t focus = r.below(embs.size());
    emb = embs[focus];
    for (auto& x : emb) x += 0.25 * r.gaussian();
    double n = 0.0;
    for (double x : emb) n += x * x;
    n = std::sqrt(std::max(n, 1e-12));
    for (auto& x : emb) x /= n;
    toks = random_tokens(r, qtok, V);
}

enum Strategy { FULL, PREFIX, FULL_REUSE, FIXED_POS, DEVIATION, KEEP };
Strategy parse_strategy(const std::string& s) {
    static const char* names[] = {"full", "prefix", "full-reuse", "fixed-pos", "deviation", "keep"};
    for (int i = 0; i < 6; ++i)
        if (s == names[i]) return Strategy(i);
    fail(KEEP_ERR_CONFIG, "unknown strategy '" + s + "'");
}
const char* strategy_name(Strategy s) {
    static const char* names[] = {"full", "prefix", "full-reuse", "fixed-pos", "deviation", "keep"};
    return names[s];
}

struct StepRow {
    int64_t step = 0, realized = 0;
    double ttft = 0, makespan = 0, refresh = 0, l2 = 0, kl = 0, reused = 0, recomputed = 0, memory = 0;
    uint64_t inval_delta = 0, slow_delta = 0;
    std::vector<int64_t> plan_sizes;
    double wall_ms = 0;
};
struct Report {
    std::string strategy;
    std::vector<StepRow> steps;
    double mean_ttft = 0, p95_ttft = 0, mean_l2 = 0, mean_kl = 0, reuse_ratio = 0, mean_realized = 0;
    uint64_t invalidated = 0, bytes_slow = 0;
};

// The device side of one query: a layout in retrieval order, its GPU prefills.
struct DeviceLayout {
    std::vector<int32_t> seg_len, tokens, ub, ue;
    std::vector<keep_owner> uo;
    keep_layout c() const {
        return keep_layout{int32_t(seg_len.size()), int32_t(ub.size()), seg_len.data(), tokens.data(), ub.data(),
                           ue.data(), uo.data()};
    }
};

class Runtime {
public:
    Runtime(void* ctx, const EpCfg& cfg, std::vector<Segment> segs)
        : ctx_(ctx), cfg_(cfg), store_(std::move(segs), cfg.store), book_(cfg.tier) {
        sched_.resize(static_cast<size_t>(cfg.L));
        ck(keep_ratio_schedule(cfg.L, cfg.r_avg, sched_.data()));
        ck(keep_memory_clear(ctx));
    }

    Store& store() { return store_; }
    TierBook& book() { return book_; }
    const std::vector<double>& schedule() const { return sched_; }

    // compute_and_put (harness.hpp:512-532) for a list of units: one batched
    // canonical refresh on the GPU, then the per-layer puts in the reference's
    // order (the LRU order of the tier accounting depends on it)
    void compute_and_put(const std::vector<Unit>& units) {
        if (units.empty()) return;
        std::vector<keep_owner> owners;
        std::vector<uint64_t> versions;
        std::vector<int32_t> nmem, mlen, toks;
        for (const auto& u : units) {
            owners.push_back(u.owner.c());
            versions.push_back(store_.version(u.owner));
            nmem.push_back(int32_t(u.segments.size()));
            for (uint32_t s : u.segments) {
                const auto& t = store_.segment(s).tokens;
                mlen.push_back(int32_t(t.size()));
                toks.insert(toks.end(), t.begin(), t.end());
            }
        }
        ck(keep_memory_compute_batch(ctx_, int32_t(owners.size()), owners.data(), versions.data(), nmem.data(),
                                     mlen.data(), toks.data(), KEEP_TIER_DEVICE));
        for (size_t i = 0; i < units.size(); ++i) {
            const uint64_t n = unit_tokens(units[i]);
            for (int l = 0; l < cfg_.L; ++l)
                book_.put(units[i].owner, versions[i], l, n, n * uint64_t(cfg_.d) * 2 * 4);  // kv_block_bytes
        }
    }
    uint64_t unit_tokens(const Unit& u) const {
        uint64_t n = 0;
        for (uint32_t s : u.segments) n += store_.segment(s).tokens.size();
        return n;
    }
    // CacheManager::invalidate on the books, keep_invalidate on the device tier
    void invalidate(const Invalidation& rec) {
        book_.invalidate(rec);
        for (const auto& [o, toks] : rec.entries) ck(keep_invalidate(ctx_, o.c(), 0, toks));
        for (const auto& [s, v] : rec.new_versions) ck(keep_invalidate(ctx_, keep_owner{KEEP_OWNER_SEGMENT, s}, v, 0));
    }

    void* ctx() const { return ctx_; }

private:
    void* ctx_;
    const EpCfg& cfg_;
    Store store_;
    TierBook book_;
    std::vector<double> sched_;
};

// plan_prefix / plan_full_reuse / plan_fixed_position (recompute.hpp:182-257)
Plan plan_fixed_position(const std::vector<int64_t>& seg_len, const std::vector<std::pair<int, int>>& units,
                         const std::vector<uint32_t>& ids, const std::vector<double>& r, int edge) {
    const int S = int(seg_len.size()), L = int(r.size());
    std::vector<int64_t> st(static_cast<size_t>(S)), en(static_cast<size_t>(S));
    int64_t pos = 0;
    for (int i = 0; i < S; ++i) {
        st[i] = pos;
        pos += seg_len[i];
        en[i] = pos;
    }
    struct Ranked {
        int64_t dist;
        uint32_t id;
        int pos;
    };
    std::vector<Ranked> el;
    for (const auto& [b, e] : units) {
        const int64_t us = st[b], ustop = en[e - 1];
        for (int i = b; i < e; ++i) {
            const bool head = st[i] < us + edge, tail = en[i] > ustop - edge;
            if (!head && !tail) continue;
            el.push_back({std::min(st[i] - us, ustop - en[i]), ids[i], i});
        }
    }
    std::sort(el.begin(), el.end(),
              [](const Ranked& a, const Ranked& b) { return a.dist != b.dist ? a.dist < b.dist : a.id < b.id; });
    Plan plan(static_cast<size_t>(L), std::vector<uint8_t>(static_cast<size_t>(S), 0));
    for (int l = 0; l < L; ++l) {
        const size_t budget = std::min<size_t>(static_cast<size_t>(keep_layer_budget(r[l], S)), el.size());
        for (size_t i = 0; i < budget; ++i) plan[l][el[i].pos] = 1;
    }
    return plan;
}

bool monotone(const Plan& p) {
    for (size_t l = 0; l + 1 < p.size(); ++l)
        for (size_t i = 0; i < p[l].size(); ++i)
            if (p[l + 1][i] && !p[l][i]) return false;
    return true;
}

// one selective prefill through the cursor (selective_prefill,
// prefill.hpp:478-497); the final hidden state [T x d] and optionally kv
void cursor_prefill(void* ctx, const DeviceLayout& dl, const Tokens& q, const Plan& plan, std::vector<float>& fh,
                    std::vector<float>* kv, int d) {
    const keep_layout lay = dl.c();
    ck(keep_prefill_begin(ctx, &lay, q.data(), int32_t(q.size())));
    for (const auto& act : plan) ck(keep_prefill_layer(ctx, act.data(), nullptr));
    const size_t T = dl.tokens.size() + q.size();
    fh.assign(T * static_cast<size_t>(d), 0.f);
    ck(keep_prefill_finish(ctx, fh.data(), kv ? kv->data() : nullptr));
}

Report run_episode(void* ctx, const Trace& trace, const std::string& sname, const EpCfg& cfg) {
    cfg.validate();
    const Strategy strategy = parse_strategy(sname);
    int32_t dims[7];
    ck(keep_ctx_dims(ctx, dims));
    if (dims[0] != cfg.L || dims[1] != cfg.H || dims[2] != cfg.d || dims[3] != cfg.mlp || dims[4] != cfg.V)
        fail(KEEP_ERR_CONFIG, "episode model config does not match the context");
    if (dims[6] != 1) fail(KEEP_ERR_CONFIG, "run_episode drives one context (world_size 1)");
    const int L = cfg.L, d = cfg.d;

    std::vector<Segment> segs;
    std::map<int64_t, std::vector<const Event*>> steps;
    for (const auto& e : trace.ev) {
        if (e.type == KEEP_EVENT_INIT_SEGMENT) {
            Segment s;
            s.id = e.id;
            s.category = e.category;
            s.tokens = e.tokens;
            s.emb = e.emb;
            segs.push_back(std::move(s));
        } else {
            steps[e.step].push_back(&e);
        }
    }
    if (segs.empty()) fail(KEEP_ERR_TRACE, "trace has no init-segment events");
    std::vector<std::vector<double>> embs;
    {
        auto sorted = segs;
        std::sort(sorted.begin(), sorted.end(), [](const Segment& a, const Segment& b) { return a.id < b.id; });
        for (const auto& s : sorted) embs.push_back(s.emb);
    }
    Runtime rt(ctx, cfg, std::move(segs));
    Report rep;
    rep.strategy = strategy_name(strategy);
    Stats prev;
    double total_reused = 0.0, total_memory = 0.0;

    for (const auto& [step, events] : steps) {
        for (const auto* e : events) {
            if (e->type != KEEP_EVENT_UPDATE) continue;
            rt.invalidate(rt.store().apply_update(e->id, e->tokens, step));
        }
        {
            std::vector<Unit> bg;  // background joint recompute of newly static groups
            for (const auto& t : rt.store().advance_step(step)) bg.push_back(Unit{Owner{KEEP_OWNER_GROUP, t.group}, t.members});
            rt.compute_and_put(bg);
        }
        for (const auto* e : events) {
            if (e->type != KEEP_EVENT_QUERY) continue;
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<double> qemb;
            Tokens q;
            derive_query(e->eseed, embs, cfg.qtok, cfg.V, qemb, q);
            const std::vector<Unit> units = rt.store().retrieve(qemb, e->k);

            DeviceLayout dl;
            std::vector<uint32_t> ids;
            std::vector<int64_t> seg_len;
            std::vector<std::pair<int, int>> upos;
            std::map<uint32_t, int> pos_of;
            for (const auto& u : units) {
                const int b = int(ids.size());
                for (uint32_t s : u.segments) {
                    const auto& t = rt.store().segment(s).tokens;
                    pos_of[s] = int(ids.size());
                    ids.push_back(s);
                    seg_len.push_back(int64_t(t.size()));
                    dl.seg_len.push_back(int32_t(t.size()));
                    dl.tokens.insert(dl.tokens.end(), t.begin(), t.end());
                }
                upos.emplace_back(b, int(ids.size()));
                dl.ub.push_back(b);
                dl.ue.push_back(int32_t(ids.size()));
                dl.uo.push_back(u.owner.c());
            }
            const int S = int(ids.size());

            // refresh missing canonical KV (full never reads the cache, prefix
            // recomputes from the first miss)
            double refresh_tu = 0.0;
            std::optional<int> first_invalid;
            {
                std::vector<Unit> todo;
                int pos = 0;
                for (const auto& u : units) {
                    if (!rt.book().has_current(u.owner, rt.store().version(u.owner), L)) {
                        if (!first_invalid) first_invalid = pos;
                        if (strategy != FULL && strategy != PREFIX) {
                            todo.push_back(u);
                            refresh_tu += double(rt.unit_tokens(u)) * L * cfg.cost.compute;
                        }
                    }
                    pos += int(u.segments.size());
                }
                rt.compute_and_put(todo);
            }

            Plan plan(static_cast<size_t>(L), std::vector<uint8_t>(static_cast<size_t>(S), 0));
            std::vector<float> fh_sel, fh_full, kv_full;
            const bool need_kv = strategy == DEVIATION;
            const Plan ones(static_cast<size_t>(L), std::vector<uint8_t>(static_cast<size_t>(S), 1));
            switch (strategy) {
                case FULL:
                    plan = ones;
                    break;
                case PREFIX:
                    if (first_invalid)
                        for (int l = 0; l < L; ++l)
                            for (int i = *first_invalid; i < S; ++i) plan[l][i] = 1;
                    break;
                case FULL_REUSE:
                    break;
                case FIXED_POS:
                    plan = plan_fixed_position(seg_len, upos, ids, rt.schedule(), cfg.edge);
                    break;
                case DEVIATION:
                case KEEP:
                    break;
            }
            // the oracle pass of run_strategy: a full prefill (plan of ones)
            if (need_kv) kv_full.assign(static_cast<size_t>(L) * 2 * (dl.tokens.size() + q.size()) * d, 0.f);
            cursor_prefill(ctx, dl, q, ones, fh_full, need_kv ? &kv_full : nullptr, d);
            if (strategy == DEVIATION) {
                // plan_deviation (recompute.hpp:262-312): fresh layer-0 K/V (the full
                // prefill's, embedding . W{k,v}) against the cached layer-0 KV
                const size_t T = dl.tokens.size() + q.size();
                std::vector<double> dev(static_cast<size_t>(S), 0.0);
                size_t row = 0;
                for (size_t ui = 0; ui < units.size(); ++ui) {
                    const uint64_t n = rt.unit_tokens(units[ui]);
                    if (rt.book().peek(units[ui].owner, 0) == 0)
                        fail(KEEP_ERR_CACHE_MISS,
                             "plan_deviation: no cached KV for segment " + std::to_string(units[ui].segments[0]));
                    std::vector<float> ck_(n * static_cast<size_t>(d)), cv_(n * static_cast<size_t>(d));
                    ck(keep_memory_read(ctx, units[ui].owner.c(), 0, ck_.data(), cv_.data()));
                    size_t off = 0;
                    for (int p = upos[ui].first; p < upos[ui].second; ++p) {
                        double acc = 0.0;
                        for (int64_t t = 0; t < seg_len[p]; ++t, ++row, ++off) {
                            const float* fk = &kv_full[(0 * T + row) * d];
                            const float* fv = &kv_full[(1 * T + row) * d];
                            double sq = 0.0;
                            for (int j = 0; j < d; ++j) {
                                const double dk = double(fk[j]) - ck_[off * d + j];
                                const double dv = double(fv[j]) - cv_[off * d + j];
                                sq += dk * dk + dv * dv;
                            }
                            acc += std::sqrt(sq);
                        }
                        dev[p] = acc / double(seg_len[p]);
                    }
                }
                std::vector<int> rank(static_cast<size_t>(S));
                for (int i = 0; i < S; ++i) rank[i] = i;
                std::sort(rank.begin(), rank.end(), [&](int a, int b) {
                    return dev[a] != dev[b] ? dev[a] > dev[b] : ids[a] < ids[b];
                });
                for (int i = 0; i < S; ++i) plan[0][i] = 1;
                for (int l = 1; l < L; ++l) {
                    const size_t budget = static_cast<size_t>(keep_layer_budget(rt.schedule()[l], S));
                    for (size_t i = 0; i < budget && i < rank.size(); ++i) plan[l][rank[i]] = 1;
                }
            }
            if (strategy == KEEP) {
                // plan_keep on the GPU (recompute.hpp:140-180); its cursor run is
                // the selective prefill of the plan it chose
                const keep_layout lay = dl.c();
                std::vector<uint8_t> pm(static_cast<size_t>(L) * S);
                fh_sel.assign((dl.tokens.size() + q.size()) * static_cast<size_t>(d), 0.f);
                keep_plan_result res{};
                res.plan = pm.data();
                res.final_hidden = fh_sel.data();
                ck(keep_plan_keep(ctx, &lay, q.data(), int32_t(q.size()), rt.schedule().data(), cfg.multihop ? 1 : 0,
                                  &res));
                for (int l = 0; l < L; ++l)
                    std::copy(pm.begin() + static_cast<size_t>(l) * S, pm.begin() + static_cast<size_t>(l + 1) * S, plan[l].begin());
            }
            // run_strategy (recompute.hpp:314-335)
            if (!monotone(plan)) fail(KEEP_ERR_PLAN, "plan is not monotone across layers");
            if (strategy == FULL)
                fh_sel = fh_full;
            else if (strategy != KEEP)
                cursor_prefill(ctx, dl, q, plan, fh_sel, nullptr, d);
            const size_t T = dl.tokens.size() + q.size();
            double l2 = 0.0, kl = 0.0;
            ck(keep_divergence(ctx, &fh_sel[(T - 1) * d], &fh_full[(T - 1) * d], &l2, &kl));
            StepRow row;
            row.plan_sizes.resize(static_cast<size_t>(L));
            for (int l = 0; l < L; ++l) {
                int64_t n = 0;
                for (int i = 0; i < S; ++i) n += plan[l][i];
                row.plan_sizes[l] = n;
            }
            double reused = 0.0, recomputed = 0.0;
            for (int i = 0; i < S; ++i) {
                int rl = 0;
                for (int l = 0; l < L; ++l) rl += plan[l][i];
                const double tok = double(seg_len[i]);
                recomputed += tok * rl / L;
                reused += tok * (L - rl) / L;
            }
            recomputed += double(q.size());
            rt.book().account(reused, recomputed);

            // workload from the tier state before this query's loads, then the
            // loads replayed so LRU order and slow-byte stats evolve
            std::vector<LoadUnit> lus;
            for (size_t ui = 0; ui < units.size(); ++ui) {
                LoadUnit lu;
                lu.owner = units[ui].owner;
                for (int p = upos[ui].first; p < upos[ui].second; ++p) lu.pos.push_back(p);
                lu.slow.assign(static_cast<size_t>(L), 0);
                for (int l = 0; l < L; ++l)
                    if (rt.book().peek(lu.owner, l) == 2) lu.slow[l] = rt.book().bytes(lu.owner, l);
                lus.push_back(std::move(lu));
            }
            const bool with_eval = strategy == KEEP;
            const Workload w = derive_workload(plan, seg_len, lus, q.size(), cfg.cost, double(cfg.tier.slow_bw), with_eval);
            int kind;
            switch (strategy) {
                case FULL:
                case PREFIX:
                    kind = KEEP_SCHEDULE_SEQUENTIAL;
                    break;
                case KEEP:
                    kind = cfg.balanced ? KEEP_SCHEDULE_BALANCED : KEEP_SCHEDULE_OVERLAP;
                    break;
                default:
                    kind = KEEP_SCHEDULE_OVERLAP;
            }
            if (cfg.sched_override != KEEP_SCHEDULE_DEFAULT) kind = cfg.sched_override;
            const Timeline tl = kind == KEEP_SCHEDULE_SEQUENTIAL ? sim_sequential(w)
                                : kind == KEEP_SCHEDULE_OVERLAP  ? sim_overlap(w, nullptr, pos_of)
                                                                 : sim_overlap(w, &plan, pos_of);
            const std::string v = validate(tl, plan, w, pos_of);
            if (!v.empty()) fail(KEEP_ERR_PLAN, "schedule produced an invalid timeline: " + v);
            for (int l = 0; l < L; ++l)
                for (size_t ui = 0; ui < units.size(); ++ui) {
                    if (!needed_at(plan, l, lus[ui].pos)) continue;
                    if (rt.book().peek(units[ui].owner, l)) rt.book().load(units[ui].owner, l);
                }

            const Stats st = rt.book().stats();
            row.step = step;
            row.realized = S;
            row.refresh = refresh_tu;
            row.makespan = tl.makespan;
            row.ttft = refresh_tu + tl.makespan;
            row.l2 = l2;
            row.kl = kl;
            row.reused = reused;
            row.recomputed = recomputed;
            row.memory = double(dl.tokens.size());
            row.inval_delta = st.invalidated - prev.invalidated;
            row.slow_delta = st.bytes_slow - prev.bytes_slow;
            row.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            prev = st;
            total_reused += reused;
            total_memory += row.memory;
            rep.steps.push_back(std::move(row));
        }
    }
    if (!rep.steps.empty()) {
        std::vector<double> tt;
        for (const auto& s : rep.steps) {
            rep.mean_ttft += s.ttft;
            rep.mean_l2 += s.l2;
            rep.mean_kl += s.kl;
            rep.mean_realized += double(s.realized);
            tt.push_back(s.ttft);
        }
        const double n = double(rep.steps.size());
        rep.mean_ttft /= n;
        rep.mean_l2 /= n;
        rep.mean_kl /= n;
        rep.mean_realized /= n;
        std::sort(tt.begin(), tt.end());
        const size_t idx = static_cast<size_t>(std::ceil(0.95 * double(tt.size()))) - 1;
        rep.p95_ttft = tt[std::min(idx, tt.size() - 1)];
        rep.reuse_ratio = total_memory > 0 ? total_reused / total_memory : 0.0;
    }
    rep.invalidated = prev.invalidated;
    rep.bytes_slow = prev.bytes_slow;
    return rep;
}

std::string fmt_tu(double v) {  // serialize.hpp:20-24
    char b[64];
    std::snprintf(b, sizeof(b), "%.10g", v);
    return b;
}
std::string fmt_json(double v) {
    if (!std::isfinite(v)) return "null";
    char b[64];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

std::string report_json(const Report& r) {  // report_to_json (harness.hpp:449-484)
    std::string o = "{\"strategy\":\"" + r.strategy + "\",\"per_step\":[";
    for (size_t i = 0; i < r.steps.size(); ++i) {
        const auto& s = r.steps[i];
        if (i) o += ",";
        o += "{\"step\":" + std::to_string(s.step) + ",\"realized_segments\":" + std::to_string(s.realized) +
             ",\"ttft_tu\":" + fmt_json(s.ttft) + ",\"makespan_tu\":" + fmt_json(s.makespan) +
             ",\"refresh_tu\":" + fmt_json(s.refresh) + ",\"div_l2\":" + fmt_json(s.l2) +
             ",\"div_kl\":" + fmt_json(s.kl) + ",\"plan_sizes\":[";
        for (size_t l = 0; l < s.plan_sizes.size(); ++l) o += (l ? "," : "") + std::to_string(s.plan_sizes[l]);
        o += "],\"reused_tokens\":" + fmt_json(s.reused) + ",\"recomputed_tokens\":" + fmt_json(s.recomputed) +
             ",\"memory_tokens\":" + fmt_json(s.memory) +
             ",\"invalidated_tokens_delta\":" + std::to_string(s.inval_delta) +
             ",\"bytes_loaded_slow_delta\":" + std::to_string(s.slow_delta) + ",\"wall_ms\":" + fmt_json(s.wall_ms) +
             "}";
    }
    o += "],\"aggregate\":{\"steps\":" + std::to_string(r.steps.size()) + ",\"mean_ttft_tu\":" + fmt_json(r.mean_ttft) +
         ",\"p95_ttft_tu\":" + fmt_json(r.p95_ttft) + ",\"mean_div_l2\":" + fmt_json(r.mean_l2) +
         ",\"mean_div_kl\":" + fmt_json(r.mean_kl) + ",\"reuse_ratio\":" + fmt_json(r.reuse_ratio) +
         ",\"mean_realized_segments\":" + fmt_json(r.mean_realized) +
         ",\"invalidated_tokens\":" + std::to_string(r.invalidated) + ",\"bytes_slow\":" + std::to_string(r.bytes_slow) +
         "}}";
    return o;
}

void copy_out(const std::string& s, char* buf, uint64_t cap, uint64_t* len) {
    if (len) *len = s.size();
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
}

Trace* T(void* p) {
    if (!p) fail(KEEP_ERR_CONFIG, "null trace");
    return static_cast<Trace*>(p);
}
Report* R(void* p) {
    if (!p) fail(KEEP_ERR_CONFIG, "null report");
    return static_cast<Report*>(p);
}
Store* ST(void* p) {
    if (!p) fail(KEEP_ERR_CONFIG, "null store");
    return static_cast<Store*>(p);
}

Event event_from(const keep_trace_event& e) {
    Event x;
    x.type = e.type;
    x.step = e.step;
    x.id = e.id;
    x.category = e.category ? e.category : "";
    if (e.n_tokens > 0) x.tokens.assign(e.tokens, e.tokens + e.n_tokens);
    if (e.embedding_dim > 0) x.emb.assign(e.embedding, e.embedding + e.embedding_dim);
    x.eseed = e.embedding_seed;
    x.k = e.k;
    return x;
}
Segment segment_from(const keep_segment& s) {
    Segment x;
    x.id = s.id;
    x.category = s.category ? s.category : "";
    if (s.n_tokens > 0) x.tokens.assign(s.tokens, s.tokens + s.n_tokens);
    if (s.embedding_dim > 0) x.emb.assign(s.embedding, s.embedding + s.embedding_dim);
    return x;
}

}  // namespace

extern "C" {

int keep_trace_generate(const keep_episode_config* cfg, void** out) {
    return guard([&] { *out = new Trace(generate(EpCfg::from(cfg))); });
}

int keep_trace_create(int32_t n, const keep_trace_event* ev, void** out) {
    return guard([&] {  // trace_from_jsonl's checks (harness.hpp:301-322)
        auto tr = std::make_unique<Trace>();
        int64_t prev = 0;
        std::set<uint32_t> known;
        for (int32_t i = 0; i < n; ++i) {
            Event e = event_from(ev[i]);
            if (e.type == KEEP_EVENT_INIT_SEGMENT) {
                if (!known.insert(e.id).second) fail(KEEP_ERR_TRACE, "duplicate init-segment id");
            } else if (e.type == KEEP_EVENT_UPDATE || e.type == KEEP_EVENT_QUERY) {
                if (e.step < prev) fail(KEEP_ERR_TRACE, "trace steps decrease");
                prev = e.step;
                if (e.type == KEEP_EVENT_UPDATE && !known.count(e.id)) fail(KEEP_ERR_TRACE, "update for unknown segment");
            } else {
                fail(KEEP_ERR_TRACE, "unknown trace event type");
            }
            tr->ev.push_back(std::move(e));
        }
        *out = tr.release();
    });
}

int keep_trace_size(void* trace, int32_t* n) {
    return guard([&] { *n = int32_t(T(trace)->ev.size()); });
}

int keep_trace_event_get(void* trace, int32_t i, keep_trace_event* out) {
    return guard([&] {
        const Trace* t = T(trace);
        if (i < 0 || static_cast<size_t>(i) >= t->ev.size()) fail(KEEP_ERR_INPUT, "trace event index out of range");
        const Event& e = t->ev[static_cast<size_t>(i)];
        *out = keep_trace_event{e.type, e.step, e.id, e.category.c_str(), int32_t(e.tokens.size()), e.tokens.data(),
                                int32_t(e.emb.size()), e.emb.data(), e.eseed, e.k};
    });
}

int keep_trace_destroy(void* trace) {
    delete static_cast<Trace*>(trace);
    return KEEP_OK;
}

int keep_store_create(int32_t n, const keep_segment* segs, const keep_store_config* cfg, void** out) {
    return guard([&] {
        if (!cfg) fail(KEEP_ERR_CONFIG, "null store config");
        std::vector<Segment> v;
        for (int32_t i = 0; i < n; ++i) v.push_back(segment_from(segs[i]));
        *out = new Store(std::move(v), StoreCfg{cfg->t, cfg->num_groups, cfg->seed, cfg->grouping == KEEP_GROUPING_FIXED});
    });
}

int keep_store_destroy(void* s) {
    delete static_cast<Store*>(s);
    return KEEP_OK;
}

int keep_store_groups(void* s, int32_t* n_out, int32_t cap, uint32_t* members, int32_t* counts, int32_t* state,
                      uint64_t* gv) {
    return guard([&] {
        const Store* st = ST(s);
        const auto& g = st->groups();
        *n_out = int32_t(g.size());
        int32_t k = 0;
        for (size_t i = 0; i < g.size(); ++i) {
            if (counts) counts[i] = int32_t(g[i].members.size());
            if (state) state[i] = g[i].is_static ? 1 : 0;
            if (gv) gv[i] = st->group_version(uint32_t(i));
            for (uint32_t m : g[i].members) {
                if (members && k < cap) members[k] = m;
                ++k;
            }
        }
        if (members && k > cap) fail(KEEP_ERR_INPUT, "member buffer too small");
    });
}

int keep_store_apply_update(void* s, uint32_t id, int32_t n_tokens, const int32_t* tokens, int64_t step, int32_t cap,
                            keep_owner* owners, uint64_t* toks_out, int32_t* n_out, uint64_t* new_version) {
    return guard([&] {
        const Invalidation rec = ST(s)->apply_update(id, Tokens(tokens, tokens + n_tokens), step);
        *n_out = int32_t(rec.entries.size());
        if (int32_t(rec.entries.size()) > cap) fail(KEEP_ERR_INPUT, "owner buffer too small");
        for (size_t i = 0; i < rec.entries.size(); ++i) {
            owners[i] = rec.entries[i].first.c();
            if (toks_out) toks_out[i] = rec.entries[i].second;
        }
        if (new_version) *new_version = rec.new_versions.front().second;
    });
}

int keep_store_advance_step(void* s, int64_t step, int32_t cap, uint32_t* groups, uint64_t* versions, int32_t* n_out) {
    return guard([&] {
        const auto tr = ST(s)->advance_step(step);
        *n_out = int32_t(tr.size());
        if (int32_t(tr.size()) > cap) fail(KEEP_ERR_INPUT, "transition buffer too small");
        for (size_t i = 0; i < tr.size(); ++i) {
            groups[i] = tr[i].group;
            if (versions) versions[i] = tr[i].version;
        }
    });
}

int keep_store_retrieve(void* s, const double* q, int32_t dim, int32_t k, int32_t cap, keep_owner* units,
                        int32_t* unit_segments, int32_t seg_cap, uint32_t* segments, int32_t* n_units) {
    return guard([&] {
        const auto u = ST(s)->retrieve(std::vector<double>(q, q + dim), k);
        *n_units = int32_t(u.size());
        if (int32_t(u.size()) > cap) fail(KEEP_ERR_INPUT, "unit buffer too small");
        int32_t j = 0;
        for (size_t i = 0; i < u.size(); ++i) {
            units[i] = u[i].owner.c();
            unit_segments[i] = int32_t(u[i].segments.size());
            for (uint32_t m : u[i].segments) {
                if (j >= seg_cap) fail(KEEP_ERR_INPUT, "segment buffer too small");
                segments[j++] = m;
            }
        }
    });
}

int keep_store_add_segment(void* s, const keep_segment* seg, int64_t step) {
    return guard([&] { ST(s)->add_segment(segment_from(*seg), step); });
}

int keep_store_state_sound(void* s, int32_t* out) {
    return guard([&] { *out = ST(s)->state_sound() ? 1 : 0; });
}

int keep_run_episode(void* ctx, void* trace, const char* strategy, const keep_episode_config* cfg, void** out) {
    return guard([&] {
        if (!ctx) fail(KEEP_ERR_CONFIG, "null context");
        *out = new Report(run_episode(ctx, *T(trace), strategy ? strategy : "", EpCfg::from(cfg)));
    });
}

int keep_report_aggregate(void* report, keep_strategy_aggregate* out) {
    return guard([&] {
        const Report& r = *R(report);
        *out = keep_strategy_aggregate{int32_t(r.steps.size()), r.mean_ttft, r.p95_ttft, r.mean_l2, r.mean_kl,
                                       r.reuse_ratio, r.mean_realized, r.invalidated, r.bytes_slow};
    });
}

int keep_report_step(void* report, int32_t i, keep_step_report* out) {
    return guard([&] {
        const Report& r = *R(report);
        if (i < 0 || static_cast<size_t>(i) >= r.steps.size()) fail(KEEP_ERR_INPUT, "step index out of range");
        const StepRow& s = r.steps[static_cast<size_t>(i)];
        *out = keep_step_report{s.step, s.realized, s.ttft, s.makespan, s.refresh, s.l2, s.kl, s.reused, s.recomputed,
                                s.memory, s.inval_delta, s.slow_delta, int32_t(s.plan_sizes.size()),
                                s.plan_sizes.data(), s.wall_ms};
    });
}

int keep_report_json(void* report, char* buf, uint64_t cap, uint64_t* len) {
    return guard([&] { copy_out(report_json(*R(report)), buf, cap, len); });
}

int keep_report_destroy(void* report) {
    delete static_cast<Report*>(report);
    return KEEP_OK;
}

int keep_compare_csv(void* ctx, void* trace, int32_t n_strategies, const char* const* strategies,
                     const keep_episode_config* cfg, int32_t n_k, const int32_t* ks, int32_t n_r, const double* rs,
                     char* buf, uint64_t cap, uint64_t* len) {
    return guard([&] {  // compare_csv (harness.hpp:828-871)
        const EpCfg base = EpCfg::from(cfg);
        const Trace& tr = *T(trace);
        std::string csv =
            "strategy,k,r_avg,mean_ttft_tu,p95_ttft_tu,mean_div_l2,mean_div_kl,reuse_ratio,invalidated_tokens,"
            "bytes_slow\n";
        std::vector<std::pair<int, double>> pts;
        if (n_k > 0)
            for (int i = 0; i < n_k; ++i) pts.emplace_back(ks[i], base.r_avg);
        else if (n_r > 0)
            for (int i = 0; i < n_r; ++i) pts.emplace_back(base.k, rs[i]);
        else
            pts.emplace_back(base.k, base.r_avg);
        for (int si = 0; si < n_strategies; ++si)
            for (const auto& [k, r] : pts) {
                EpCfg c = base;
                c.k = k;
                c.r_avg = r;
                Trace adj = tr;
                for (auto& e : adj.ev)
                    if (e.type == KEEP_EVENT_QUERY) e.k = k;
                const Report rep = run_episode(ctx, adj, strategies[si], c);
                csv += std::string(strategies[si]) + "," + std::to_string(k) + "," + fmt_tu(r) + "," +
                       fmt_tu(rep.mean_ttft) + "," + fmt_tu(rep.p95_ttft) + "," + fmt_tu(rep.mean_l2) + "," +
                       fmt_tu(rep.mean_kl) + "," + fmt_tu(rep.reuse_ratio) + "," + std::to_string(rep.invalidated) +
                       "," + std::to_string(rep.bytes_slow) + "\n";
            }
        copy_out(csv, buf, cap, len);
    });
}

}  // extern "C"
