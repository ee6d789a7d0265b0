// demo.cpp -- the reference's own plan_keep on the CPU (unmodified headers)
// beside the same call through integration/b200_backend.hpp on the B200, on
// identical weights, memory and query.  Exit 0 iff the plans are identical
// (cursor + converge adapter and the one-call device loop) and the final
// query row agrees within 2e-6 of its max magnitude.
//
//   integration/_bin/keep_b200_demo [seed] [S] [L] [H] [d] [mlp] [V]
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "b200_backend.hpp"
#include "keep/prng.hpp"

using namespace keep;

int main(int argc, char** argv) {
    const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 2;
    const int S = argc > 2 ? std::atoi(argv[2]) : 24;
    ModelConfig cfg;
    cfg.num_layers = argc > 3 ? std::atoi(argv[3]) : 4;
    cfg.num_heads = argc > 4 ? std::atoi(argv[4]) : 4;
    cfg.model_dim = argc > 5 ? std::atoi(argv[5]) : 32;
    cfg.mlp_dim = argc > 6 ? std::atoi(argv[6]) : 64;
    cfg.vocab_size = argc > 7 ? std::atoi(argv[7]) : 128;
    cfg.seed = seed;
    try {
        // memory: segments of 8-12 tokens; every third block of 4 is a static group
        Rng rng = Rng::stream(seed, "demo");
        Layout layout;
        std::vector<OwnerRef> owners;
        for (int i = 0; i < S; ++i) {
            TokenSeq t(8 + rng.next_below(5));
            for (auto& x : t) x = int(rng.next_below(uint64_t(cfg.vocab_size)));
            layout.segments.push_back({SegmentId(i), t});
        }
        for (int b = 0, u = 0; b < S; b += 4, ++u) {
            const int e = std::min(S, b + 4);
            if (u % 3 == 0) {
                layout.units.emplace_back(b, e);
                owners.push_back(OwnerRef::group(GroupId(u)));
            } else {
                for (int i = b; i < e; ++i) {
                    layout.units.emplace_back(i, i + 1);
                    owners.push_back(OwnerRef::segment(SegmentId(i)));
                }
            }
        }
        TokenSeq query(8);
        for (auto& x : query) x = int(rng.next_below(uint64_t(cfg.vocab_size)));
        const RatioSchedule sched = ratio_schedule(cfg.num_layers, 0.5);

        // the reference on the CPU: cached KV as the harness builds it
        // (harness.hpp:512-532, 659-677), then plan_keep
        const Model model = Model::init(cfg);
        CachedKV cached;
        for (size_t u = 0; u < layout.units.size(); ++u) {
            const auto [b, e] = layout.units[u];
            Layout members;
            for (int i = b; i < e; ++i) members.segments.push_back(layout.segments[i]);
            members.units.emplace_back(0, e - b);
            const auto kv = full_prefill(model, members, {}).kv;
            int off = 0;
            for (int i = b; i < e; ++i) {
                const int n = int(layout.segments[i].tokens.size());
                std::vector<LayerKV> per;
                for (int l = 0; l < cfg.num_layers; ++l) {
                    LayerKV s{Mat(n, cfg.model_dim), Mat(n, cfg.model_dim)};
                    for (int t = 0; t < n; ++t)
                        for (int j = 0; j < cfg.model_dim; ++j) {
                            s.keys.at(t, j) = kv[l].keys.at(off + t, j);
                            s.values.at(t, j) = kv[l].values.at(off + t, j);
                        }
                    per.push_back(std::move(s));
                }
                cached[layout.segments[i].id] = std::move(per);
                off += n;
            }
        }
        const RecomputePlan ref = plan_keep(model, layout, cached, query, sched);
        const PrefillResult refres = selective_prefill(model, layout, cached, ref, query);

        // the B200 through the adapter
        B200Model bm(cfg);
        const B200Layout bl(layout, owners);
        b200_compute_and_put(bm, bl, 1);
        const RecomputePlan via_cursor = b200_plan_keep(bm, layout, bl, query, sched);
        const RecomputePlan via_device = b200_plan_keep_device(bm, layout, bl, query, sched);
        // final hidden state of the reference plan through the B200 cursor
        B200PrefillCursor cur(bm, bl, query);
        for (int l = 0; l < cfg.num_layers; ++l) {
            std::vector<char> act(size_t(S), 0);
            for (SegmentId s : ref.layers[l]) act[layout.position_of(s)] = 1;
            cur.step(act);
        }
        const int T = int(layout.total_tokens() + query.size());
        const std::vector<float> fh = cur.finish(T, cfg.model_dim);
        double mx = 0.0, err = 0.0;
        for (int j = 0; j < cfg.model_dim; ++j) {
            const double r = refres.final_hidden.at(T - 1, j);
            mx = std::max(mx, std::fabs(r));
            err = std::max(err, std::fabs(double(fh[size_t(T - 1) * cfg.model_dim + j]) - r));
        }
        const bool ok = via_cursor.layers == ref.layers && via_device.layers == ref.layers && err <= 2e-6 * mx;
        std::printf("reference plan sizes:");
        for (auto n : ref.sizes()) std::printf(" %zu", n);
        std::printf(" | b200 cursor+converge %s, b200 plan_keep %s, last row rel err %.2e -> %s\n",
                    via_cursor.layers == ref.layers ? "==" : "!=", via_device.layers == ref.layers ? "==" : "!=",
                    mx > 0 ? err / mx : err, ok ? "OK" : "MISMATCH");
        return ok ? 0 : 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
