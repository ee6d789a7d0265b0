// abi.cu -- the C ABI (include/keep_b200.h) and the host-side engine:
// model weights, the two-tier memory store (load_memory), the prefill cursor
// (prefill_layer), the device selector (importance_evaluation) and the
// plan_keep per-layer loop.  C++ host code; all arithmetic runs in the sm_100a
// kernels -- there is no CPU compute path.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include <unistd.h>

#include "engine.hpp"

using namespace keep_b200;

namespace {

thread_local std::string g_err;
}  // namespace

namespace keep_b200 {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace keep_b200

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return KEEP_OK;
    } catch (const KeepError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return KEEP_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return KEEP_ERR_CUDA;
    }
}

Context* C(void* p) {
    if (!p) raise(KEEP_ERR_CONFIG, "null context");
    auto* c = static_cast<Context*>(p);
    KEEP_CUDA(cudaSetDevice(c->cfg.device));
    return c;
}

uint16_t f2bf(float x) {  // round-to-nearest-even (finite inputs)
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
float bf2f(uint16_t b) {
    uint32_t u = uint32_t(b) << 16;
    float x;
    std::memcpy(&x, &u, 4);
    return x;
}

// ------------------------------------------------------------------ buffers --
}  // namespace

namespace keep_b200 {

void DevBuf::release() {
    if (p) {
        if (host) cudaFreeHost(p);
        else cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
}

void DevBuf::ensure(size_t nbytes) {
    if (nbytes <= bytes && p && !host) return;
    release();  // (cudaFree synchronises the device: growth must stay rare)
    if (nbytes == 0) nbytes = 16;
    if (cudaMalloc(&p, nbytes) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        raise(KEEP_ERR_CUDA, "device out of memory allocating " + std::to_string(nbytes) + " bytes");
    }
    bytes = nbytes;
    host = false;
}

void DevBuf::alloc(size_t nbytes, bool pinned_host) {
    release();
    if (nbytes == 0) nbytes = 16;
    cudaError_t e = pinned_host ? cudaHostAlloc(&p, nbytes, cudaHostAllocDefault) : cudaMalloc(&p, nbytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        raise(KEEP_ERR_CUDA, std::string(pinned_host ? "pinned host" : "device") +
                                 " allocation failed: " + std::to_string(nbytes) + " bytes");
    }
    bytes = nbytes;
    host = pinned_host;
}

// Grow-only with 25% headroom: per-call sizes that drift (a refresh batch of
// a random subset of owners) settle after a few calls instead of reallocating
// -- and synchronising the device -- whenever a call is a little larger.
void ensure_headroom(DevBuf& b, size_t nbytes) {
    if (nbytes <= b.bytes && b.p && !b.host) return;
    b.ensure(nbytes + nbytes / 4);
}

cudaEvent_t Profiler::get() {
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    KEEP_CUDA(cudaEventCreate(&e));
    return e;
}

void Profiler::collect() {
    for (auto& r : pending) {
        KEEP_CUDA(cudaEventSynchronize(r.b));
        float ms = 0.f;
        KEEP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        acc.ms[r.cat] += ms;
        acc.flops[r.cat] += r.flops;
        acc.bytes[r.cat] += r.bytes;
        acc.launches[r.cat] += 1;
        acc.kernels[r.cat] += r.kernels;
        pool.push_back(r.a);
        pool.push_back(r.b);
    }
    pending.clear();
}

Profiler::~Profiler() {
    for (auto& r : pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
}

ProfScope::ProfScope(Profiler& prof, int c, cudaStream_t s, double fl, double by, int nk)
    : p(prof.on ? &prof : nullptr), cat(c), st(s), flops(fl), bytes(by), kernels(nk) {
    if (!p) return;
    a = p->get();
    KEEP_CUDA(cudaEventRecord(a, st));
}

ProfScope::~ProfScope() {
    if (!p) return;
    cudaEvent_t b = p->get();
    if (cudaEventRecord(b, st) != cudaSuccess) return;
    p->pending.push_back(Profiler::Rec{cat, a, b, flops, bytes, kernels});
}

}  // namespace keep_b200

namespace {

template <typename T>
void upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
    b.ensure(sizeof(T) * std::max<size_t>(v.size(), 1));
    if (!v.empty()) upload_bytes(b.p, v.data(), sizeof(T) * v.size(), st);
}

void check_cfg(const keep_config& c) {  // ModelConfig::validate, model.hpp:28-38
    if (c.num_layers < 1) raise(KEEP_ERR_CONFIG, "num_layers must be positive");
    if (c.num_heads < 1) raise(KEEP_ERR_CONFIG, "num_heads must be positive");
    if (c.model_dim < 1) raise(KEEP_ERR_CONFIG, "model_dim must be positive");
    if (c.mlp_dim < 1) raise(KEEP_ERR_CONFIG, "mlp_dim must be positive");
    if (c.vocab_size < 1) raise(KEEP_ERR_CONFIG, "vocab_size must be positive");
    if (c.model_dim % c.num_heads != 0) raise(KEEP_ERR_CONFIG, "model_dim not divisible by num_heads");
    if (c.numerics != KEEP_NUMERICS_PARITY && c.numerics != KEEP_NUMERICS_FAST &&
        c.numerics != KEEP_NUMERICS_PARITY_EXACT)
        raise(KEEP_ERR_CONFIG, "unknown numerics mode");
    if (c.model_dim % 4 != 0) raise(KEEP_ERR_CONFIG, "model_dim must be a multiple of 4");
    if (c.model_dim / c.num_heads > 128) raise(KEEP_ERR_CONFIG, "head_dim > 128 not supported");
    if (c.numerics == KEEP_NUMERICS_FAST && (c.model_dim % 64 != 0 || c.mlp_dim % 64 != 0))
        raise(KEEP_ERR_CONFIG, "FAST numerics needs model_dim and mlp_dim multiples of 64");
    if (c.world_size < 1 || c.rank < 0 || c.rank >= c.world_size) raise(KEEP_ERR_CONFIG, "bad world_size / rank");
    if (c.max_hops < 0) raise(KEEP_ERR_CONFIG, "max_hops must be >= 0 (0 = uncapped)");
    if (c.num_heads % c.world_size != 0) raise(KEEP_ERR_CONFIG, "num_heads must divide by world_size (KV-head shards)");
    if (c.numerics == KEEP_NUMERICS_FAST && (c.model_dim / c.world_size) % 64 != 0)
        raise(KEEP_ERR_CONFIG, "FAST numerics needs model_dim / world_size to be a multiple of 64");
}

// ------------------------------------------------------------ memory store --
uint8_t* layer_keys(const Context& c, const Payload& p, int l) {
    const int64_t sheet = p.arena->rows * c.dl * c.elem;
    if (l >= p.arena->mirror_from)  // HBM-resident layer of a pinned-host arena
        return static_cast<uint8_t*>(p.arena->mirror.p) + (int64_t(l - p.arena->mirror_from) * 2) * sheet +
               p.row0 * c.dl * c.elem;
    return static_cast<uint8_t*>(p.arena->buf.p) + (int64_t(l) * 2) * sheet + p.row0 * c.dl * c.elem;
}

// HBM held by the resident layers of pinned-host arenas
uint64_t resident_bytes(const Context& c) {
    std::vector<const Arena*> seen;
    uint64_t t = 0;
    for (const auto& [k, pl] : c.store) {
        const Arena* a = pl.arena.get();
        if (a->tier != KEEP_TIER_HOST || a->mirror_from >= (1 << 30)) continue;
        if (std::find(seen.begin(), seen.end(), a) != seen.end()) continue;
        seen.push_back(a);
        t += a->mirror.bytes;
    }
    return t;
}

// a write to an arena invalidates its HBM mirror (the mirror is a read copy)
void drop_mirror(Arena& a) {
    if (a.mirror_from >= (1 << 30) || a.split) return;  // a split arena's resident layers live only in HBM
    KEEP_CUDA(cudaDeviceSynchronize());
    a.mirror.release();
    a.mirror_from = 1 << 30;
}
uint8_t* layer_values(const Context& c, const Payload& p, int l) {
    return layer_keys(c, p, l) + p.arena->rows * c.dl * c.elem;
}

constexpr int64_t kArenaPad = 128;  // spare rows per arena layer sheet (query rows of aliased layers)
constexpr int kTpRows = 32;         // sharded layers of at most this many rows split the weights, not the rows

uint64_t resident_bytes(const Context& c);

std::shared_ptr<Arena> make_arena(Context& c, int64_t rows, int tier) {
    auto a = std::make_shared<Arena>();
    a->rows = rows;
    a->used = rows;
    a->tier = tier;
    const size_t per_layer = size_t(2) * rows * c.dl * c.elem;
    int m = 0;  // pinned-host arena under an HBM budget: its deepest m layers live in HBM only
    if (tier == KEEP_TIER_HOST && c.hbm_budget > 0) {
        const uint64_t used = resident_bytes(c);
        m = c.hbm_budget > used ? int(std::min<uint64_t>(uint64_t(c.L), (c.hbm_budget - used) / per_layer)) : 0;
    }
    if (tier == KEEP_TIER_HOST) {
        // pinned pages cannot be swapped: refuse an arena that would leave the
        // host under 16 GB of available RAM rather than invite the OOM killer
        const uint64_t avail = uint64_t(sysconf(_SC_AVPHYS_PAGES)) * uint64_t(sysconf(_SC_PAGESIZE));
        const uint64_t need = uint64_t(per_layer) * uint64_t(c.L - m);
        if (need + (uint64_t(16) << 30) > avail)
            raise(KEEP_ERR_CONFIG, "pinned host arena of " + std::to_string(need >> 30) + " GB would leave less than 16 GB of " +
                                       std::to_string(avail >> 30) + " GB available host RAM (raise the HBM budget)");
    }
    a->buf.alloc(per_layer * size_t(c.L - m), tier == KEEP_TIER_HOST);
    if (m > 0) {
        a->mirror.ensure(per_layer * m);
        a->mirror_from = c.L - m;
        a->split = true;
    }
    return a;
}

bool block_current(const Context& c, const OwnerKey& k, int layer, const Payload** out) {
    auto it = c.store.find(k);
    if (it == c.store.end()) return false;
    auto cv = c.current_version.find(k);
    if (cv == c.current_version.end()) return false;
    if (layer < 0 || layer >= c.L) return false;
    if (!it->second.present[layer] || it->second.layer_version[layer] != cv->second) return false;
    if (out) *out = &it->second;
    return true;
}

std::string owner_str(const OwnerKey& k) {
    return (k.kind == KEEP_OWNER_SEGMENT ? "s" : "g") + std::to_string(k.id);
}

// Resolve each layout segment's owner payload and current version (once per
// prefill, again only if the memory store changed in between).
void resolve_segments(Context& c, int S) {
    c.seg_pl.assign(S, nullptr);
    c.seg_cur.assign(S, 0);
    for (int i = 0; i < S; ++i) {
        auto it = c.store.find(c.seg_owner[i]);
        auto cv = c.current_version.find(c.seg_owner[i]);
        if (it != c.store.end() && cv != c.current_version.end()) {
            c.seg_pl[i] = &it->second;
            c.seg_cur[i] = cv->second;
        }
    }
    c.seg_gen = c.store_gen;
}

// The segment's cached block for layer l if current (cache_manager.hpp:104-116),
// from the per-prefill resolution of cursor_begin (no map lookups per layer).
const Payload* seg_block_current(const Context& c, int i, int l) {
    const Payload* pl = c.seg_pl[i];
    if (!pl || l < 0 || l >= c.L || !pl->present[l] || pl->layer_version[l] != c.seg_cur[i]) return nullptr;
    return pl;
}

// ----------------------------------------------------------- weight access --
void model_alloc_init(Context& c) {
    const int L = c.L, d = c.d, f = c.f, V = c.V, dl = c.dl;
    const int64_t j0 = int64_t(c.R) * dl;  // this rank's head columns of wq / wk / wv
    const double std_ = 1.0 / std::sqrt(double(d));  // model.hpp:56
    cudaStream_t st = c.s_main;
    c.embed.ensure(sizeof(float) * size_t(V) * d);
    c.unembed.ensure(sizeof(float) * size_t(d) * V);
    launch_init_tensor(c.cfg.seed, "embed", V, d, std_, c.embed.p, d, 0, false, st);
    launch_init_tensor(c.cfg.seed, "unembed", d, V, std_, c.unembed.p, V, 0, false, st);
    c.w.clear();
    for (int i = 0; i < L * 4; ++i) c.w.emplace_back(new DevBuf());
    char name[64];
    for (int l = 0; l < L; ++l) {
        auto nm = [&](const char* part) {
            std::snprintf(name, sizeof name, "layer%d.%s", l, part);
            return name;
        };
        if (!c.fast) {
            c.w[l * 4 + W_QKV]->ensure(sizeof(float) * size_t(d) * 3 * dl);
            c.w[l * 4 + W_O]->ensure(sizeof(float) * size_t(d) * d);
            c.w[l * 4 + W_IN]->ensure(sizeof(float) * size_t(d) * f);
            c.w[l * 4 + W_OUT]->ensure(sizeof(float) * size_t(f) * d);
            launch_init_tensor(c.cfg.seed, nm("wq"), d, d, std_, c.wslot(l, W_QKV), 3 * dl, 0, false, st, j0, dl);
            launch_init_tensor(c.cfg.seed, nm("wk"), d, d, std_, c.wslot(l, W_QKV), 3 * dl, dl, false, st, j0, dl);
            launch_init_tensor(c.cfg.seed, nm("wv"), d, d, std_, c.wslot(l, W_QKV), 3 * dl, 2 * dl, false, st, j0, dl);
            launch_init_tensor(c.cfg.seed, nm("wo"), d, d, std_, c.wslot(l, W_O), d, 0, false, st);
            launch_init_tensor(c.cfg.seed, nm("mlp_in"), d, f, std_, c.wslot(l, W_IN), f, 0, false, st);
            launch_init_tensor(c.cfg.seed, nm("mlp_out"), f, d, std_, c.wslot(l, W_OUT), d, 0, false, st);
        } else {
            const size_t b = sizeof(__nv_bfloat16);
            c.w[l * 4 + W_QKV]->ensure(b * size_t(3 * dl) * d);
            c.w[l * 4 + W_O]->ensure(b * size_t(d) * d);
            c.w[l * 4 + W_IN]->ensure(b * size_t(f) * d);
            c.w[l * 4 + W_OUT]->ensure(b * size_t(d) * f);
            launch_init_tensor(c.cfg.seed, nm("wq"), d, d, std_, c.wslot(l, W_QKV), d, 0, true, st, j0, dl);
            launch_init_tensor(c.cfg.seed, nm("wk"), d, d, std_, c.wslot(l, W_QKV), d, dl, true, st, j0, dl);
            launch_init_tensor(c.cfg.seed, nm("wv"), d, d, std_, c.wslot(l, W_QKV), d, 2 * dl, true, st, j0, dl);
            launch_init_tensor(c.cfg.seed, nm("wo"), d, d, std_, c.wslot(l, W_O), d, 0, true, st);
            launch_init_tensor(c.cfg.seed, nm("mlp_in"), d, f, std_, c.wslot(l, W_IN), d, 0, true, st);
            launch_init_tensor(c.cfg.seed, nm("mlp_out"), f, d, std_, c.wslot(l, W_OUT), f, 0, true, st);
        }
    }
    KEEP_CUDA(cudaStreamSynchronize(st));
    c.weights_ready = true;
}

void need_weights(const Context& c) {
    if (!c.weights_ready) raise(KEEP_ERR_CONFIG, "keep_model_init has not been called");
}

// ----------------------------------------------------------------- passes --
// Segment-aligned key splits so that every (row, destination segment) bin is
// produced by exactly one CTA (deterministic, no atomics).
// KEEP_ATTN_SIMT=1 forces the CUDA-core attention in FAST mode (A/B checks).
bool use_tc_attention(const Context& c) {
    static const bool simt = [] {
        const char* e = std::getenv("KEEP_ATTN_SIMT");
        return e && *e == '1';
    }();
    return c.fast && c.dh == 128 && !simt;
}

// Per layer: a 128-row tensor-core tile is mostly padding when only a few
// rows are recomputed (the deep layers: the query alone); those layers take
// the CUDA-core path when n <= KEEP_ATTN_SMALL_N (A/B knob).
int small_n_threshold() {
    static const int v = [] {
        const char* e = std::getenv("KEEP_ATTN_SMALL_N");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}
bool use_tc_attention(const Context& c, const Pass& p) { return use_tc_attention(c) && p.n > small_n_threshold(); }

bool batch_multi_decode() {  // KEEP_BATCH_MULTI=0: per-query decode in batches (A/B)
    static const bool on = [] {
        const char* e = std::getenv("KEEP_BATCH_MULTI");
        return !(e && *e == '0');
    }();
    return on;
}

// Few computed rows and no summary to bin (the layers after the walk):
// flash decoding (attn_decode.cu).  KEEP_ATTN_DECODE=0 keeps the two-pass
// tensor-core kernel (A/B).
bool use_decode_attention(const Context& c, const Pass& p) {
    static const bool on = [] {
        const char* e = std::getenv("KEEP_ATTN_DECODE");
        return !(e && *e == '0');
    }();
    return on && c.fast && c.dh == 128 && !p.with_summary && !p.block_diag && decode_attention_fits(p.n);
}

void plan_splits(Context& c, Pass& p) {
    const bool tc = use_tc_attention(c, p);
    // the split plan depends only on (n, T, path): layers of equal size reuse
    // the uploaded arrays (no host->device staging on the deep layers)
    const int64_t key = (int64_t(p.n) << 32) ^ (int64_t(p.T) << 2) ^ (tc ? 1 : 0) ^ (p.block_diag ? 2 : 0) ^
                        (int64_t(p.with_summary) << 62);
    if (key == p.split_key) return;
    p.split_key = key;
    const bool dmma = !c.fast && !c.exact && parity_attention_dmma(c.dh);
    const int tiles = int(ceil_div(p.n, tc ? 128 : (dmma ? attention_dmma_rows_per_tile() : 16)));
    int nsplit = 1;
    if (tc && !p.block_diag) {
        // stats / context: unaligned key splits.  One CTA per SM (smem), so
        // pick the split count minimising (waves of CTAs) x (chunks per CTA):
        // few-row layers (the query alone) otherwise lose a third of a wave.
        int na = 1;
        static const int forced = [] {
            const char* e = std::getenv("KEEP_ATTN_SPLITS");  // A/B knob
            return e ? std::atoi(e) : 0;
        }();
        if (forced > 0) {
            na = forced;
        } else if (int64_t(tiles) * c.H < 2 * kNumSMs) {
            int64_t best = INT64_MAX;
            const int64_t nch = ceil_div(p.T, 128);
            for (int cand = 1; cand <= std::min<int64_t>(32, nch); ++cand) {
                const int64_t waves = ceil_div(int64_t(tiles) * c.H * cand, kNumSMs);
                const int64_t cost = waves * (ceil_div(nch, cand) + 2);  // +2: per-CTA prologue / epilogue
                if (cost < best) {
                    best = cost;
                    na = cand;
                }
            }
        }
        std::vector<int32_t> lo, hi;
        const int64_t step = ceil_div(ceil_div(p.T, na), 128) * 128;
        for (int64_t k = 0; k < p.T; k += step) {
            lo.push_back(int32_t(k));
            hi.push_back(int32_t(std::min<int64_t>(p.T, k + step)));
        }
        upload(p.split_lo_a, lo, c.s_main);
        upload(p.split_hi_a, hi, c.s_main);
        p.split_count_a = int(lo.size());
    } else {
        std::vector<int32_t> lo{0}, hi{p.T};
        upload(p.split_lo_a, lo, c.s_main);
        upload(p.split_hi_a, hi, c.s_main);
        p.split_count_a = 1;
    }
    if (!p.block_diag) {
        const int target = tc ? 2 * kNumSMs : 4 * kNumSMs;
        // (the DMMA kernels run one 256-thread CTA per (row tile, head, split) and SM)
        const int64_t ctas = dmma ? int64_t(tiles) * c.Hl : tiles;
        // (the fp64 decode kernel: one CTA per (head, split), two per SM, a few waves)
        const bool f64dec = dmma && attention_f64_decode(p.n, c.dh, p.with_summary);
        const int64_t want = f64dec ? 6 * kNumSMs : (dmma ? 2 * kNumSMs : target);
        nsplit = int(std::min<int64_t>(ceil_div(want, ctas), std::max(1, p.T / 128)));
        // bound the fp64 partial-context scratch to ~512 MB
        const int64_t per_split = int64_t(p.n) * c.dl * 8;
        nsplit = int(std::max<int64_t>(1, std::min<int64_t>(nsplit, (512ll << 20) / std::max<int64_t>(per_split, 1))));
    }
    // segment-aligned key splits (a segment's keys never straddle two splits:
    // every rowbin (row, segment) entry is written by exactly one CTA)
    auto seg_splits = [&](int ns_want, std::vector<int32_t>& lo, std::vector<int32_t>& hi) {
        lo.clear();
        hi.clear();
        if (ns_want <= 1) {
            lo.push_back(0);
            hi.push_back(p.T);
            return;
        }
        // candidate cut points: segment starts and the query start
        std::vector<int32_t> cuts;
        for (int i = 0; i < p.S; ++i) cuts.push_back(p.seg_start[i]);
        cuts.push_back(p.Tm);
        int32_t prev = 0;
        lo.push_back(0);
        for (int k = 1; k < ns_want; ++k) {
            const int64_t want = int64_t(k) * p.T / ns_want;
            auto it = std::lower_bound(cuts.begin(), cuts.end(), int32_t(want));
            if (it == cuts.end()) break;
            if (*it <= prev) continue;
            hi.push_back(*it);
            lo.push_back(*it);
            prev = *it;
        }
        hi.push_back(p.T);
    };
    std::vector<int32_t> lo, hi;
    seg_splits(nsplit, lo, hi);
    upload(p.split_lo, lo, c.s_main);
    upload(p.split_hi, hi, c.s_main);
    if (dmma && !p.block_diag) {
        // the DMMA bins pass loops the heads inside one CTA per (row tile,
        // split): it needs its own, finer split plan to fill the machine
        std::vector<int32_t> blo, bhi;
        seg_splits(int(std::min<int64_t>(ceil_div(8 * kNumSMs, tiles), std::max(1, p.T / 256))), blo, bhi);
        upload(p.split_lo_b, blo, c.s_main);
        upload(p.split_hi_b, bhi, c.s_main);
        p.split_count_b = int(blo.size());
    } else {
        upload(p.split_lo_b, lo, c.s_main);
        upload(p.split_hi_b, hi, c.s_main);
        p.split_count_b = int(lo.size());
    }
    const int ns = int(lo.size());
    const int nm = std::max(ns, p.split_count_a);
    p.m_part.ensure(sizeof(double) * size_t(nm) * p.n * c.H);
    p.l_part.ensure(sizeof(double) * size_t(nm) * p.n * c.H);
    p.m_fin.ensure(sizeof(double) * size_t(p.n) * c.H);
    p.l_fin.ensure(sizeof(double) * size_t(p.n) * c.H);
    if (ns > 1 && !tc) p.o_part.ensure(sizeof(double) * size_t(ns) * p.n * c.dl);
    if (tc && p.split_count_a > 1) p.o_part.ensure(sizeof(float) * size_t(p.split_count_a) * p.n * c.dl);
    p.split_count = ns;
}

// MLP rows per chunk: the hidden activation [rows x f] is bounded (4 GB), so a
// batch of queries with ~10^5 active rows each (BASELINE configs[4]) does not
// need a [rows x f] buffer of tens of GB; chunks of >= 32K rows keep the
// GEMMs in their full-wave regime
size_t mlp_chunk_rows(const Context& c) {
    static const size_t forced = [] {  // tests: small chunks at test sizes
        const char* e = std::getenv("KEEP_MLP_CHUNK_ROWS");
        return e ? size_t(std::max(1, std::atoi(e))) : size_t(0);
    }();
    if (forced) return forced;
    const size_t es = c.fast ? 2 : 4;
    return std::max<size_t>(32768, (size_t(4) << 30) / (es * size_t(c.f)));
}

// KEEP_LAZY_SUMMARY=0: always compute the summary a walk would read (A/B)
bool lazy_summary_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KEEP_LAZY_SUMMARY");
        return !(e && *e == '0');
    }();
    return on;
}

void ensure_layer_scratch(Context& c, Pass& p) {
    const size_t n = size_t(std::max(p.n, 1));
    // sharded: ctx rows padded to G equal row blocks (all-to-all), Wo / MLP on one block
    const size_t cpr = size_t(ceil_div(int64_t(n), c.G));
    const size_t es = c.fast ? 2 : 4;
    ensure_headroom(p.q, es * n * c.dl);
    ensure_headroom(c.fast ? p.ctxb : p.ctx, es * cpr * c.G * c.dl);
    ensure_headroom(c.fast ? p.hb : p.h, es * std::min<size_t>(cpr, mlp_chunk_rows(c)) * c.f);
    if (c.G > 1) {
        p.xrecv.ensure(es * cpr * c.G * c.dl);
        p.xrows.ensure(es * cpr * c.d);
    }
}

void ensure_attn_scratch(Context& c, Pass& p) {
    const size_t n = size_t(std::max(p.n, 1));
    if (p.with_summary && !use_tc_attention(c, p)) p.rowbin.ensure((c.fast ? 4 : 8) * n * std::max(p.S, 1));
}

// Algorithmic attention work of a layer: sum over computed rows of visible keys.
double visible_pairs(const Pass& p) {
    double s = 0.0;
    for (int32_t r : p.rows_h) s += double(r + 1 - (p.block_diag ? p.key_lo_h[r] : 0));
    return s;
}

// One transformer layer over the compact rows of a pass
// (PrefillCursor::step body, prefill.hpp:245-304 minus the cached copy), in
// three phases so that a batch of queries can share the projections and run
// attention per query: layer_qkv (K3), layer_attention (K5 + K6),
// layer_dense (K8 + K9, with the sharded exchanges around them).
// run_layer's after_summary runs once the layer's segment summary is complete
// (the selector for layer l+1 overlaps this layer's Wo + MLP; SPEC D2).
//
// KV-head sharding (G > 1): QKV and attention run for this
// rank's heads over all compact rows (q/k/v/ctx are dl = d/G columns wide,
// the merged KV holds this rank's head columns); the fp64 summary is summed
// over ranks (identical bits everywhere, so the selector runs replicated);
// ctx goes head-sharded -> row-sharded by all-to-all; Wo + MLP run with the
// full weights on this rank's block of rows (every k-reduction stays on one
// GPU, as on a single GPU); the fp32 residual rows are all-gathered.
void layer_qkv(Context& c, Pass& p, int l) {
    const int n = p.n, d = c.d, dl = c.dl;
    cudaStream_t st = c.s_main;
    const int32_t* rows = p.d_rows.as<int32_t>();
    const double wb = c.fast ? 2.0 : 4.0;
    const double gq = 2.0 * n * 3.0 * dl * d;
    const double bq = wb * (3.0 * dl * d + n * double(d)) + c.elem * 3.0 * n * dl;
    ProfScope ps(c.prof, KEEP_PROF_QKV, st, gq, bq);
    if (!c.fast) {
        EpiArgs e{EPI_QKV, dl, p.q.as<float>(), dl, p.kdst[l], p.vdst[l], rows, nullptr};
        launch_gemm_parity(p.x.as<float>(), d, static_cast<const float*>(c.wslot(l, W_QKV)), 3 * dl, n, 3 * dl, d, e,
                           st, c.oz, c.exact);
    } else {
        EpiArgs e{EPI_QKV, dl, nullptr, dl, p.kdst[l], p.vdst[l], rows, p.q.as<__nv_bfloat16>()};
        if (use_tc_attention(c, p)) e.q_scale = float(1.4426950408889634 / std::sqrt(double(c.dh)));
        launch_gemm_bf16(p.xb.as<__nv_bfloat16>(), d, static_cast<const __nv_bfloat16*>(c.wslot(l, W_QKV)), d, n,
                         3 * dl, d, e, st);
    }
    if (c.rope_theta > 0.0)  // opt-in RoPE: q and the new key rows at their positions (owner-local in a refresh)
        launch_rope_qk(p.q.p, p.kdst[l], n, rows, p.block_diag ? p.d_key_lo.as<int32_t>() : nullptr, dl, c.dh,
                       c.rope_theta, c.fast, st);
}

// Attention of the pass's compact rows against a [p.T x dl] merged KV (k, v;
// p.rows are positions in it), q / ctx given explicitly: a batch runs one
// query instance at a time on slices of its shared buffers.  With a summary
// the normalised AttentionSummary lands in p.summ.
void layer_attention(Context& c, Pass& p, int l, const void* q, void* ctx, const void* k, const void* v) {
    const int n = p.n, dl = c.dl;
    cudaStream_t st = c.s_main;
    (void)l;
    ensure_attn_scratch(c, p);
    plan_splits(c, p);
    const int32_t* rows = p.d_rows.as<int32_t>();
    AttnArgs a{};
    a.n = n;
    a.T = p.T;
    a.H = c.Hl;
    a.dh = c.dh;
    a.d = dl;
    a.inv_heads = 1.0 / c.H;
    a.k = k;
    a.v = v;
    a.rows = rows;
    a.row_seg = p.d_row_seg.as<int32_t>();
    a.key_lo = p.block_diag ? p.d_key_lo.as<int32_t>() : nullptr;
    a.with_bins = p.with_summary;
    a.exact = c.exact;
    a.S = p.S;
    a.nsplit = p.split_count;
    a.split_lo = p.split_lo.as<int32_t>();
    a.split_hi = p.split_hi.as<int32_t>();
    a.nsplit_b = p.split_count_b;
    a.split_lo_b = p.split_lo_b.as<int32_t>();
    a.split_hi_b = p.split_hi_b.as<int32_t>();
    a.rows_per_tile = 16;
    a.m_part = p.m_part.as<double>();
    a.l_part = p.l_part.as<double>();
    a.m_fin = p.m_fin.as<double>();
    a.l_fin = p.l_fin.as<double>();
    a.o_part = p.o_part.as<double>();
    a.rowbin = p.rowbin.p;
    a.ebin = nullptr;
    a.seg_start = p.d_seg_start.as<int32_t>();
    a.Tm = p.Tm;
    if (!c.fast && !c.exact && p.with_summary && !p.block_diag && parity_attention_dmma(c.dh) &&
        dmma_fused_bins(c.dh)) {
        // per-head segment sums of the fused bins: fp64 [H x n x S], grown only
        // while the device keeps 4 GB free (else the separate bins pass)
        const size_t need = sizeof(double) * size_t(c.Hl) * n * size_t(p.S);
        bool fits = need <= p.ebin.bytes;
        if (!fits) {
            size_t fr = 0, tot = 0;
            KEEP_CUDA(cudaMemGetInfo(&fr, &tot));
            fits = need + (size_t(4) << 30) <= fr + p.ebin.bytes;
        }
        if (fits) {
            p.ebin.ensure(need);
            a.ebin = p.ebin.as<double>();
            p.attn_flag.ensure(16 + sizeof(double) * size_t(c.Hl));  // flag + per-head key-norm max
            a.flag = p.attn_flag.as<int>();
        }
    }

    const double pairs = visible_pairs(p);
    // algorithmic attention: QK^T and PV over visible keys; K+V of the layer read once
    const double fa = 4.0 * dl * pairs, ba = double(c.elem) * (2.0 * p.T * dl + 2.0 * n * dl);
    if (!c.fast) {
        a.q = q;
        a.ctx = static_cast<float*>(ctx);
        {
            ProfScope ps(c.prof, KEEP_PROF_ATTN, st, fa, ba, 5);
            launch_attention_parity(a, st);
        }
    } else {
        a.q = q;
        a.ctx_bf16 = static_cast<__nv_bfloat16*>(ctx);
        if (use_tc_attention(c, p) && use_decode_attention(c, p)) {
            // the query rows alone (walk over): HBM-bound single-pass decoding
            const int kv_hi = p.rows_h.back() + 1;
            const int ns = decode_splits(c.Hl, kv_hi);
            p.m_part.ensure(sizeof(float) * size_t(ns) * n * c.Hl);
            p.l_part.ensure(sizeof(float) * size_t(ns) * n * c.Hl);
            p.o_part.ensure(sizeof(float) * size_t(ns) * n * dl);
            ProfScope ps(c.prof, KEEP_PROF_DECODE, st, fa, double(c.elem) * (2.0 * kv_hi * dl + 2.0 * n * dl), 2);
            AttnTcLaunch t{};
            t.n = n;
            t.T = p.T;
            t.H = c.Hl;
            t.d = dl;
            t.q = q;
            t.k = k;
            t.v = v;
            t.rows = rows;
            t.m_part = p.m_part.as<float>();
            t.l_part = p.l_part.as<float>();
            t.o_part = p.o_part.as<float>();
            t.ctx = static_cast<__nv_bfloat16*>(ctx);
            ps.kernels = launch_attention_decode(t, kv_hi, st);
        } else if (use_tc_attention(c, p)) {
            ProfScope ps(c.prof, KEEP_PROF_ATTN, st, fa, ba, p.split_count_a > 1 ? 6 : 5);
            p.vt.ensure(2 * size_t(dl) * size_t(ceil_div(p.T, 64) * 64));
            AttnTcLaunch t{};
            t.n = n;
            t.T = p.T;
            t.H = c.Hl;
            t.d = dl;
            t.S = p.S;
            t.inv_heads = 1.0 / c.H;
            t.q = q;
            t.k = k;
            t.v = v;
            t.vt = p.vt.as<__nv_bfloat16>();
            t.rows = rows;
            t.row_seg = p.d_row_seg.as<int32_t>();
            t.key_lo = a.key_lo;
            t.with_bins = p.with_summary;
            t.nsplit_a = p.split_count_a;
            t.split_lo_a = p.split_lo_a.as<int32_t>();
            t.split_hi_a = p.split_hi_a.as<int32_t>();
            t.m_part = p.m_part.as<float>();
            t.l_part = p.l_part.as<float>();
            t.m_fin = p.m_fin.as<float>();
            t.inv_l = p.l_fin.as<float>();
            t.o_part = p.o_part.as<float>();
            t.ctx = static_cast<__nv_bfloat16*>(ctx);
            if (p.with_summary) {
                const size_t ns = size_t(p.S) + size_t(p.S) * p.S;
                p.summ_raw.ensure(sizeof(double) * ns);
                p.summ.ensure(sizeof(double) * ns);
                t.summ_raw = p.summ_raw.as<double>();
                t.summ = p.summ.as<double>();
            }
            t.seg_len = p.d_seg_len.as<int32_t>();
            t.qlen = p.qlen;
            t.chunk_tab = p.chunk_tab.p;
            t.zt = p.zt.p;
            t.nb = p.nb;
            ps.kernels = launch_attention_tc(t, st);
        } else {
            ProfScope ps(c.prof, KEEP_PROF_ATTN, st, fa, ba, 5);
            launch_attention_fast(a, st);
        }
    }
    if (p.with_summary && !use_tc_attention(c, p)) {  // (the tensor-core path bins inside attention)
        ProfScope ps(c.prof, KEEP_PROF_SUMMARY, st, 0.0, (c.fast ? 4.0 : 8.0) * n * double(p.S) + 8.0 * p.S * double(p.S));
        // compact row range per segment (rows of a segment are contiguous)
        std::vector<int32_t> cb(p.S, 0), ce(p.S, 0);
        int qb = n, qe = n;
        for (int i = 0; i < n;) {
            const int sg = p.row_seg[p.rows_h[i]];
            int j = i;
            while (j < n && p.row_seg[p.rows_h[j]] == sg) ++j;
            if (sg >= 0) {
                cb[sg] = i;
                ce[sg] = j;
            } else {
                qb = i;
                qe = j;
            }
            i = j;
        }
        upload(p.seg_cbeg, cb, st);
        upload(p.seg_cend, ce, st);
        p.summ.ensure(sizeof(double) * (size_t(p.S) + size_t(p.S) * p.S));
        if (!c.fast)
            launch_summary_reduce<double>(p.rowbin.as<double>(), p.S, p.seg_cbeg.as<int32_t>(), p.seg_cend.as<int32_t>(),
                                          p.d_seg_len.as<int32_t>(), qb, qe, p.qlen, p.summ.as<double>(), st);
        else
            launch_summary_reduce<float>(p.rowbin.as<float>(), p.S, p.seg_cbeg.as<int32_t>(), p.seg_cend.as<int32_t>(),
                                         p.d_seg_len.as<int32_t>(), qb, qe, p.qlen, p.summ.as<double>(), st);
    }
}

void layer_dense(Context& c, Pass& p, int l) {
    const int n = p.n, d = c.d, f = c.f, dl = c.dl;
    cudaStream_t st = c.s_main;
    const int G = c.G;
    const int cpr = int(ceil_div(n, G));
    const int r0 = std::min(n, c.R * cpr);
    const int m = std::min(n, r0 + cpr) - r0;
    const double wb = c.fast ? 2.0 : 4.0;  // weight / activation element bytes
    const double go = 2.0 * m * double(d) * d, gi = 2.0 * m * double(d) * f;
    const double bo = wb * (double(d) * d + m * double(d)) + 8.0 * m * d;
    const double bi = wb * (double(d) * f + m * double(d) + m * double(f));
    const double bout = wb * (double(d) * f + m * double(f)) + 8.0 * m * d;
    (void)dl;
    if (G > 1 && !c.fast && !c.exact && n <= kTpRows && f % G == 0) {
        // Few rows (every layer after the walk: the query alone).  Wo + MLP are
        // a weight stream here, so the ranks split the WEIGHTS instead of the
        // rows: Wo row-parallel over this rank's head columns of ctx (no
        // all-to-all), MLP-in column-parallel (relu on this rank's f / G
        // columns), MLP-out row-parallel; each row-parallel product is an fp64
        // partial sum all-reduced in a fixed order (identical bits on every
        // rank), then x += float(sum) as prefill.hpp:289-291 / 302-303 round
        // it.  Only the order of the fp64 k-sum changes.
        const int c0 = c.R * dl, fl = f / G, f0 = c.R * fl;
        p.tp_part.ensure(sizeof(double) * size_t(n) * d);
        p.tp_h.ensure(sizeof(float) * size_t(n) * fl);
        double* part = p.tp_part.as<double>();
        float* x = p.x.as<float>();
        const EpiArgs ef{EPI_F64, d, reinterpret_cast<float*>(part), d, nullptr, nullptr, nullptr, nullptr};
        {
            ProfScope ps(c.prof, KEEP_PROF_WO, st, 2.0 * n * double(dl) * d, 4.0 * double(dl) * d);
            launch_gemm_f64acc(p.ctx.as<float>(), dl, static_cast<const float*>(c.wslot(l, W_O)) + size_t(c0) * d, d, n,
                               d, dl, ef, st, false);
        }
        {
            ProfScope ps(c.prof, KEEP_PROF_COMM, st, 0.0, 8.0 * n * double(d) * 2.0 * (G - 1) / G, 2);
            c.comm->allreduce_f64(part, size_t(n) * d, st);
        }
        launch_f64_resid(part, x, n, d, d, st);
        {
            ProfScope ps(c.prof, KEEP_PROF_MLP_IN, st, 2.0 * n * double(d) * fl, 4.0 * double(d) * fl);
            const EpiArgs ei{EPI_RELU, d, p.tp_h.as<float>(), fl, nullptr, nullptr, nullptr, nullptr};
            launch_gemm_f64acc(x, d, static_cast<const float*>(c.wslot(l, W_IN)) + f0, f, n, fl, d, ei, st, false);
        }
        {
            ProfScope ps(c.prof, KEEP_PROF_MLP_OUT, st, 2.0 * n * double(fl) * d, 4.0 * double(fl) * d);
            launch_gemm_f64acc(p.tp_h.as<float>(), fl, static_cast<const float*>(c.wslot(l, W_OUT)) + size_t(f0) * d, d, n,
                               d, fl, ef, st, false);
        }
        {
            ProfScope ps(c.prof, KEEP_PROF_COMM, st, 0.0, 8.0 * n * double(d) * 2.0 * (G - 1) / G, 2);
            c.comm->allreduce_f64(part, size_t(n) * d, st);
        }
        launch_f64_resid(part, x, n, d, d, st);
        return;
    }
    // attention context for the Wo + MLP rows of this rank
    const int es = c.fast ? 2 : 4;
    const void* ctx_rows = c.fast ? static_cast<const void*>(p.ctxb.p) : static_cast<const void*>(p.ctx.p);
    if (G > 1) {
        {
            ProfScope ps(c.prof, KEEP_PROF_COMM, st, 0.0, double(es) * cpr * dl * (G - 1), 1);
            c.comm->alltoall(c.fast ? p.ctxb.p : p.ctx.p, p.xrecv.p, size_t(es) * cpr * dl, st);
        }
        ProfScope ps(c.prof, KEEP_PROF_XCHG, st, 0.0, 2.0 * es * double(m) * d);
        launch_pack_heads(p.xrecv.p, G, cpr, m, dl, es, p.xrows.p, st);
        ctx_rows = p.xrows.p;
    }
    float* xr = p.x.as<float>() + int64_t(r0) * d;
    if (m > 0) {
        if (!c.fast) {
            EpiArgs eo{EPI_RESID, d, xr, d, nullptr, nullptr, nullptr, nullptr};
            {
                ProfScope ps(c.prof, KEEP_PROF_WO, st, go, bo);
                launch_gemm_parity(static_cast<const float*>(ctx_rows), d, static_cast<const float*>(c.wslot(l, W_O)), d, m,
                                   d, d, eo, st, c.oz, c.exact);
            }
            const int mc = int(std::min<size_t>(size_t(m), mlp_chunk_rows(c)));
            for (int q0 = 0; q0 < m; q0 += mc) {  // row chunks: the hidden buffer stays bounded
                const int mq = std::min(mc, m - q0);
                float* xq = xr + int64_t(q0) * d;
                {
                    ProfScope ps(c.prof, KEEP_PROF_MLP_IN, st, gi * mq / m, bi);
                    EpiArgs ei{EPI_RELU, d, p.h.as<float>(), f, nullptr, nullptr, nullptr, nullptr};
                    launch_gemm_parity(xq, d, static_cast<const float*>(c.wslot(l, W_IN)), f, mq, f, d, ei, st, c.oz,
                                       c.exact);
                }
                {
                    ProfScope ps(c.prof, KEEP_PROF_MLP_OUT, st, gi * mq / m, bout);
                    EpiArgs eq{EPI_RESID, d, xq, d, nullptr, nullptr, nullptr, nullptr};
                    launch_gemm_parity(p.h.as<float>(), f, static_cast<const float*>(c.wslot(l, W_OUT)), d, mq, d, f, eq, st,
                                       c.oz, c.exact);
                }
            }
        } else {
            auto* xbr = p.xb.as<__nv_bfloat16>() + int64_t(r0) * d;
            const int mc = c.gemm_ctas;
            EpiArgs eo{EPI_RESID, d, xr, d, nullptr, nullptr, nullptr, xbr};
            {
                ProfScope ps(c.prof, KEEP_PROF_WO, st, go, bo);
                launch_gemm_bf16(static_cast<const __nv_bfloat16*>(ctx_rows), d,
                                 static_cast<const __nv_bfloat16*>(c.wslot(l, W_O)), d, m, d, d, eo, st, mc);
            }
            const int rc = int(std::min<size_t>(size_t(m), mlp_chunk_rows(c)));
            for (int q0 = 0; q0 < m; q0 += rc) {  // row chunks: the hidden buffer stays bounded
                const int mq = std::min(rc, m - q0);
                {
                    ProfScope ps(c.prof, KEEP_PROF_MLP_IN, st, gi * mq / m, bi);
                    EpiArgs ei{EPI_RELU, d, nullptr, f, nullptr, nullptr, nullptr, p.hb.as<__nv_bfloat16>()};
                    launch_gemm_bf16(xbr + int64_t(q0) * d, d, static_cast<const __nv_bfloat16*>(c.wslot(l, W_IN)), d, mq,
                                     f, d, ei, st, mc);
                }
                {
                    ProfScope ps(c.prof, KEEP_PROF_MLP_OUT, st, gi * mq / m, bout);
                    EpiArgs eq{EPI_RESID, d, xr + int64_t(q0) * d, d, nullptr, nullptr, nullptr, xbr + int64_t(q0) * d};
                    launch_gemm_bf16(p.hb.as<__nv_bfloat16>(), f, static_cast<const __nv_bfloat16*>(c.wslot(l, W_OUT)), f,
                                     mq, d, f, eq, st, mc);
                }
            }
        }
    }
    if (G > 1) {
        {
            ProfScope ps(c.prof, KEEP_PROF_COMM, st, 0.0, 4.0 * cpr * double(d) * (G - 1), 1);
            c.comm->allgather(p.x.as<float>() + int64_t(c.R) * cpr * d, p.x.p, sizeof(float) * size_t(cpr) * d, st);
        }
        if (c.fast) {
            ProfScope ps(c.prof, KEEP_PROF_XCHG, st, 0.0, 6.0 * double(n) * d);
            launch_to_bf16(p.x.as<float>(), int64_t(n) * d, p.xb.as<__nv_bfloat16>(), st);
        }
    }
}

template <class AfterSummary>
void run_layer(Context& c, Pass& p, int l, AfterSummary&& after_summary) {
    if (p.n == 0) return;
    ensure_layer_scratch(c, p);
    layer_qkv(c, p, l);
    if (p.walk_probe && p.with_summary) {
        // lazy summary: when no candidate segment can receive query probability this
        // layer, the walk's first hop adds nothing (recompute.hpp:110-121) and the
        // summary is never read -- the layer runs its plain attention pass
        p.d_probe.ensure(16 + sizeof(uint64_t) * 17 * size_t(c.Hl));
        int* flag = p.d_probe.as<int>();
        launch_walk_probe(p.q.as<float>(), static_cast<const float*>(p.kdst[l]), p.d_rows.as<int32_t>(),
                          p.d_row_seg.as<int32_t>(), p.d_walk_cand.as<uint8_t>(), p.n, p.qlen, p.Tm, c.Hl, c.dh, c.dl,
                          reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(p.d_probe.p) + 16), flag, c.s_main);
        int need = 1;
        KEEP_CUDA(cudaMemcpyAsync(&need, flag, sizeof(int), cudaMemcpyDeviceToHost, c.s_main));
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
        if (!need) {
            p.with_summary = false;
            p.walk_empty = true;
        }
    }
    layer_attention(c, p, l, p.q.p, c.fast ? p.ctxb.p : p.ctx.p, p.kdst[l], p.vdst[l]);
    if (c.G > 1 && p.with_summary && p.summary_global) {
        // per-rank partials (sum over this rank's heads of p / H) -> the summary
        const size_t ns = size_t(p.S) + size_t(p.S) * p.S;
        ProfScope ps(c.prof, KEEP_PROF_COMM, c.s_main, 0.0, 8.0 * ns * 2.0 * (c.G - 1) / c.G, 2);
        c.comm->allreduce_f64(p.summ.as<double>(), ns, c.s_main);
    }
    after_summary();
    layer_dense(c, p, l);
}

void run_layer(Context& c, Pass& p, int l) {
    run_layer(c, p, l, [] {});
}

// Planning estimate of one layer's device time (the K10 pre-load window):
// recompute GEMMs at ~1.1 PFLOP/s and attention at ~0.35 PFLOP/s per GPU
// (the measured C3 rates), the analogue of the reference's CostModel.
double layer_estimate_ms(const Context& c, const Pass& p) {
    const double n = p.n, d = c.d, f = c.f, dl = c.dl;
    const double m = std::ceil(n / c.G);
    const double gemm = 2.0 * n * 3.0 * dl * d + 2.0 * m * (d * d + 2.0 * d * f);
    const double attn = 4.0 * dl * visible_pairs(p);
    return (gemm / 1.1e15 + attn / 0.35e15) * 1e3;
}

// The four K4 argument arrays in one device buffer and one upload:
// [ksrc ptrs][vsrc ptrs][dst rows][row counts].
void upload_copy_args(Context& c, const std::vector<void*>& ks, const std::vector<void*>& vs,
                      const std::vector<int32_t>& dr, const std::vector<int32_t>& nr, cudaStream_t st,
                      const void* const** kp, const void* const** vp, const int32_t** dp, const int32_t** np) {
    const size_t n = ks.size();
    std::vector<uint8_t> blob(n * (2 * sizeof(void*) + 2 * sizeof(int32_t)));
    std::memcpy(blob.data(), ks.data(), n * sizeof(void*));
    std::memcpy(blob.data() + n * sizeof(void*), vs.data(), n * sizeof(void*));
    std::memcpy(blob.data() + 2 * n * sizeof(void*), dr.data(), n * sizeof(int32_t));
    std::memcpy(blob.data() + 2 * n * sizeof(void*) + n * sizeof(int32_t), nr.data(), n * sizeof(int32_t));
    upload(c.d_ksrc, blob, st);
    const uint8_t* b = c.d_ksrc.as<const uint8_t>();
    *kp = reinterpret_cast<const void* const*>(b);
    *vp = reinterpret_cast<const void* const*>(b + n * sizeof(void*));
    *dp = reinterpret_cast<const int32_t*>(b + 2 * n * sizeof(void*));
    *np = reinterpret_cast<const int32_t*>(b + 2 * n * sizeof(void*) + n * sizeof(int32_t));
}

// Replace the compact row set (rows only shrink): gather the residual rows.
void set_rows(Context& c, Pass& p, const std::vector<int32_t>& rows_new, bool first) {
    cudaStream_t st = c.s_main;
    const int n_new = int(rows_new.size());
    if (!first) {
        if (rows_new == p.rows_h) return;
        std::vector<int32_t> idx(n_new);
        size_t j = 0;
        for (int i = 0; i < n_new; ++i) {
            while (j < p.rows_h.size() && p.rows_h[j] != rows_new[i]) ++j;
            if (j == p.rows_h.size()) raise(KEEP_ERR_PLAN, "internal: row set grew");
            idx[i] = int32_t(j);
        }
        upload(p.d_idx, idx, st);
        ProfScope ps(c.prof, KEEP_PROF_COMPACT, st, 0.0, double(n_new) * c.d * (8.0 + (c.fast ? 2.0 : 0.0)));
        ensure_headroom(p.x_alt, sizeof(float) * size_t(std::max(n_new, 1) + c.G) * c.d);
        launch_gather_rows(p.x.as<float>(), p.d_idx.as<int32_t>(), n_new, c.d, p.x_alt.as<float>(),
                           c.fast ? p.xb.as<__nv_bfloat16>() : nullptr, st);
        std::swap(p.x.p, p.x_alt.p);
        std::swap(p.x.bytes, p.x_alt.bytes);
    }
    p.rows_h = rows_new;
    p.n = n_new;
    upload(p.d_rows, p.rows_h, st);
}

// The layout side of a pass: segment offsets, key -> segment map and the
// attention's per-chunk segment tables (no rows, no hidden states).
void pass_layout(Context& c, Pass& p, const std::vector<int32_t>& seg_len, int qlen) {
    p.S = int(seg_len.size());
    p.seg_len = seg_len;
    p.split_key = -1;  // new layout: re-plan the attention splits
    p.seg_start.assign(p.S, 0);
    int pos = 0;
    for (int i = 0; i < p.S; ++i) {
        p.seg_start[i] = pos;
        pos += seg_len[i];
    }
    p.Tm = pos;
    p.qlen = qlen;
    p.T = pos + qlen;
    p.row_seg.assign(p.T, -1);
    for (int i = 0; i < p.S; ++i)
        for (int t = 0; t < seg_len[i]; ++t) p.row_seg[p.seg_start[i] + t] = i;
    cudaStream_t st = c.s_main;
    upload(p.d_row_seg, p.row_seg, st);
    upload(p.d_seg_len, p.seg_len, st);
    upload(p.d_seg_start, p.seg_start, st);
    if (use_tc_attention(c)) {
        p.chunk_tab.ensure(32 * size_t(std::max<int64_t>(1, ceil_div(p.T, 128))));
        launch_chunk_table(p.d_row_seg.as<int32_t>(), p.T, p.chunk_tab.p, st);
        p.nb = summary_bins_width(p.row_seg);
        if (p.nb > 0 && bins_on_tensor_core()) {
            p.zt.ensure(2 * size_t(ceil_div(p.T, 128)) * p.nb * 128);
            launch_zt_build(p.d_row_seg.as<int32_t>(), p.T, p.chunk_tab.p, p.nb, p.zt.p, st);
        }
    }
}

void check_tokens(const Context& c, const int32_t* t, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (t[i] < 0 || t[i] >= c.V) raise(KEEP_ERR_INPUT, "token " + std::to_string(t[i]) + " out of vocab range");
}

// Build a pass over a token sequence.  seg_len partitions the memory rows;
// query rows follow.
void pass_init(Context& c, Pass& p, const std::vector<int32_t>& seg_len, const int32_t* tokens,
               const int32_t* query, int qlen) {
    pass_layout(c, p, seg_len, qlen);
    std::vector<int32_t> toks(p.T);
    std::copy(tokens, tokens + p.Tm, toks.begin());
    for (int k = 0; k < qlen; ++k) toks[p.Tm + k] = query[k];
    check_tokens(c, toks.data(), p.T);
    cudaStream_t st = c.s_main;
    upload(p.d_tokens, toks, st);
    std::vector<int32_t> all(p.T);
    std::iota(all.begin(), all.end(), 0);
    // (+G rows: the sharded all-gather moves G equal row blocks)
    // (x and x_alt swap at every compaction: both sized for every row)
    ensure_headroom(p.x, sizeof(float) * size_t(std::max(p.T, 1) + c.G) * c.d);
    ensure_headroom(p.x_alt, sizeof(float) * size_t(std::max(p.T, 1) + c.G) * c.d);
    if (c.fast) ensure_headroom(p.xb, 2 * size_t(std::max(p.T, 1) + c.G) * c.d);
    set_rows(c, p, all, true);
    ProfScope ps(c.prof, KEEP_PROF_EMBED, st, 0.0, double(p.T) * c.d * (8.0 + (c.fast ? 2.0 : 0.0)), c.fast ? 2 : 1);
    launch_embed(c.embed.as<float>(), p.d_tokens.as<int32_t>(), p.d_rows.as<int32_t>(), p.T, c.d,
                 p.x.as<float>(), st);
    if (c.fast) launch_to_bf16(p.x.as<float>(), int64_t(p.T) * c.d, p.xb.as<__nv_bfloat16>(), st);
    p.prev.assign(p.S, 1);
    p.dropped.assign(p.S, 0);
    p.layer = 0;
}

// ------------------------------------------------------------------ cursor --
template <class AfterSummary>
void cursor_layer(Context& c, const uint8_t* active, AfterSummary&& after_summary) {
    Pass& p = *c.pf;
    const int S = p.S, l = p.layer;
    if (l >= c.L) raise(KEEP_ERR_PLAN, "stepped past last layer");  // prefill.hpp:227
    for (int i = 0; i < S; ++i)
        if (active[i] && !p.prev[i]) raise(KEEP_ERR_PLAN, "plan is not monotone across layers");
    if (c.seg_gen != c.store_gen) resolve_segments(c, S);  // the store changed mid-prefill
    // all-reused layer over an in-order arena: run it on the arena sheets
    // (the cached rows are already in place; only the query rows -- in the
    // arena's spare rows -- are written), no merged-KV copy
    bool any_active = false;
    for (int i = 0; i < S && !any_active; ++i) any_active = active[i] != 0;
    bool alias_l = c.alias_arena != nullptr && !any_active;
    for (int i = 0; i < S && alias_l; ++i) alias_l = seg_block_current(c, i, l) != nullptr;
    if (alias_l) {
        const int64_t sheet = c.alias_arena->rows * int64_t(c.dl) * c.elem;
        p.kdst[l] = static_cast<uint8_t*>(c.alias_arena->buf.p) + size_t(l) * 2 * sheet;
        p.vdst[l] = static_cast<uint8_t*>(p.kdst[l]) + sheet;
    }
    // cached rows of this layer (prefill.hpp:255-263, 340-350): resolve first
    std::vector<void*> ks, vs;
    std::vector<int32_t> dr, nr, rope;
    int maxr = 0;
    for (int i = 0; i < S; ++i) {
        if (active[i] || loader_covers(c, i, l) || alias_l) continue;  // host-tier owners: K10 loader
        const OwnerKey& ok = c.seg_owner[i];
        const Payload* pl = seg_block_current(c, i, l);
        if (!pl) {
            c.stats.cache_misses++;
            raise(KEEP_ERR_CACHE_MISS, "missing cached KV for segment " + std::to_string(i) + " (owner " +
                                           owner_str(ok) + ") layer " + std::to_string(l));
        }
        if (c.seg_owner_row[i] + p.seg_len[i] > pl->tokens)
            raise(KEEP_ERR_INPUT, "cached block of " + owner_str(ok) + " is shorter than its members");
        ks.push_back(layer_keys(c, *pl, l) + c.seg_owner_row[i] * c.dl * c.elem);
        vs.push_back(layer_values(c, *pl, l) + c.seg_owner_row[i] * c.dl * c.elem);
        if (c.rope_theta > 0.0) {  // re-shift: owner-local rows -> layout rows
            rope.push_back(p.seg_start[i]);
            rope.push_back(p.seg_len[i]);
            rope.push_back(int32_t(p.seg_start[i] - c.seg_owner_row[i]));
        }
        dr.push_back(p.seg_start[i]);
        nr.push_back(p.seg_len[i]);
        maxr = std::max(maxr, p.seg_len[i]);
    }
    // newly dropped rows leave the compact set for good (prefill.hpp:233-239)
    std::vector<int32_t> rows_new;
    rows_new.reserve(p.n);
    for (int32_t r : p.rows_h) {
        const int sg = p.row_seg[r];
        if (sg < 0 || active[sg]) rows_new.push_back(r);
    }
    for (int i = 0; i < S; ++i)
        if (!active[i]) p.dropped[i] = 1;
    set_rows(c, p, rows_new, false);
    cudaStream_t st = c.s_main;
    loader_before_layer(c, p, l, active);  // pinned-host owners (K10): urgent loads + D1 wait
    if (!ks.empty()) {
        double rows_copied = 0.0;
        for (int32_t r : nr) rows_copied += r;
        ProfScope ps(c.prof, KEEP_PROF_CACHED, st, 0.0, rows_copied * c.dl * c.elem * 4.0);
        const void* const* kp;
        const void* const* vp;
        const int32_t *dp, *np;
        upload_copy_args(c, ks, vs, dr, nr, st, &kp, &vp, &dp, &np);
        launch_copy_cached(kp, vp, dp, np, int(ks.size()), int64_t(c.dl) * c.elem, p.kdst[l], p.vdst[l], maxr, st);
        if (!rope.empty()) {
            upload(p.rope_tab, rope, st);
            launch_rope_shift(p.kdst[l], p.rope_tab.as<int32_t>(), int(rope.size() / 3), maxr, c.dl, c.dh, c.rope_theta,
                              c.fast, st);
        }
    }
    p.with_summary = p.summary_wanted;
    if (p.n == 0) {  // no computed rows: the summary is all zero
        p.summ.ensure(sizeof(double) * (size_t(S) + size_t(S) * S));
        KEEP_CUDA(cudaMemsetAsync(p.summ.p, 0, sizeof(double) * (size_t(S) + size_t(S) * S), st));
        after_summary();
    } else {
        run_layer(c, p, l, after_summary);
    }
    loader_after_layer(c, p, l, active, layer_estimate_ms(c, p));
    std::copy(active, active + S, p.prev.begin());
    p.layer++;
}

void cursor_layer(Context& c, const uint8_t* active) {
    cursor_layer(c, active, [] {});
}

// Owners of the cached KV of each layout segment (units = static groups or
// dynamic segments, prefill.hpp:41-54); returns the segment lengths.
std::vector<int32_t> bind_owners(Context& c, const keep_layout* lay) {
    need_weights(c);
    if (!lay || lay->num_segments < 1) raise(KEEP_ERR_INPUT, "layout is empty");  // prefill.hpp:177
    const int S = lay->num_segments;
    std::vector<int32_t> sl(lay->seg_len, lay->seg_len + S);
    for (int x : sl)
        if (x < 1) raise(KEEP_ERR_INPUT, "empty segment in layout");
    c.seg_owner.assign(S, OwnerKey{KEEP_OWNER_SEGMENT, 0});
    c.seg_owner_row.assign(S, 0);
    if (lay->num_units == 0) {
        for (int i = 0; i < S; ++i) c.seg_owner[i] = OwnerKey{KEEP_OWNER_SEGMENT, uint32_t(i)};
    } else {
        std::vector<int> covered(S, 0);
        for (int u = 0; u < lay->num_units; ++u) {
            const int b = lay->unit_begin[u], e = lay->unit_end[u];
            if (b < 0 || e > S || b >= e) raise(KEEP_ERR_INPUT, "bad unit range");
            int64_t off = 0;
            for (int i = b; i < e; ++i) {
                c.seg_owner[i] = OwnerKey{lay->unit_owner[u].kind, lay->unit_owner[u].id};
                c.seg_owner_row[i] = off;
                off += sl[i];
                covered[i]++;
            }
        }
        for (int i = 0; i < S; ++i)
            if (covered[i] != 1) raise(KEEP_ERR_INPUT, "units must partition the layout");
    }
    resolve_segments(c, S);
    return sl;
}

// Is the layout one HBM arena in order, with spare rows for the query?  Then
// all-reused layers run on the arena sheets (no merged-KV copy).
// The arena of `tier` that holds every layout segment at its layout row, or null.
Arena* in_order_arena(Context& c, const std::vector<int32_t>& seg_start, int tier) {
    Arena* ar = nullptr;
    for (size_t i = 0; i < seg_start.size(); ++i) {
        auto it = c.store.find(c.seg_owner[i]);
        if (it == c.store.end() || it->second.arena->tier != tier) return nullptr;
        if (!ar) ar = it->second.arena.get();
        if (it->second.arena.get() != ar || it->second.row0 + c.seg_owner_row[i] != seg_start[i]) return nullptr;
    }
    return ar;
}

// Aliasing writes the query's K/V into arena rows [Tm, T): only safe when the
// layout covers the arena's whole payload extent (Tm == used), so those rows
// are the spare pad and no other owner's cached KV lives there.
void detect_alias(Context& c, const std::vector<int32_t>& seg_start, int Tm, int T) {
    c.alias_arena = nullptr;
    c.alias_hold.reset();
    if (c.rope_theta > 0.0) return;  // arena rows hold owner-local positions; the merged KV needs re-shifted keys
    Arena* ar = in_order_arena(c, seg_start, KEEP_TIER_DEVICE);
    if (ar && ar->used == Tm && ar->rows >= T) {
        c.alias_arena = ar;
        c.alias_hold = c.store.find(c.seg_owner[0])->second.arena;  // kept alive for the prefill
    }
}

void cursor_begin(Context& c, const keep_layout* lay, const int32_t* query, int qlen) {
    if (qlen < 0) raise(KEEP_ERR_INPUT, "negative query length");
    const std::vector<int32_t> sl = bind_owners(c, lay);
    // the workspace persists across prefills: buffers only grow (no per-step
    // cudaMalloc / cudaFree on the TTFT path)
    if (!c.pf) c.pf.reset(new Pass());
    Pass& p = *c.pf;
    p.block_diag = false;
    p.summary_global = true;
    p.summary_wanted = true;
    p.key_lo_h.clear();
    pass_init(c, p, sl, lay->tokens, query, qlen);
    const size_t sheet = size_t(p.T) * c.dl * c.elem;
    c.kv.ensure(std::max<size_t>(size_t(c.L) * 2 * sheet, 16));
    p.kdst.resize(c.L);
    p.vdst.resize(c.L);
    for (int l = 0; l < c.L; ++l) {
        p.kdst[l] = static_cast<uint8_t*>(c.kv.p) + size_t(l) * 2 * sheet;
        p.vdst[l] = static_cast<uint8_t*>(c.kv.p) + (size_t(l) * 2 + 1) * sheet;
    }
    detect_alias(c, p.seg_start, p.Tm, p.T);
    loader_begin(c, p);
    if (c.rope_theta > 0.0 && c.loader.on && c.loader.any_host)
        raise(KEEP_ERR_CONFIG, "the RoPE hook re-shifts HBM-resident blocks only (memory in pinned host DRAM)");
}

// Row T-1 of the final hidden state (device pointer or nullptr if dropped).
const float* last_row_ptr(const Context& c, const Pass& p) {
    if (p.n > 0 && p.rows_h.back() == p.T - 1) return p.x.as<float>() + int64_t(p.n - 1) * c.d;
    return nullptr;
}

void cursor_finish(Context& c, float* final_hidden, float* kv_out) {
    Pass& p = *c.pf;
    if (p.layer != c.L) raise(KEEP_ERR_PLAN, "cursor finished before the last layer");
    KEEP_CUDA(cudaStreamSynchronize(c.s_main));
    const int d = c.d;
    if (final_hidden) {
        std::memset(final_hidden, 0, sizeof(float) * size_t(p.T) * d);
        std::vector<float> xc(size_t(p.n) * d);
        if (p.n) KEEP_CUDA(cudaMemcpy(xc.data(), p.x.p, sizeof(float) * xc.size(), cudaMemcpyDeviceToHost));
        for (int i = 0; i < p.n; ++i)
            std::memcpy(final_hidden + size_t(p.rows_h[i]) * d, xc.data() + size_t(i) * d, sizeof(float) * d);
    }
    if (kv_out) {
        // per layer and K / V: the merged buffer or an aliased arena sheet
        const size_t nel = size_t(p.T) * c.dl;
        std::vector<uint16_t> tmp(c.fast ? nel : 0);
        for (int l = 0; l < c.L; ++l)
            for (int kv = 0; kv < 2; ++kv) {
                const void* src = kv ? p.vdst[l] : p.kdst[l];
                float* dst = kv_out + (size_t(l) * 2 + kv) * nel;
                if (!c.fast) {
                    KEEP_CUDA(cudaMemcpy(dst, src, sizeof(float) * nel, cudaMemcpyDeviceToHost));
                } else {
                    KEEP_CUDA(cudaMemcpy(tmp.data(), src, 2 * nel, cudaMemcpyDeviceToHost));
                    for (size_t i = 0; i < nel; ++i) dst[i] = bf2f(tmp[i]);
                }
            }
    }
}

// rows [0, n) of every layer sheet of a device arena (src_rows rows per sheet)
// -> rows [row0, row0 + n) of an arena, host part or its HBM-resident part
void place_rows(Context& c, Arena& dst, int64_t row0, const uint8_t* src, int64_t src_rows, int64_t n) {
    const size_t rowb = size_t(c.dl) * c.elem;
    const size_t ssheet = size_t(src_rows) * rowb, dsheet = size_t(dst.rows) * rowb;
    for (int l = 0; l < c.L; ++l)
        for (int kv = 0; kv < 2; ++kv) {
            uint8_t* d = l >= dst.mirror_from
                             ? static_cast<uint8_t*>(dst.mirror.p) + (size_t(l - dst.mirror_from) * 2 + kv) * dsheet
                             : static_cast<uint8_t*>(dst.buf.p) + (size_t(l) * 2 + kv) * dsheet;
            KEEP_CUDA(cudaMemcpyAsync(d + row0 * rowb, src + (size_t(l) * 2 + kv) * ssheet, size_t(n) * rowb,
                                      cudaMemcpyDefault, c.s_main));
        }
}

// --------------------------------------------------- canonical KV refresh --
// compute_and_put (harness.hpp:512-532) for a batch of owners: one pass over
// all their rows with block-diagonal attention (each owner is its own causal
// context: segment_prefill for a segment, joint full_prefill for a group).
void memory_compute_batch(Context& c, int n_owners, const keep_owner* owners, const uint64_t* versions,
                          const int32_t* owner_members, const int32_t* member_len, const int32_t* tokens,
                          int tier) {
    need_weights(c);
    ++c.store_gen;
    if (n_owners < 1) return;
    if (tier != KEEP_TIER_DEVICE && tier != KEEP_TIER_HOST) raise(KEEP_ERR_CONFIG, "unknown tier");
    std::vector<int32_t> seglen;  // one "segment" per owner (the owner's rows)
    std::vector<int64_t> row0(n_owners);
    int mi = 0;
    int64_t rows = 0;
    for (int o = 0; o < n_owners; ++o) {
        if (owner_members[o] < 1) raise(KEEP_ERR_INPUT, "owner without members");
        if (owners[o].kind == KEEP_OWNER_SEGMENT && owner_members[o] != 1)
            raise(KEEP_ERR_INPUT, "a segment owner has exactly one member");
        int32_t tot = 0;
        for (int k = 0; k < owner_members[o]; ++k, ++mi) {
            if (member_len[mi] < 1) raise(KEEP_ERR_INPUT, "segment is empty");
            tot += member_len[mi];
        }
        row0[o] = rows;
        rows += tot;
        seglen.push_back(tot);
    }
    // A new pinned-host memory larger than a quarter of the free HBM (BASELINE
    // configs[4]: 128K tokens, 172 GB of bf16 canonical KV) is computed in
    // owner chunks: each chunk on the device, then placed into one in-order
    // host arena (its HBM-resident layers, under keep_memory_residency's
    // budget, go to the arena's HBM part).
    if (tier == KEEP_TIER_HOST) {
        bool fresh = true;
        for (int o = 0; o < n_owners && fresh; ++o) fresh = !c.store.count(OwnerKey{owners[o].kind, owners[o].id});
        const size_t per_row = size_t(c.L) * 2 * c.dl * c.elem;
        size_t fr = 0, tot = 0;
        KEEP_CUDA(cudaMemGetInfo(&fr, &tot));
        int64_t chunk_rows = int64_t(std::max<size_t>(8192, fr / 4 / per_row));
        if (const char* e = std::getenv("KEEP_HOST_CHUNK_ROWS")) chunk_rows = std::max(1, std::atoi(e));  // tests
        if (fresh && rows + kArenaPad > chunk_rows && n_owners > 1) {
            auto arena = make_arena(c, rows + kArenaPad, KEEP_TIER_HOST);
            arena->used = rows;
            std::vector<int64_t> mo(n_owners + 1, 0), to(n_owners + 1, 0);
            for (int o = 0; o < n_owners; ++o) {
                mo[o + 1] = mo[o] + owner_members[o];
                to[o + 1] = to[o] + seglen[o];
            }
            for (int o0 = 0; o0 < n_owners;) {
                int o1 = o0 + 1;
                while (o1 < n_owners && to[o1 + 1] - to[o0] <= chunk_rows) ++o1;
                memory_compute_batch(c, o1 - o0, owners + o0, versions + o0, owner_members + o0, member_len + mo[o0],
                                     tokens + to[o0], KEEP_TIER_DEVICE);
                const Payload& first = c.store.at(OwnerKey{owners[o0].kind, owners[o0].id});
                place_rows(c, *arena, to[o0], static_cast<const uint8_t*>(first.arena->buf.p), first.arena->rows,
                           to[o1] - to[o0]);
                KEEP_CUDA(cudaStreamSynchronize(c.s_main));
                for (int o = o0; o < o1; ++o) {
                    Payload& pl = c.store.at(OwnerKey{owners[o].kind, owners[o].id});
                    pl.arena = arena;
                    pl.row0 = to[o];
                }
                o0 = o1;
            }
            c.refresh_ws.release();
            c.refresh.reset();  // the chunk pass's row buffers: the memory is built, HBM goes back to the queries
            return;
        }
    }
    if (rows > INT32_MAX / 2) raise(KEEP_ERR_CONFIG, "refresh batch too large");
    if (!c.refresh) c.refresh.reset(new Pass());
    Pass& p = *c.refresh;
    p.block_diag = true;
    p.with_summary = false;
    pass_init(c, p, seglen, tokens, nullptr, 0);
    p.key_lo_h.resize(p.T);
    for (int o = 0; o < n_owners; ++o)
        for (int t = 0; t < seglen[o]; ++t) p.key_lo_h[row0[o] + t] = int32_t(row0[o]);
    upload(p.d_key_lo, p.key_lo_h, c.s_main);
    // In place (an update of owners that already have a block of the same
    // size in this tier): compute into the grow-only refresh workspace and
    // copy every block into its slot -- no allocation on the query path
    // (harness.hpp:609-628 refreshes invalidated owners before each query).
    bool in_place = true;
    for (int o = 0; o < n_owners && in_place; ++o) {
        auto it = c.store.find(OwnerKey{owners[o].kind, owners[o].id});
        in_place = it != c.store.end() && it->second.tokens == seglen[o] && it->second.arena->tier == tier;
    }
    std::shared_ptr<Arena> dev;
    uint8_t* base = nullptr;
    // new arenas carry kArenaPad spare rows per layer sheet: a prefill whose
    // layout is the arena in order can run its all-reused layers directly on
    // the arena sheets, writing only the query rows into the spare rows
    const int64_t arows = in_place ? rows : rows + kArenaPad;
    const size_t sheet = size_t(arows) * c.dl * c.elem;
    if (in_place) {
        ensure_headroom(c.refresh_ws, size_t(c.L) * 2 * sheet);
        base = static_cast<uint8_t*>(c.refresh_ws.p);
    } else {
        dev = make_arena(c, arows, KEEP_TIER_DEVICE);
        dev->used = rows;
        base = static_cast<uint8_t*>(dev->buf.p);
    }
    p.kdst.resize(c.L);
    p.vdst.resize(c.L);
    for (int l = 0; l < c.L; ++l) {
        p.kdst[l] = base + size_t(l) * 2 * sheet;
        p.vdst[l] = base + (size_t(l) * 2 + 1) * sheet;
    }
    for (int l = 0; l < c.L; ++l) run_layer(c, p, l);
    if (in_place) {
        std::vector<void*> dsts, srcs;
        std::vector<size_t> sizes;
        for (int o = 0; o < n_owners; ++o) {
            const Payload& old = c.store[OwnerKey{owners[o].kind, owners[o].id}];
            drop_mirror(*old.arena);
            const size_t blk = size_t(seglen[o]) * c.dl * c.elem;
            for (int l = 0; l < c.L; ++l) {
                dsts.push_back(layer_keys(c, old, l));
                srcs.push_back(static_cast<uint8_t*>(p.kdst[l]) + size_t(row0[o]) * c.dl * c.elem);
                sizes.push_back(blk);
                dsts.push_back(layer_values(c, old, l));
                srcs.push_back(static_cast<uint8_t*>(p.vdst[l]) + size_t(row0[o]) * c.dl * c.elem);
                sizes.push_back(blk);
            }
        }
        if (tier == KEEP_TIER_DEVICE && (c.dl * c.elem) % 16 == 0) {
            // one gather/scatter kernel (copy-engine batches of ~10^4 small
            // blocks cost ~100x more at C3)
            std::vector<int64_t> nb(sizes.begin(), sizes.end());
            upload(c.d_ksrc, srcs, c.s_main);
            upload(c.d_vsrc, dsts, c.s_main);
            upload(c.d_bytes, nb, c.s_main);
            launch_batch_copy(c.d_ksrc.as<const void*>(), c.d_vsrc.as<void*>(), c.d_bytes.as<int64_t>(), int(dsts.size()),
                              c.s_main);
        } else {
            // host tier (or rows not 16-byte aligned): one async copy per block
            for (size_t k = 0; k < dsts.size(); ++k)
                KEEP_CUDA(cudaMemcpyAsync(dsts[k], srcs[k], sizes[k], cudaMemcpyDefault, c.s_main));
        }
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
        for (int o = 0; o < n_owners; ++o) {
            const OwnerKey k{owners[o].kind, owners[o].id};
            auto& cur = c.current_version[k];
            cur = std::max(cur, versions[o]);
            Payload& pl = c.store[k];
            pl.layer_version.assign(c.L, versions[o]);
            pl.present.assign(c.L, 1);
        }
        return;
    }
    std::shared_ptr<Arena> arena = dev;
    if (tier == KEEP_TIER_HOST) {
        arena = make_arena(c, arows, KEEP_TIER_HOST);
        arena->used = rows;
        place_rows(c, *arena, 0, static_cast<const uint8_t*>(dev->buf.p), arows, arows);
    }
    KEEP_CUDA(cudaStreamSynchronize(c.s_main));
    for (int o = 0; o < n_owners; ++o) {
        const OwnerKey k{owners[o].kind, owners[o].id};
        auto& cur = c.current_version[k];
        cur = std::max(cur, versions[o]);
        Payload pl;
        pl.arena = arena;
        pl.row0 = row0[o];
        pl.tokens = seglen[o];
        pl.layer_version.assign(c.L, versions[o]);
        pl.present.assign(c.L, 1);
        c.store[k] = std::move(pl);
    }
}

// ------------------------------------------------ batched multi-query prefill --
// plan_keep (recompute.hpp:140-180) for B queries over one memory layout
// (SURVEY.md 8(f2)).  Every instance gets exactly the plan, walk and rows a
// lone plan_keep would: the rows of instance b are computed with the same
// arithmetic (row-local projections, attention against the instance's own
// merged KV), only scheduled together:
//   - layer 0: every segment is in every plan and memory rows precede the
//     query, so the memory rows are computed once (instance 0); the other
//     instances compute their query rows against instance 0's layer-0 keys
//     and copy its segment-to-segment summary; at layer 1 their memory rows
//     start from instance 0's hidden states;
//   - the projections (QKV, Wo, MLP) run once per layer over the rows of all
//     instances (each weight streamed once for the batch);
//   - attention runs per instance; an instance with no active segment at a
//     layer reads the in-order arena in place (its query rows copied into the
//     arena's spare rows just before), so all-reused layers copy nothing;
//   - the walks of all instances run on the selector stream behind Wo + MLP;
//   - the first-token logits of the batch stream the unembedding once.
// With `plans` ([B][L][S], selective_prefill for each query, prefill.hpp:
// 478-497) the given monotone plans replace the walks.
void plan_keep_batch(Context& c, const keep_layout* lay, int B, const int32_t* queries, int qlen, const double* sched,
                     bool multihop, keep_plan_result* outs, const uint8_t* plans = nullptr) {
    if (B < 1) raise(KEEP_ERR_CONFIG, "batch needs at least one query");
    if (qlen < 1) raise(KEEP_ERR_INPUT, "batched prefill needs query tokens");
    if (c.G > 1) raise(KEEP_ERR_CONFIG, "batched prefill runs on one GPU (G = 1)");
    if (c.fast && small_n_threshold() > 0) raise(KEEP_ERR_CONFIG, "batched prefill needs KEEP_ATTN_SMALL_N=0");
    cudaStream_t st = c.s_main;
    const int L = c.L, d = c.d, dl = c.dl;
    const size_t es = c.fast ? 2 : 4;
    if (c.pk_evs.size() != size_t(L + 1)) {
        for (auto e : c.pk_evs) cudaEventDestroy(e);
        c.pk_evs.assign(L + 1, nullptr);
        for (auto& e : c.pk_evs) KEEP_CUDA(cudaEventCreate(&e));
    }
    if (!c.ev_sum) {
        KEEP_CUDA(cudaEventCreateWithFlags(&c.ev_sum, cudaEventDisableTiming));
        KEEP_CUDA(cudaEventCreateWithFlags(&c.ev_sel, cudaEventDisableTiming));
    }
    std::vector<cudaEvent_t>& evs = c.pk_evs;
    KEEP_CUDA(cudaEventRecord(evs[0], st));
    const std::vector<int32_t> sl = bind_owners(c, lay);
    const int S = int(sl.size());
    bool any_host = false;
    for (int i = 0; i < S; ++i) {
        auto it = c.store.find(c.seg_owner[i]);
        any_host = any_host || (it != c.store.end() && it->second.arena->tier != KEEP_TIER_DEVICE);
    }
    if (!c.batch) c.batch.reset(new Batch());
    Batch& bt = *c.batch;
    if (int(bt.views.size()) < B) bt.views.resize(B);
    for (int b = 0; b < B; ++b) {
        if (!bt.views[b]) bt.views[b].reset(new Pass());
        Pass& v = *bt.views[b];
        v.block_diag = false;
        v.key_lo_h.clear();
        v.rows_h.clear();
        pass_layout(c, v, sl, qlen);
    }
    const Pass& v0 = *bt.views[0];
    const int Tm = v0.Tm, T = v0.T;
    const int64_t Tp = ceil_div(T, 128) * 128;
    if (int64_t(B) * Tp > INT32_MAX / 4) raise(KEEP_ERR_CONFIG, "batch too large");
    check_tokens(c, lay->tokens, Tm);
    check_tokens(c, queries, int64_t(B) * qlen);
    detect_alias(c, v0.seg_start, Tm, T);
    // Memory in pinned host DRAM (BASELINE configs[4]): one in-order arena,
    // streamed a whole layer sheet at a time into two HBM staging sheets on
    // the copy stream, one layer ahead of compute -- every query of the batch
    // reads the same staged sheet, so each byte crosses PCIe once per layer
    // for the whole batch.  The staged sheet then serves exactly as the
    // in-order HBM arena does (cached-row source, aliased layers in place).
    Arena* host_ar = nullptr;
    if (any_host) {
        host_ar = in_order_arena(c, v0.seg_start, KEEP_TIER_HOST);
        if (!host_ar)
            raise(KEEP_ERR_CONFIG, "batched prefill over host memory needs the layout as one in-order pinned arena");
        if (qlen > kArenaPad) raise(KEEP_ERR_CONFIG, "query longer than the staging spare rows");
    }
    const size_t rowb = size_t(dl) * c.elem;
    const size_t ssheet = size_t(Tm + kArenaPad) * rowb;  // staged sheet: memory rows + spare rows
    // A ring of NS staged layers: the copy stream runs up to NS - 1 layers
    // ahead, so the loads of the cheap all-reused layers at the end overlap the
    // recompute-heavy layers before them (layer-balanced loading,
    // pipeline_sim.hpp:261-338, with whole layers as the unit).
    int NS = 0;
    std::vector<uint8_t*> stage;
    if (host_ar) {
        size_t free_b = 0, total_b = 0;
        KEEP_CUDA(cudaMemGetInfo(&free_b, &total_b));
        // (at most a quarter of the free HBM and a sixth of the device: the pass
        // needs the rest; no deeper than the layers that live in host DRAM)
        const size_t have = bt.stage.bytes + std::min(free_b / 4, total_b / 6);
        const int host_layers = std::max(1, std::min(host_ar->mirror_from, L) - 1);
        NS = int(std::max<size_t>(2, std::min<size_t>(size_t(host_layers), have / (2 * ssheet))));
        bt.stage.ensure(size_t(NS) * 2 * ssheet);
        for (int k = 0; k < NS; ++k) stage.push_back(static_cast<uint8_t*>(bt.stage.p) + size_t(k) * 2 * ssheet);
        for (size_t k = bt.ev_load.size(); k < size_t(NS); ++k) {
            cudaEvent_t a = nullptr, u = nullptr;
            KEEP_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            KEEP_CUDA(cudaEventCreateWithFlags(&u, cudaEventDisableTiming));
            bt.ev_load.push_back(a);
            bt.ev_used.push_back(u);
        }
        for (int k = 0; k < NS; ++k) KEEP_CUDA(cudaEventRecord(bt.ev_used[k], st));  // slots free from here
    }
    // a layer resident in HBM (keep_memory_residency) is read in place: no load
    const int res_from = host_ar ? std::min(host_ar->mirror_from, L) : L;
    auto sheet_of = [&](int l) -> uint8_t* {
        if (l >= res_from) return static_cast<uint8_t*>(host_ar->mirror.p) + size_t(l - res_from) * 2 * ssheet;
        return stage[l % NS];
    };
    auto load_sheet = [&](int l) {  // layer l's canonical K / V of every memory row -> stage[l % NS]
        if (l >= res_from) return;
        const int k = l % NS;
        uint8_t* dst = stage[k];
        const size_t asheet = size_t(host_ar->rows) * rowb;
        const uint8_t* src = static_cast<const uint8_t*>(host_ar->buf.p) + size_t(l) * 2 * asheet;
        KEEP_CUDA(cudaStreamWaitEvent(c.s_copy, bt.ev_used[k], 0));  // its readers of layer l - NS are done
        {
            ProfScope ps(c.prof, KEEP_PROF_LOADER, c.s_copy, 0.0, 2.0 * Tm * rowb, 2);
            KEEP_CUDA(cudaMemcpyAsync(dst, src, size_t(Tm) * rowb, cudaMemcpyHostToDevice, c.s_copy));
            KEEP_CUDA(cudaMemcpyAsync(dst + ssheet, src + asheet, size_t(Tm) * rowb, cudaMemcpyHostToDevice, c.s_copy));
        }
        KEEP_CUDA(cudaEventRecord(bt.ev_load[k], c.s_copy));
        c.stats.bytes_loaded_slow += 2ull * Tm * rowb;
    };
    // layer 0 recomputes every segment: loads start with layer 1
    for (int l = 1; host_ar && l < std::min(L, NS + 1); ++l) load_sheet(l);
    const size_t sheet = size_t(B) * Tp * rowb;
    bt.kv.ensure(2 * sheet);
    uint8_t* kvK = static_cast<uint8_t*>(bt.kv.p);
    uint8_t* kvV = kvK + sheet;
    Pass& P = bt.all;
    P.S = S;
    P.T = int(B * Tp);
    P.Tm = Tm;
    P.qlen = qlen;
    P.block_diag = false;
    P.with_summary = false;
    P.kdst.assign(L, kvK);
    P.vdst.assign(L, kvV);

    // layer 0 rows: instance 0 in full, the query rows of the others
    std::vector<int32_t> rows, toks;
    std::vector<int> off(B), nrow(B);
    for (int b = 0; b < B; ++b) {
        off[b] = int(rows.size());
        for (int t = (b == 0 ? 0 : Tm); t < T; ++t) {
            rows.push_back(int32_t(b * Tp + t));
            toks.push_back(t < Tm ? lay->tokens[t] : queries[size_t(b) * qlen + (t - Tm)]);
        }
        nrow[b] = int(rows.size()) - off[b];
    }
    const int n0 = int(rows.size());
    // Row buffers sized once for the whole pass (layer 1 is the widest after
    // layer 0: plans only shrink).  x and x_alt swap at every compaction, so a
    // grow-on-demand x_alt would reallocate -- and a cudaFree synchronises the
    // device, i.e. waits behind every layer load queued on the copy engines.
    int64_t max_rows = n0;
    {
        int64_t widest = 0;
        if (plans) {
            for (int l = 1; l < L; ++l) {
                int64_t r = 0;
                for (int b = 0; b < B; ++b)
                    for (int i = 0; i < S; ++i) r += plans[(size_t(b) * L + l) * S + i] ? sl[i] : 0;
                widest = std::max(widest, r + int64_t(B) * qlen);
            }
        } else if (L > 1) {
            const int64_t bud = keep_layer_budget(sched[1], S);
            std::vector<int32_t> len(sl);
            std::sort(len.begin(), len.end(), std::greater<int32_t>());
            int64_t r = 0;
            for (int64_t i = 0; i < std::min<int64_t>(bud, S); ++i) r += len[i];
            widest = int64_t(B) * (r + qlen);
        }
        max_rows = std::max(max_rows, widest);
    }
    P.x.ensure(sizeof(float) * size_t(max_rows) * d);
    P.x_alt.ensure(sizeof(float) * size_t(max_rows) * d);
    if (c.fast) P.xb.ensure(2 * size_t(max_rows) * d);
    upload(bt.tokens, toks, st);
    {
        std::vector<int32_t> iota(n0);
        std::iota(iota.begin(), iota.end(), 0);
        upload(bt.iota, iota, st);
    }
    {
        ProfScope ps(c.prof, KEEP_PROF_EMBED, st, 0.0, double(n0) * d * (8.0 + (c.fast ? 2.0 : 0.0)), c.fast ? 2 : 1);
        launch_embed(c.embed.as<float>(), bt.tokens.as<int32_t>(), bt.iota.as<int32_t>(), n0, d, P.x.as<float>(), st);
        if (c.fast) launch_to_bf16(P.x.as<float>(), int64_t(n0) * d, P.xb.as<__nv_bfloat16>(), st);
    }
    P.rows_h = rows;
    P.n = n0;
    upload(P.d_rows, P.rows_h, st);
    auto set_views = [&] {
        std::vector<int32_t> loc;
        for (int b = 0; b < B; ++b) {
            Pass& v = *bt.views[b];
            loc.resize(nrow[b]);
            for (int i = 0; i < nrow[b]; ++i) loc[i] = int32_t(P.rows_h[off[b] + i] - b * Tp);
            v.n = nrow[b];
            if (loc == v.rows_h) continue;
            v.rows_h = loc;
            upload(v.d_rows, v.rows_h, st);
        }
    };
    set_views();

    bt.sel_order.ensure(sizeof(int32_t) * size_t(B) * (S + 2));
    bt.sel_cand.ensure(size_t(B) * S);
    if (bt.walk_host.bytes < sizeof(int32_t) * size_t(B) * (S + 2) || !bt.walk_host.host)
        bt.walk_host.alloc(sizeof(int32_t) * size_t(B) * (S + 2), true);
    int32_t* hbuf = bt.walk_host.as<int32_t>();
    std::vector<std::vector<uint8_t>> active(B, std::vector<uint8_t>(S, 1));
    std::vector<uint8_t> candh(size_t(B) * S, 0);
    std::vector<int32_t> pos;

    for (int l = 0; l < L; ++l) {
        int64_t budget = 0;
        if (plans) {
            for (int b = 0; b < B; ++b) {
                const uint8_t* pl = plans + (size_t(b) * L + l) * S;
                for (int i = 0; i < S; ++i) {
                    if (pl[i] && !active[b][i]) raise(KEEP_ERR_PLAN, "plan is not monotone across layers");
                    active[b][i] = pl[i] ? 1 : 0;
                }
                if (l == 0 && std::count(active[b].begin(), active[b].end(), 1) != S)
                    raise(KEEP_ERR_PLAN, "a batched prefill computes every segment at layer 0");
            }
        } else if (l + 1 < L) {
            budget = keep_layer_budget(sched[l + 1], S);
        }
        std::vector<int64_t> live(B, 0);
        std::vector<char> walk(B, 0), wanted(B, 0);
        bool any_walk = false, any_wanted = false;
        for (int b = 0; b < B; ++b) {
            keep_plan_result* o = outs ? &outs[b] : nullptr;
            if (o && o->plan) std::copy(active[b].begin(), active[b].end(), o->plan + size_t(l) * S);
            if (o && o->order_len) o->order_len[l] = -1;
            if (o && o->hops) o->hops[l] = 0;
            for (uint8_t x : active[b]) live[b] += x;
            walk[b] = !plans && l + 1 < L && budget < live[b] && multihop;
            wanted[b] = walk[b] || (o && o->summaries) || (!plans && l + 1 < L && budget < live[b] && !multihop);
            any_walk = any_walk || walk[b];
            any_wanted = any_wanted || wanted[b];
        }
        if (l == 0) wanted[0] = any_wanted;  // the others take instance 0's segment rows
        if (l > 0) {
            // newly dropped rows leave for good (prefill.hpp:233-239); at layer 1
            // instances b > 0 take their memory rows from instance 0
            std::vector<int32_t> nr_rows;
            std::vector<int> noff(B), nn(B);
            for (int b = 0; b < B; ++b) {
                noff[b] = int(nr_rows.size());
                for (int i = 0; i < nrow[b]; ++i) {
                    const int32_t g = P.rows_h[off[b] + i];
                    const int t = int(g - b * Tp);
                    const int sg = v0.row_seg[t];
                    if (sg < 0 || active[b][sg]) nr_rows.push_back(g);
                }
                if (l == 1 && b > 0) {  // + the memory rows computed by instance 0
                    std::vector<int32_t> mem;
                    for (int t = 0; t < Tm; ++t)
                        if (active[b][v0.row_seg[t]]) mem.push_back(int32_t(b * Tp + t));
                    nr_rows.insert(nr_rows.begin() + noff[b], mem.begin(), mem.end());
                }
                nn[b] = int(nr_rows.size()) - noff[b];
            }
            if (nr_rows != P.rows_h) {
                pos.assign(size_t(B) * Tp, -1);
                for (int i = 0; i < P.n; ++i) pos[P.rows_h[i]] = i;
                std::vector<int32_t> idx(nr_rows.size());
                for (size_t i = 0; i < nr_rows.size(); ++i) {
                    int32_t j = pos[nr_rows[i]];
                    if (j < 0 && l == 1) j = pos[nr_rows[i] % Tp];  // instance 0's row of the same position
                    if (j < 0) raise(KEEP_ERR_PLAN, "internal: batched row set grew");
                    idx[i] = j;
                }
                const int n_new = int(nr_rows.size());
                upload(P.d_idx, idx, st);
                ProfScope ps(c.prof, KEEP_PROF_COMPACT, st, 0.0, double(n_new) * d * (8.0 + (c.fast ? 2.0 : 0.0)));
                P.x_alt.ensure(sizeof(float) * size_t(std::max(n_new, 1)) * d);
                if (c.fast) P.xb.ensure(2 * size_t(std::max(n_new, 1)) * d);
                launch_gather_rows(P.x.as<float>(), P.d_idx.as<int32_t>(), n_new, d, P.x_alt.as<float>(),
                                   c.fast ? P.xb.as<__nv_bfloat16>() : nullptr, st);
                std::swap(P.x.p, P.x_alt.p);
                std::swap(P.x.bytes, P.x_alt.bytes);
                P.rows_h = std::move(nr_rows);
                P.n = n_new;
                upload(P.d_rows, P.rows_h, st);
                off = noff;
                nrow = nn;
                set_views();
            }
        }
        // cached rows of this layer (prefill.hpp:255-263, 340-350) per
        // instance -- nothing for an all-reused instance over the arena
        std::vector<char> alias(B, 0);
        if (host_ar && l > 0 && l < res_from) KEEP_CUDA(cudaStreamWaitEvent(st, bt.ev_load[l % NS], 0));
        {
            std::vector<void*> ks, vs;
            std::vector<int32_t> dr, nrr;
            int maxr = 0;
            for (int b = 0; b < B && l > 0; ++b) {
                bool any_active = false;
                for (int i = 0; i < S && !any_active; ++i) any_active = active[b][i] != 0;
                bool al = (c.alias_arena != nullptr || host_ar != nullptr) && !any_active;
                for (int i = 0; i < S && al; ++i) al = seg_block_current(c, i, l) != nullptr;
                alias[b] = al;
                if (al) continue;
                for (int i = 0; i < S; ++i) {
                    if (active[b][i]) continue;
                    const Payload* pl = seg_block_current(c, i, l);
                    if (!pl) {
                        c.stats.cache_misses++;
                        raise(KEEP_ERR_CACHE_MISS, "missing cached KV for segment " + std::to_string(i) + " (owner " +
                                                       owner_str(c.seg_owner[i]) + ") layer " + std::to_string(l));
                    }
                    if (c.seg_owner_row[i] + sl[i] > pl->tokens)
                        raise(KEEP_ERR_INPUT, "cached block of " + owner_str(c.seg_owner[i]) + " is shorter than its members");
                    if (host_ar) {  // the staged sheet, in layout order
                        ks.push_back(sheet_of(l) + size_t(v0.seg_start[i]) * rowb);
                        vs.push_back(sheet_of(l) + ssheet + size_t(v0.seg_start[i]) * rowb);
                    } else {
                        ks.push_back(layer_keys(c, *pl, l) + c.seg_owner_row[i] * rowb);
                        vs.push_back(layer_values(c, *pl, l) + c.seg_owner_row[i] * rowb);
                    }
                    dr.push_back(int32_t(b * Tp + v0.seg_start[i]));
                    nrr.push_back(sl[i]);
                    maxr = std::max(maxr, sl[i]);
                }
            }
            if (!ks.empty()) {
                double rows_copied = 0.0;
                for (int32_t r : nrr) rows_copied += r;
                ProfScope ps(c.prof, KEEP_PROF_CACHED, st, 0.0, rows_copied * rowb * 4.0);
                const void* const* kp;
                const void* const* vp;
                const int32_t *dp, *np;
                upload_copy_args(c, ks, vs, dr, nrr, st, &kp, &vp, &dp, &np);
                launch_copy_cached(kp, vp, dp, np, int(ks.size()), int64_t(rowb), kvK, kvV, maxr, st);
            }
        }
        ensure_layer_scratch(c, P);
        layer_qkv(c, P, l);
        const size_t qbytes = size_t(qlen) * rowb;
        // all-reused queries (FAST, no summary read): one multi-query decode over
        // the shared sheet instead of one attention each (the sheet is read
        // once through L2 for all of them, and their query rows stay put)
        std::vector<char> multi(B, 0);
        int n_multi = 0;
        if (l > 0 && c.fast && c.dh == 128 && qlen <= 16 && batch_multi_decode()) {
            for (int b = 0; b < B; ++b)
                if (alias[b] && !wanted[b]) {
                    multi[b] = 1;
                    ++n_multi;
                }
            if (n_multi < 2) std::fill(multi.begin(), multi.end(), 0), n_multi = 0;
        }
        for (int b = 0; b < B; ++b) {
            if (multi[b]) continue;
            Pass& v = *bt.views[b];
            v.with_summary = wanted[b] != 0;
            const uint8_t* qb = static_cast<const uint8_t*>(P.q.p) + size_t(off[b]) * dl * es;
            uint8_t* cb = static_cast<uint8_t*>(c.fast ? P.ctxb.p : P.ctx.p) + size_t(off[b]) * dl * es;
            const uint8_t* kb = kvK + size_t(b) * Tp * rowb;
            const uint8_t* vb = kvV + size_t(b) * Tp * rowb;
            uint8_t* qk = nullptr;  // where this instance's query rows must be for its attention
            uint8_t* qv = nullptr;
            if (l == 0 && b > 0) {  // instance 0's layer-0 keys, this query's rows in place
                qk = kvK + size_t(Tm) * rowb;
                qv = kvV + size_t(Tm) * rowb;
                kb = kvK;
                vb = kvV;
            } else if (alias[b]) {  // the arena sheets of layer l, query rows in the spare rows
                const size_t asheet = host_ar ? ssheet : size_t(c.alias_arena->rows) * rowb;
                uint8_t* ak = host_ar ? sheet_of(l)
                                      : static_cast<uint8_t*>(c.alias_arena->buf.p) + size_t(l) * 2 * asheet;
                qk = ak + size_t(Tm) * rowb;
                qv = ak + asheet + size_t(Tm) * rowb;
                kb = ak;
                vb = ak + asheet;
            }
            if (qk) {
                ProfScope ps(c.prof, KEEP_PROF_CACHED, st, 0.0, 4.0 * double(qbytes), 1);
                launch_copy2(qk, kvK + (size_t(b) * Tp + Tm) * rowb, qv, kvV + (size_t(b) * Tp + Tm) * rowb, int64_t(qbytes),
                             st);
            }
            layer_attention(c, v, l, qb, cb, kb, vb);
            if (l == 0 && b > 0 && v.with_summary)
                KEEP_CUDA(cudaMemcpyAsync(v.summ.as<double>() + S, bt.views[0]->summ.as<double>() + S,
                                          sizeof(double) * size_t(S) * S, cudaMemcpyDeviceToDevice, st));
        }
        if (n_multi > 0) {
            const size_t asheet = host_ar ? ssheet : size_t(c.alias_arena->rows) * rowb;
            uint8_t* ak = host_ar ? sheet_of(l) : static_cast<uint8_t*>(c.alias_arena->buf.p) + size_t(l) * 2 * asheet;
            DecodeMulti dm;
            dm.H = c.Hl;
            dm.d = dl;
            dm.qlen = qlen;
            dm.kv_mem = Tm;
            dm.own_rows = int(B * Tp);
            dm.k_mem = ak;
            dm.v_mem = ak + asheet;
            dm.k_own = kvK;
            dm.v_own = kvV;
            dm.q = P.q.p;
            dm.ctx = P.ctxb.as<__nv_bfloat16>();
            int first = -1;
            for (int b = 0; b < B; ++b) {
                if (!multi[b]) continue;
                if (first < 0) first = b;
                bt.views[b]->with_summary = false;
                dm.qrow0.push_back(int(b * Tp + Tm));
                dm.qoff.push_back(off[b]);
            }
            dm.rows = bt.views[first]->d_rows.as<int32_t>();  // positions Tm.. (the same for every query)
            const double pairs = double(n_multi) * qlen * (Tm + (qlen + 1) / 2.0);
            ProfScope ps(c.prof, KEEP_PROF_DECODE, st, 4.0 * dl * pairs, 2.0 * rowb * (Tm + double(n_multi) * qlen), 1);
            ps.kernels = launch_attention_decode_multi(dm, st);
        }
        if (host_ar && l > 0) {  // this layer's slot is free once its attention has run
            KEEP_CUDA(cudaEventRecord(bt.ev_used[l % NS], st));
            if (l + NS < L) load_sheet(l + NS);
        }
        if (any_walk) {  // the walks for layer l+1 (one CTA each) overlap this layer's Wo + MLP
            std::vector<uint8_t> run(B, 0);
            std::vector<const double*> sp(B);
            for (int b = 0; b < B; ++b) {
                run[b] = walk[b] ? 1 : 0;
                sp[b] = bt.views[b]->summ.as<double>();
                if (walk[b]) std::copy(active[b].begin(), active[b].end(), candh.begin() + size_t(b) * S);
            }
            candh.resize(size_t(B) * S + B);
            std::copy(run.begin(), run.end(), candh.begin() + size_t(B) * S);
            bt.sel_cand.ensure(size_t(B) * S + B);
            upload_bytes(bt.sel_cand.p, candh.data(), size_t(B) * S + B, c.s_sel);
            upload(bt.sel_ptrs, sp, c.s_sel);
            KEEP_CUDA(cudaEventRecord(c.ev_sum, st));
            KEEP_CUDA(cudaStreamWaitEvent(c.s_sel, c.ev_sum, 0));
            {
                ProfScope ps(c.prof, KEEP_PROF_SELECT, c.s_sel, 0.0, 8.0 * double(S) * S * B);
                launch_select_batch(S, B, bt.sel_ptrs.as<const double*>(), budget, bt.sel_cand.as<uint8_t>(),
                                    bt.sel_cand.as<uint8_t>() + size_t(B) * S, bt.sel_order.as<int32_t>(), c.s_sel,
                                    c.cfg.max_hops);
            }
            KEEP_CUDA(cudaMemcpyAsync(hbuf, bt.sel_order.p, sizeof(int32_t) * size_t(B) * (S + 2), cudaMemcpyDeviceToHost,
                                      c.s_sel));
            KEEP_CUDA(cudaEventRecord(c.ev_sel, c.s_sel));
        }
        // (one SM per concurrent walk stays free of the GEMMs)
        c.gemm_ctas = any_walk ? kNumSMs - std::min<int>(int(std::count(walk.begin(), walk.end(), 1)), 32) : kNumSMs;
        layer_dense(c, P, l);
        c.gemm_ctas = kNumSMs;
        KEEP_CUDA(cudaEventRecord(evs[l + 1], st));
        for (int b = 0; b < B; ++b) {
            keep_plan_result* o = outs ? &outs[b] : nullptr;
            // N_act of the query's own plan (layer 0: every row, although the
            // batch computed the memory rows once)
            if (o && o->rows_per_layer) o->rows_per_layer[l] = l == 0 ? T : nrow[b];
            if (o && o->summaries)
                KEEP_CUDA(cudaMemcpyAsync(o->summaries + size_t(l) * (S + size_t(S) * S), bt.views[b]->summ.p,
                                          sizeof(double) * (S + size_t(S) * S), cudaMemcpyDeviceToHost, st));
        }
        if (l + 1 >= L) break;
        if (any_walk) KEEP_CUDA(cudaEventSynchronize(c.ev_sel));
        for (int b = 0; b < B && !plans; ++b) {
            if (budget >= live[b]) continue;  // recompute everything still live
            keep_plan_result* o = outs ? &outs[b] : nullptr;
            std::vector<uint8_t> next(S, 0);
            if (multihop) {
                const int32_t* h = hbuf + size_t(b) * (S + 2);
                for (int k = 0; k < h[0]; ++k) next[h[2 + k]] = 1;
                if (o && o->orders) std::copy(h + 2, h + 2 + h[0], o->orders + size_t(l) * S);
                if (o && o->order_len) o->order_len[l] = h[0];
                if (o && o->hops) o->hops[l] = h[1];
            } else {  // single-hop ablation (recompute.hpp:166-176): ranked on the device
                upload(c.d_live, active[b], st);
                c.d_next.ensure(size_t(S));
                launch_single_hop(bt.views[b]->summ.as<double>(), c.d_live.as<uint8_t>(), S, budget,
                                  c.d_next.as<uint8_t>(), st);
                KEEP_CUDA(cudaMemcpyAsync(next.data(), c.d_next.p, size_t(S), cudaMemcpyDeviceToHost, st));
                KEEP_CUDA(cudaStreamSynchronize(st));
            }
            active[b] = std::move(next);
        }
    }
    // first-token logits of every instance (model.hpp:76-85): the last row of
    // an instance is its last query row, never dropped
    std::vector<int32_t> last(B);
    for (int b = 0; b < B; ++b) last[b] = off[b] + nrow[b] - 1;
    upload(bt.last_idx, last, st);
    bt.last_x.ensure(sizeof(float) * size_t(B) * d);
    bt.logits.ensure(sizeof(double) * size_t(B) * c.V);
    {
        ProfScope ps(c.prof, KEEP_PROF_LOGITS, st, 2.0 * B * c.d * double(c.V), 4.0 * c.d * double(c.V));
        launch_gather_rows(P.x.as<float>(), bt.last_idx.as<int32_t>(), B, d, bt.last_x.as<float>(), nullptr, st);
        launch_logits_multi(bt.last_x.as<float>(), B, c.unembed.as<float>(), d, c.V, bt.logits.as<double>(), st);
    }
    KEEP_CUDA(cudaEventRecord(c.ev_b, st));
    for (int b = 0; b < B && outs; ++b)
        if (outs[b].last_logits)
            KEEP_CUDA(cudaMemcpyAsync(outs[b].last_logits, bt.logits.as<double>() + size_t(b) * c.V,
                                      sizeof(double) * c.V, cudaMemcpyDeviceToHost, st));
    KEEP_CUDA(cudaStreamSynchronize(st));
    if (!outs) return;
    float ms = 0.f;
    KEEP_CUDA(cudaEventElapsedTime(&ms, evs[0], c.ev_b));
    std::vector<double> lms(L, 0.0);
    for (int l = 0; l < L; ++l) {
        float m = 0.f;
        KEEP_CUDA(cudaEventElapsedTime(&m, evs[l], evs[l + 1]));
        lms[l] = m;
    }
    std::vector<float> xc;
    for (int b = 0; b < B; ++b) {
        keep_plan_result& o = outs[b];
        o.ttft_ms = ms;
        if (o.layer_ms) std::copy(lms.begin(), lms.end(), o.layer_ms);
        if (o.final_hidden) {  // finish (prefill.hpp:324-337): dropped rows are zero
            std::memset(o.final_hidden, 0, sizeof(float) * size_t(T) * d);
            xc.resize(size_t(nrow[b]) * d);
            KEEP_CUDA(cudaMemcpy(xc.data(), P.x.as<float>() + size_t(off[b]) * d, sizeof(float) * xc.size(),
                                 cudaMemcpyDeviceToHost));
            for (int i = 0; i < nrow[b]; ++i)
                std::memcpy(o.final_hidden + size_t(P.rows_h[off[b] + i] - b * Tp) * d, xc.data() + size_t(i) * d,
                            sizeof(float) * d);
        }
    }
}

}  // namespace

// =================================================================== C ABI ==
extern "C" {

const char* keep_last_error(void) { return g_err.c_str(); }
const char* keep_version(void) { return "keep_b200 0.1 (sm_100a)"; }

int keep_ctx_create(const keep_config* cfg, void** out) {
    return guard([&] {
        if (!cfg || !out) raise(KEEP_ERR_CONFIG, "null argument");
        check_cfg(*cfg);
        int ndev = 0;
        KEEP_CUDA(cudaGetDeviceCount(&ndev));
        if (cfg->device < 0 || cfg->device >= ndev) raise(KEEP_ERR_CONFIG, "no such CUDA device");
        KEEP_CUDA(cudaSetDevice(cfg->device));
        cudaDeviceProp prop{};
        KEEP_CUDA(cudaGetDeviceProperties(&prop, cfg->device));
        if (prop.major != 10) raise(KEEP_ERR_CONFIG, "keep_b200 requires an sm_100 (B200) device");
        std::unique_ptr<Context> c(new Context());
        c->cfg = *cfg;
        c->L = cfg->num_layers;
        c->H = cfg->num_heads;
        c->d = cfg->model_dim;
        c->dh = c->d / c->H;
        c->f = cfg->mlp_dim;
        c->V = cfg->vocab_size;
        c->fast = cfg->numerics == KEEP_NUMERICS_FAST;
        c->exact = cfg->numerics == KEEP_NUMERICS_PARITY_EXACT;
        c->elem = c->fast ? 2 : 4;
        c->G = cfg->world_size;
        c->R = cfg->rank;
        c->Hl = c->H / c->G;
        c->dl = c->Hl * c->dh;
        c->comm = make_comm(*cfg);
        KEEP_CUDA(cudaStreamCreateWithFlags(&c->s_main, cudaStreamNonBlocking));
        KEEP_CUDA(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
        KEEP_CUDA(cudaStreamCreateWithFlags(&c->s_sel, cudaStreamNonBlocking));
        KEEP_CUDA(cudaEventCreate(&c->ev_a));
        KEEP_CUDA(cudaEventCreate(&c->ev_b));
        *out = c.release();
    });
}

int keep_ctx_destroy(void* ctx) {
    return guard([&] {
        if (!ctx) return;
        Context* c = C(ctx);
        cudaDeviceSynchronize();
        c->pf.reset();
        c->refresh.reset();
        c->store.clear();
        c->comm.reset();
        for (auto e : c->pk_evs) cudaEventDestroy(e);
        if (c->ev_sum) cudaEventDestroy(c->ev_sum);
        if (c->ev_sel) cudaEventDestroy(c->ev_sel);
        cudaStreamDestroy(c->s_main);
        cudaStreamDestroy(c->s_copy);
        cudaStreamDestroy(c->s_sel);
        cudaEventDestroy(c->ev_a);
        cudaEventDestroy(c->ev_b);
        delete c;
    });
}

int keep_ctx_trim(void* ctx) {
    return guard([&] {
        Context& c = *C(ctx);
        KEEP_CUDA(cudaDeviceSynchronize());
        c.batch.reset();  // workspaces grow back on demand
        c.pf.reset();
        c.refresh.reset();
        c.refresh_ws.release();
        c.kv.release();
        c.alias_arena = nullptr;
        c.alias_hold.reset();
    });
}

int keep_ctx_synchronize(void* ctx) {
    return guard([&] { KEEP_CUDA(cudaStreamSynchronize(C(ctx)->s_main)); });
}

int keep_model_init(void* ctx) {
    return guard([&] { model_alloc_init(*C(ctx)); });
}

int keep_model_export(void* ctx, float* hw, uint64_t count) {
    return guard([&] {
        Context& c = *C(ctx);
        const int64_t d = c.d, f = c.f, V = c.V;
        const uint64_t need = 2ull * V * d + uint64_t(c.L) * (4ull * d * d + 2ull * d * f);
        if (count < need) raise(KEEP_ERR_INPUT, "export buffer too small");
        const double std_ = 1.0 / std::sqrt(double(d));
        DevBuf tmp;
        tmp.ensure(sizeof(float) * size_t(std::max(V * d, std::max(d * f, d * d))));
        float* o = hw;
        auto one = [&](const char* name, int64_t r, int64_t cols) {
            launch_init_tensor(c.cfg.seed, name, r, cols, std_, tmp.p, cols, 0, false, c.s_main);
            KEEP_CUDA(cudaMemcpyAsync(o, tmp.p, sizeof(float) * r * cols, cudaMemcpyDeviceToHost, c.s_main));
            KEEP_CUDA(cudaStreamSynchronize(c.s_main));
            o += r * cols;
        };
        one("embed", V, d);
        one("unembed", d, V);
        char nm[64];
        const char* parts[6] = {"wq", "wk", "wv", "wo", "mlp_in", "mlp_out"};
        for (int l = 0; l < c.L; ++l)
            for (int k = 0; k < 6; ++k) {
                std::snprintf(nm, sizeof nm, "layer%d.%s", l, parts[k]);
                one(nm, k == 5 ? f : d, k == 4 ? f : d);
            }
    });
}

int keep_memory_put(void* ctx, keep_owner owner, uint64_t version, int32_t layer, int64_t tokens,
                    const float* keys, const float* values, int32_t tier) {
    return guard([&] {
        Context& c = *C(ctx);
        ++c.store_gen;
        if (layer < 0 || layer >= c.L) raise(KEEP_ERR_INPUT, "layer out of range");
        if (tokens < 1) raise(KEEP_ERR_INPUT, "empty block");
        if (tier != KEEP_TIER_DEVICE && tier != KEEP_TIER_HOST) raise(KEEP_ERR_CONFIG, "unknown tier");
        const OwnerKey k{owner.kind, owner.id};
        auto& cur = c.current_version[k];
        cur = std::max(cur, version);  // cache_manager.hpp:80-81
        auto it = c.store.find(k);
        if (it == c.store.end() || it->second.tokens != tokens || it->second.arena->tier != tier ||
            it->second.arena.use_count() > 1) {
            Payload pl;
            if (it != c.store.end() && it->second.tokens == tokens && it->second.arena->tier == tier) {
                // keep the other layers of a shared arena by copying them out
                pl.arena = make_arena(c, tokens, tier);
                pl.tokens = tokens;
                pl.layer_version = it->second.layer_version;
                pl.present = it->second.present;
                const size_t blk = size_t(tokens) * c.dl * c.elem;
                for (int l = 0; l < c.L; ++l) {
                    if (!pl.present[l]) continue;
                    KEEP_CUDA(cudaMemcpy(layer_keys(c, pl, l), layer_keys(c, it->second, l), blk, cudaMemcpyDefault));
                    KEEP_CUDA(cudaMemcpy(layer_values(c, pl, l), layer_values(c, it->second, l), blk, cudaMemcpyDefault));
                }
            } else {
                // A block of another size or tier.  The reference keys blocks by
                // (owner, layer) (cache_manager.hpp:69-99), so a put never
                // discards the owner's other layers; here an owner's layers share
                // one row block.  Stale layers may go (a load of them misses
                // either way); still-current ones of the old shape are an error
                // instead of a silent drop.
                if (it != c.store.end())
                    for (int l = 0; l < c.L; ++l)
                        if (l != layer && it->second.present[l] && it->second.layer_version[l] >= cur)
                            raise(KEEP_ERR_INPUT, "put of " + std::to_string(tokens) + " tokens for " + owner_str(k) +
                                                      " would drop its current layer " + std::to_string(l) + " of " +
                                                      std::to_string(it->second.tokens) +
                                                      " tokens (different size or tier); invalidate the owner first");
                pl.arena = make_arena(c, tokens, tier);
                pl.tokens = tokens;
                pl.layer_version.assign(c.L, 0);
                pl.present.assign(c.L, 0);
            }
            c.store[k] = std::move(pl);
        }
        Payload& pl = c.store[k];
        drop_mirror(*pl.arena);
        // this rank's head columns of the full rows
        const int64_t dl = c.dl, c0 = int64_t(c.R) * dl;
        const size_t nel = size_t(tokens) * dl;
        if (!c.fast) {
            KEEP_CUDA(cudaMemcpy2D(layer_keys(c, pl, layer), dl * 4, keys + c0, size_t(c.d) * 4, dl * 4, tokens,
                                   cudaMemcpyDefault));
            KEEP_CUDA(cudaMemcpy2D(layer_values(c, pl, layer), dl * 4, values + c0, size_t(c.d) * 4, dl * 4, tokens,
                                   cudaMemcpyDefault));
        } else {
            std::vector<uint16_t> tk(nel), tv(nel);
            for (int64_t t = 0; t < tokens; ++t)
                for (int64_t j = 0; j < dl; ++j) {
                    tk[t * dl + j] = f2bf(keys[t * c.d + c0 + j]);
                    tv[t * dl + j] = f2bf(values[t * c.d + c0 + j]);
                }
            KEEP_CUDA(cudaMemcpy(layer_keys(c, pl, layer), tk.data(), 2 * nel, cudaMemcpyDefault));
            KEEP_CUDA(cudaMemcpy(layer_values(c, pl, layer), tv.data(), 2 * nel, cudaMemcpyDefault));
        }
        pl.layer_version[layer] = version;
        pl.present[layer] = 1;
    });
}

int keep_memory_compute(void* ctx, keep_owner owner, uint64_t version, int32_t n_members,
                        const int32_t* member_len, const int32_t* tokens, int32_t tier) {
    return guard([&] {
        memory_compute_batch(*C(ctx), 1, &owner, &version, &n_members, member_len, tokens, tier);
    });
}

int keep_memory_compute_batch(void* ctx, int32_t n_owners, const keep_owner* owners, const uint64_t* versions,
                              const int32_t* owner_members, const int32_t* member_len, const int32_t* tokens,
                              int32_t tier) {
    return guard([&] {
        Context& c = *C(ctx);
        // one profiler region for the whole refresh (its layers are not prefill phases)
        int64_t toks = 0;
        for (int o = 0, mi = 0; o < n_owners; ++o)
            for (int k = 0; k < owner_members[o]; ++k) toks += member_len[mi++];
        ProfScope ps(c.prof, KEEP_PROF_REFRESH, c.s_main,
                     2.0 * double(toks) * c.L * (3.0 * c.dl * c.d + (c.d * double(c.d) + 2.0 * c.d * c.f) / c.G), 0.0);
        const bool was = c.prof.on;
        c.prof.on = false;
        try {
            memory_compute_batch(c, n_owners, owners, versions, owner_members, member_len, tokens, tier);
        } catch (...) {
            c.prof.on = was;
            throw;
        }
        c.prof.on = was;
    });
}

namespace {
// CacheManager::load (cache_manager.hpp:103-130).  A slow-tier block is copied
// to HBM on the copy stream and the owner promoted; async: the copies are
// only enqueued (c.ev_b completes them), the old host arena is held until then.
void load_memory_impl(Context& c, keep_owner owner, int32_t layer, keep_kv_view* out, bool async) {
    ++c.store_gen;
    const OwnerKey k{owner.kind, owner.id};
    const Payload* pl = nullptr;
    if (!block_current(c, k, layer, &pl)) {  // cache_manager.hpp:104-116
        c.stats.cache_misses++;
        const bool absent = c.store.find(k) == c.store.end();
        raise(KEEP_ERR_CACHE_MISS, std::string(absent ? "no block for " : "stale block for ") + owner_str(k) +
                                       " layer " + std::to_string(layer));
    }
    Payload& P = c.store[k];
    out->tokens = P.tokens;
    out->elem_bytes = c.elem;
    out->tier = P.arena->tier;
    out->load_ms = 0.0;
    out->row_elems = c.dl;
    out->col0 = c.R * c.dl;
    if (!async) c.load_hold.clear();
    KEEP_CUDA(cudaEventRecord(c.ev_a, c.s_copy));
    if (P.arena->tier == KEEP_TIER_HOST) {
        // slow tier: copy the block to HBM and promote the owner (117-127)
        const size_t blk = size_t(P.tokens) * c.dl * c.elem;
        auto dev = make_arena(c, P.tokens, KEEP_TIER_DEVICE);
        Payload np;
        np.arena = dev;
        np.tokens = P.tokens;
        np.layer_version = P.layer_version;
        np.present = P.present;
        for (int l = 0; l < c.L; ++l) {
            if (!np.present[l]) continue;
            KEEP_CUDA(cudaMemcpyAsync(layer_keys(c, np, l), layer_keys(c, P, l), blk, cudaMemcpyDefault, c.s_copy));
            KEEP_CUDA(cudaMemcpyAsync(layer_values(c, np, l), layer_values(c, P, l), blk, cudaMemcpyDefault, c.s_copy));
            if (l < P.arena->mirror_from) c.stats.bytes_loaded_slow += 2 * blk;
        }
        c.load_hold.push_back(P.arena);  // the source stays alive until the copies complete
        c.store[k] = std::move(np);
    }
    KEEP_CUDA(cudaEventRecord(c.ev_b, c.s_copy));
    if (async) {
        out->load_ms = -1.0;  // (measured only by the blocking form)
    } else {
        KEEP_CUDA(cudaEventSynchronize(c.ev_b));
        float ms = 0.f;
        KEEP_CUDA(cudaEventElapsedTime(&ms, c.ev_a, c.ev_b));
        out->load_ms = out->tier == KEEP_TIER_HOST ? ms : 0.0;
        c.load_hold.clear();
    }
    const Payload& Q = c.store[k];
    out->keys = layer_keys(c, Q, layer);
    out->values = layer_values(c, Q, layer);
}
}  // namespace

int keep_load_memory(void* ctx, keep_owner owner, int32_t layer, keep_kv_view* out) {
    return guard([&] { load_memory_impl(*C(ctx), owner, layer, out, false); });
}

int keep_load_memory_async(void* ctx, keep_owner owner, int32_t layer, keep_kv_view* out, void** done) {
    return guard([&] {
        Context& c = *C(ctx);
        load_memory_impl(c, owner, layer, out, true);
        if (done) *done = c.ev_b;
    });
}

int keep_load_wait(void* ctx) {
    return guard([&] {
        Context& c = *C(ctx);
        KEEP_CUDA(cudaEventSynchronize(c.ev_b));
        c.load_hold.clear();
    });
}

int keep_memory_has_current(void* ctx, keep_owner owner, uint64_t version, int32_t* out) {
    return guard([&] {  // cache_manager.hpp:151-159
        Context& c = *C(ctx);
        const OwnerKey k{owner.kind, owner.id};
        *out = 0;
        auto cv = c.current_version.find(k);
        if (cv != c.current_version.end() && cv->second > version) return;
        auto it = c.store.find(k);
        if (it == c.store.end()) return;
        for (int l = 0; l < c.L; ++l)
            if (!it->second.present[l] || it->second.layer_version[l] != version) return;
        *out = 1;
    });
}

int keep_invalidate(void* ctx, keep_owner owner, uint64_t new_version, uint64_t tokens) {
    return guard([&] {  // cache_manager.hpp:163-184
        Context& c = *C(ctx);
        ++c.store_gen;
        const OwnerKey k{owner.kind, owner.id};
        auto it = c.store.find(k);
        if (it != c.store.end()) {
            c.store.erase(it);
            c.stats.tokens_invalidated += tokens;
        }
        auto& cur = c.current_version[k];
        cur = std::max(cur, new_version);
    });
}

int keep_memory_clear(void* ctx) {
    return guard([&] {  // a fresh CacheManager (harness.hpp:490-497 builds one per episode)
        Context& c = *C(ctx);
        KEEP_CUDA(cudaDeviceSynchronize());
        ++c.store_gen;
        c.alias_arena = nullptr;
        c.alias_hold.reset();
        c.store.clear();
        c.current_version.clear();
        c.stats = keep_memory_stats{};
    });
}

int keep_memory_residency(void* ctx, uint64_t hbm_budget_bytes, uint64_t* resident_bytes) {
    return guard([&] {  // CacheManager's capacity-bounded fast tier (cache_manager.hpp:23-35, 103-130)
        Context& c = *C(ctx);
        KEEP_CUDA(cudaDeviceSynchronize());
        ++c.store_gen;
        // the budget also places the deepest layers of pinned-host arenas
        // created from here on (canonical KV computed straight into HBM)
        c.hbm_budget = hbm_budget_bytes;
        std::vector<Arena*> host;
        uint64_t split_bytes = 0;
        for (auto& [k, pl] : c.store)
            if (pl.arena->tier == KEEP_TIER_HOST &&
                std::find(host.begin(), host.end(), pl.arena.get()) == host.end()) {
                if (pl.arena->split) split_bytes += pl.arena->mirror.bytes;  // (its layers cannot move)
                else host.push_back(pl.arena.get());
            }
        uint64_t per_layer = 0;
        for (Arena* a : host) {
            drop_mirror(*a);
            per_layer += uint64_t(2) * a->rows * c.dl * c.elem;
        }
        // the deepest layers first: plans only shrink with depth (monotone,
        // prefill.hpp:95-104), so deep layers reuse the most cached KV
        const uint64_t avail = hbm_budget_bytes > split_bytes ? hbm_budget_bytes - split_bytes : 0;
        const int m = per_layer ? int(std::min<uint64_t>(uint64_t(c.L), avail / per_layer)) : 0;
        uint64_t total = split_bytes;
        for (Arena* a : host) {
            if (m == 0) break;
            const size_t sheet2 = size_t(2) * a->rows * c.dl * c.elem;
            a->mirror.ensure(sheet2 * m);
            KEEP_CUDA(cudaMemcpy(a->mirror.p, static_cast<uint8_t*>(a->buf.p) + sheet2 * (c.L - m), sheet2 * m,
                                 cudaMemcpyHostToDevice));
            a->mirror_from = c.L - m;
            total += sheet2 * m;
        }
        if (resident_bytes) *resident_bytes = total;
    });
}

int keep_ctx_dims(void* ctx, int32_t* dims) {
    return guard([&] {
        const Context& c = *C(ctx);
        const int32_t v[7] = {c.L, c.H, c.d, c.f, c.V, c.cfg.numerics, c.cfg.world_size};
        std::copy(v, v + 7, dims);
    });
}

int keep_memory_stats_get(void* ctx, keep_memory_stats* out) {
    return guard([&] {
        Context& c = *C(ctx);
        keep_memory_stats s = c.stats;
        s.blocks = 0;
        s.device_bytes = s.host_bytes = 0;
        std::vector<const Arena*> seen;
        for (const auto& [k, p] : c.store) {
            for (int l = 0; l < c.L; ++l) s.blocks += p.present[l];
            const Arena* a = p.arena.get();
            if (std::find(seen.begin(), seen.end(), a) != seen.end()) continue;
            seen.push_back(a);
            (a->tier == KEEP_TIER_HOST ? s.host_bytes : s.device_bytes) += a->buf.bytes;
            if (a->mirror_from < (1 << 30)) s.device_bytes += a->mirror.bytes;
        }
        *out = s;
    });
}

int keep_memory_read(void* ctx, keep_owner owner, int32_t layer, float* keys, float* values) {
    return guard([&] {
        Context& c = *C(ctx);
        const Payload* pl = nullptr;
        if (!block_current(c, OwnerKey{owner.kind, owner.id}, layer, &pl))
            raise(KEEP_ERR_CACHE_MISS, "no current block");
        const size_t nel = size_t(pl->tokens) * c.dl;
        if (!c.fast) {
            KEEP_CUDA(cudaMemcpy(keys, layer_keys(c, *pl, layer), 4 * nel, cudaMemcpyDefault));
            KEEP_CUDA(cudaMemcpy(values, layer_values(c, *pl, layer), 4 * nel, cudaMemcpyDefault));
        } else {
            std::vector<uint16_t> t(nel);
            KEEP_CUDA(cudaMemcpy(t.data(), layer_keys(c, *pl, layer), 2 * nel, cudaMemcpyDefault));
            for (size_t i = 0; i < nel; ++i) keys[i] = bf2f(t[i]);
            KEEP_CUDA(cudaMemcpy(t.data(), layer_values(c, *pl, layer), 2 * nel, cudaMemcpyDefault));
            for (size_t i = 0; i < nel; ++i) values[i] = bf2f(t[i]);
        }
    });
}

int keep_prefill_begin(void* ctx, const keep_layout* layout, const int32_t* query, int32_t qlen) {
    return guard([&] { cursor_begin(*C(ctx), layout, query, qlen); });
}

int keep_prefill_layer(void* ctx, const uint8_t* active, double* summary_out) {
    return guard([&] {
        Context& c = *C(ctx);
        if (!c.pf) raise(KEEP_ERR_PLAN, "no prefill in progress");
        c.pf->summary_wanted = summary_out != nullptr;  // (nobody reads it otherwise)
        cursor_layer(c, active);
        if (summary_out) {
            const size_t ns = size_t(c.pf->S) + size_t(c.pf->S) * c.pf->S;
            KEEP_CUDA(cudaMemcpyAsync(summary_out, c.pf->summ.p, sizeof(double) * ns, cudaMemcpyDeviceToHost, c.s_main));
        }
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
    });
}

int keep_prefill_finish(void* ctx, float* final_hidden, float* kv_out) {
    return guard([&] {
        Context& c = *C(ctx);
        if (!c.pf) raise(KEEP_ERR_PLAN, "no prefill in progress");
        cursor_finish(c, final_hidden, kv_out);
    });
}

int keep_importance_evaluation(void* ctx, int32_t S, const double* qts, const double* sts, int64_t budget,
                               const uint8_t* candidates, int32_t* order_out, int32_t* n_out, int32_t* hops_out) {
    return guard([&] {
        Context& c = *C(ctx);
        if (S < 0) raise(KEEP_ERR_INPUT, "negative segment count");
        DevBuf dq, ds, dc;
        cudaStream_t st = c.s_sel;
        dq.ensure(sizeof(double) * std::max(S, 1));
        ds.ensure(sizeof(double) * std::max<size_t>(size_t(S) * S, 1));
        KEEP_CUDA(cudaMemcpyAsync(dq.p, qts, sizeof(double) * S, cudaMemcpyHostToDevice, st));
        KEEP_CUDA(cudaMemcpyAsync(ds.p, sts, sizeof(double) * size_t(S) * S, cudaMemcpyHostToDevice, st));
        if (candidates) {
            dc.ensure(std::max(S, 1));
            KEEP_CUDA(cudaMemcpyAsync(dc.p, candidates, S, cudaMemcpyHostToDevice, st));
        }
        c.sel_order.ensure(sizeof(int32_t) * (std::max(S, 1) + 2));
        int32_t* o = c.sel_order.as<int32_t>();
        launch_select(S, dq.as<double>(), ds.as<double>(), budget, candidates ? dc.as<uint8_t>() : nullptr, o + 2,
                      o, o + 1, st, c.cfg.max_hops);
        std::vector<int32_t> h(S + 2);
        KEEP_CUDA(cudaMemcpyAsync(h.data(), o, sizeof(int32_t) * (S + 2), cudaMemcpyDeviceToHost, st));
        KEEP_CUDA(cudaStreamSynchronize(st));
        *n_out = h[0];
        *hops_out = h[1];
        std::copy(h.begin() + 2, h.begin() + 2 + h[0], order_out);
    });
}

int keep_shard_heads(int32_t H, int32_t d, int32_t G, int32_t R, int32_t* h0, int32_t* hn, int32_t* c0,
                     int32_t* cn) {
    return guard([&] {
        if (G < 1 || R < 0 || R >= G || H < 1 || H % G != 0 || d % H != 0)
            raise(KEEP_ERR_CONFIG, "bad head partition");
        const int32_t hl = H / G, dh = d / H;
        *h0 = R * hl;
        *hn = hl;
        *c0 = R * hl * dh;
        *cn = hl * dh;
    });
}

int keep_shard_rows(int64_t n, int32_t G, int32_t R, int64_t* r0, int64_t* m) {
    return guard([&] {
        if (G < 1 || R < 0 || R >= G || n < 0) raise(KEEP_ERR_CONFIG, "bad row partition");
        const int64_t cpr = ceil_div(n, G);
        *r0 = std::min<int64_t>(n, int64_t(R) * cpr);
        *m = std::min<int64_t>(n, *r0 + cpr) - *r0;
    });
}

int keep_ratio_schedule(int32_t L, double r_avg, double* r) {
    return guard([&] {  // recompute.hpp:33-70
        if (L < 1) raise(KEEP_ERR_CONFIG, "num_layers must be >= 1");
        if (L == 1) {
            r[0] = 1.0;
            return;
        }
        if (r_avg < 1.0 / L - 1e-9 || r_avg > 1.0 + 1e-9) raise(KEEP_ERR_CONFIG, "infeasible r_avg " + std::to_string(r_avg));
        double lo = 0.0, hi = 1.0;
        for (int it = 0; it < 200; ++it) {
            const double g = 0.5 * (lo + hi);
            double sum = 0.0, term = 1.0;
            for (int l = 0; l < L; ++l) {
                sum += term;
                term *= g;
            }
            if (sum / L < r_avg) lo = g;
            else hi = g;
        }
        const double g = 0.5 * (lo + hi);
        double term = 1.0;
        for (int l = 0; l < L; ++l) {
            r[l] = term;
            term *= g;
        }
        r[0] = 1.0;
    });
}

int64_t keep_layer_budget(double ratio, int64_t S) {  // recompute.hpp:73-77
    int64_t b = int64_t(std::ceil(ratio * double(S) - 1e-9));
    b = std::min(b, S);
    return std::max<int64_t>(1, b);
}

int keep_profile_enable(void* ctx, int32_t on) {
    return guard([&] { C(ctx)->prof.on = on != 0; });
}

int keep_profile_read(void* ctx, keep_profile* out, int32_t reset) {
    return guard([&] {
        Context& c = *C(ctx);
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
        KEEP_CUDA(cudaStreamSynchronize(c.s_sel));
        c.prof.collect();
        *out = c.prof.acc;
        if (reset) c.prof.acc = keep_profile{};
    });
}

int keep_logits(void* ctx, const float* row, double* out) {
    return guard([&] {
        Context& c = *C(ctx);
        need_weights(c);
        DevBuf dr;
        dr.ensure(sizeof(float) * c.d);
        c.logits.ensure(sizeof(double) * c.V);
        KEEP_CUDA(cudaMemcpyAsync(dr.p, row, sizeof(float) * c.d, cudaMemcpyHostToDevice, c.s_main));
        launch_logits(dr.as<float>(), c.unembed.as<float>(), c.d, c.V, c.logits.as<double>(), c.s_main);
        KEEP_CUDA(cudaMemcpyAsync(out, c.logits.p, sizeof(double) * c.V, cudaMemcpyDeviceToHost, c.s_main));
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
    });
}

int keep_divergence(void* ctx, const float* row_a, const float* row_b, double* l2, double* sym_kl) {
    return guard([&] {  // prefill.hpp:501-531
        Context& c = *C(ctx);
        need_weights(c);
        DevBuf rows, lg, out;
        rows.ensure(sizeof(float) * 2 * c.d);
        lg.ensure(sizeof(double) * 2 * size_t(c.V));
        out.ensure(sizeof(double) * 2);
        float* ra = rows.as<float>();
        KEEP_CUDA(cudaMemcpyAsync(ra, row_a, sizeof(float) * c.d, cudaMemcpyHostToDevice, c.s_main));
        KEEP_CUDA(cudaMemcpyAsync(ra + c.d, row_b, sizeof(float) * c.d, cudaMemcpyHostToDevice, c.s_main));
        launch_logits(ra, c.unembed.as<float>(), c.d, c.V, lg.as<double>(), c.s_main);
        launch_logits(ra + c.d, c.unembed.as<float>(), c.d, c.V, lg.as<double>() + c.V, c.s_main);
        launch_divergence(ra, ra + c.d, c.d, lg.as<double>(), lg.as<double>() + c.V, c.V, out.as<double>(), c.s_main);
        double h[2];
        KEEP_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, c.s_main));
        KEEP_CUDA(cudaStreamSynchronize(c.s_main));
        *l2 = h[0];
        *sym_kl = h[1];
    });
}

// plan_keep (recompute.hpp:140-180) with every layer, the selection and the
// last-row logits on the device.  The host only decides keep-all vs walk from
// the budget and applies the returned order (one small D2H per layer).
int keep_plan_keep_batch(void* ctx, const keep_layout* layout, int32_t batch, const int32_t* queries, int32_t qlen,
                         const double* sched, int32_t multihop, keep_plan_result* outs) {
    return guard([&] {
        if (C(ctx)->rope_theta > 0.0) raise(KEEP_ERR_CONFIG, "the RoPE hook is single-query (keep_plan_keep)");
        plan_keep_batch(*C(ctx), layout, batch, queries, qlen, sched, multihop != 0, outs);
    });
}

int keep_set_rope(void* ctx, double theta) {
    return guard([&] {
        if (!(theta >= 0.0)) raise(KEEP_ERR_CONFIG, "rope theta must be >= 0 (0 = off)");
        Context& c = *C(ctx);
        if (c.G > 1) raise(KEEP_ERR_CONFIG, "the RoPE hook is single-GPU");
        c.rope_theta = theta;
    });
}

int keep_selective_prefill_batch(void* ctx, const keep_layout* layout, int32_t batch, const int32_t* queries,
                                 int32_t qlen, const uint8_t* plans, keep_plan_result* outs) {
    return guard([&] {
        if (!plans) raise(KEEP_ERR_PLAN, "null plans");
        if (C(ctx)->rope_theta > 0.0) raise(KEEP_ERR_CONFIG, "the RoPE hook is single-query");
        plan_keep_batch(*C(ctx), layout, batch, queries, qlen, nullptr, true, outs, plans);
    });
}

int keep_plan_keep(void* ctx, const keep_layout* layout, const int32_t* query, int32_t qlen,
                   const double* sched, int32_t multihop, keep_plan_result* out) {
    return guard([&] {
        Context& c = *C(ctx);
        cudaStream_t st = c.s_main;
        // per-context events and pinned walk buffer, created once (no
        // cudaHostAlloc / event churn on the TTFT path)
        if (c.pk_evs.size() != size_t(c.L + 1)) {
            for (auto e : c.pk_evs) cudaEventDestroy(e);
            c.pk_evs.assign(c.L + 1, nullptr);
            for (auto& e : c.pk_evs) KEEP_CUDA(cudaEventCreate(&e));
        }
        std::vector<cudaEvent_t>& evs = c.pk_evs;
        KEEP_CUDA(cudaEventRecord(evs[0], st));
        cursor_begin(c, layout, query, qlen);
        Pass& p = *c.pf;
        const int S = p.S, L = c.L;
        std::vector<uint8_t> active(S, 1);
        c.sel_order.ensure(sizeof(int32_t) * (S + 2));
        c.sel_cand.ensure(std::max(S, 1));
        // pinned: the async D2H of the walk must not stage
        if (c.walk_host.bytes < sizeof(int32_t) * size_t(S + 2) || !c.walk_host.host)
            c.walk_host.alloc(sizeof(int32_t) * size_t(S + 2), true);
        int32_t* hbuf = c.walk_host.as<int32_t>();
        if (!c.ev_sum) {
            KEEP_CUDA(cudaEventCreateWithFlags(&c.ev_sum, cudaEventDisableTiming));
            KEEP_CUDA(cudaEventCreateWithFlags(&c.ev_sel, cudaEventDisableTiming));
        }
        cudaEvent_t ev_sum = c.ev_sum, ev_sel = c.ev_sel;
        for (int l = 0; l < L; ++l) {
            if (out && out->plan) std::copy(active.begin(), active.end(), out->plan + size_t(l) * S);
            if (out && out->order_len) out->order_len[l] = -1;
            if (out && out->hops) out->hops[l] = 0;
            int64_t budget = 0, live = 0;
            if (l + 1 < L) {
                budget = keep_layer_budget(sched[l + 1], S);
                for (uint8_t x : active) live += x;
            }
            const bool walk = l + 1 < L && budget < live && multihop;
            // the walk for layer l+1 runs on the selector stream as soon as the
            // summary of layer l exists, overlapping this layer's Wo + MLP
            auto launch_walk = [&] {
                if (!walk) return;
                if (p.walk_empty) {  // the probe's proof: the first hop adds nothing
                    hbuf[0] = 0;
                    hbuf[1] = 1;
                    KEEP_CUDA(cudaEventRecord(ev_sel, c.s_sel));
                    return;
                }
                upload_bytes(c.sel_cand.p, active.data(), S, c.s_sel);
                KEEP_CUDA(cudaEventRecord(ev_sum, st));
                KEEP_CUDA(cudaStreamWaitEvent(c.s_sel, ev_sum, 0));
                const bool trace = c.loader.on;  // the realised timeline (keep_timeline_trace)
                if (trace) {
                    c.loader.has_eval[l] = 1;
                    KEEP_CUDA(cudaEventRecord(c.loader.attn_end[l], st));
                    KEEP_CUDA(cudaEventRecord(c.loader.eval_a[l], c.s_sel));
                }
                int32_t* o = c.sel_order.as<int32_t>();
                {
                    ProfScope ps(c.prof, KEEP_PROF_SELECT, c.s_sel, 0.0, 8.0 * double(S) * S);
                    launch_select(S, p.summ.as<double>(), p.summ.as<double>() + S, budget, c.sel_cand.as<uint8_t>(), o + 2,
                                  o, o + 1, c.s_sel, c.cfg.max_hops);
                }
                if (trace) KEEP_CUDA(cudaEventRecord(c.loader.eval_b[l], c.s_sel));
                KEEP_CUDA(cudaMemcpyAsync(hbuf, o, sizeof(int32_t) * (S + 2), cudaMemcpyDeviceToHost, c.s_sel));
                KEEP_CUDA(cudaEventRecord(ev_sel, c.s_sel));
            };
            c.gemm_ctas = walk ? kNumSMs - 1 : kNumSMs;
            // The summary is consumed only by a walk (or the single-hop ablation)
            // and by callers asking for it; plan_keep's plans are unchanged when
            // the other layers skip it (the reference computes and discards it).
            // Sharded: the per-rank partials are summed only when read.
            p.summary_wanted = walk || (out && out->summaries) || (l + 1 < L && budget < live && !multihop);
            p.summary_global = p.summary_wanted;
            p.walk_probe = walk && !(out && out->summaries) && !c.fast && !c.exact && c.G == 1 && lazy_summary_enabled();
            if (p.walk_probe) {
                p.d_walk_cand.ensure(size_t(S));
                upload_bytes(p.d_walk_cand.p, active.data(), S, st);
            }
            cursor_layer(c, active.data(), launch_walk);
            p.walk_probe = false;
            p.walk_empty = false;
            p.summary_global = true;
            p.summary_wanted = true;
            c.gemm_ctas = kNumSMs;
            if (out && out->rows_per_layer) out->rows_per_layer[l] = p.n;
            if (out && out->summaries)
                KEEP_CUDA(cudaMemcpyAsync(out->summaries + size_t(l) * (S + size_t(S) * S), p.summ.p,
                                          sizeof(double) * (S + size_t(S) * S), cudaMemcpyDeviceToHost, st));
            KEEP_CUDA(cudaEventRecord(evs[l + 1], st));
            if (l + 1 >= L) break;
            if (budget >= live) continue;  // recompute everything still live
            std::vector<uint8_t> next(S, 0);
            if (multihop) {
                KEEP_CUDA(cudaEventSynchronize(ev_sel));
                for (int k = 0; k < hbuf[0]; ++k) next[hbuf[2 + k]] = 1;
                if (out && out->orders) std::copy(hbuf + 2, hbuf + 2 + hbuf[0], out->orders + size_t(l) * S);
                if (out && out->order_len) out->order_len[l] = hbuf[0];
                if (out && out->hops) out->hops[l] = hbuf[1];
            } else {  // single-hop ablation (recompute.hpp:166-176): ranked on the device
                upload(c.d_live, active, st);
                c.d_next.ensure(size_t(S));
                launch_single_hop(p.summ.as<double>(), c.d_live.as<uint8_t>(), S, budget, c.d_next.as<uint8_t>(), st);
                KEEP_CUDA(cudaMemcpyAsync(next.data(), c.d_next.p, size_t(S), cudaMemcpyDeviceToHost, st));
                KEEP_CUDA(cudaStreamSynchronize(st));
            }
            active = std::move(next);
        }
        // last-row logits (model.hpp:76-85) close the TTFT
        c.logits.ensure(sizeof(double) * c.V);
        const float* lr = last_row_ptr(c, p);
        DevBuf zero;
        if (!lr) {
            zero.ensure(sizeof(float) * c.d);
            KEEP_CUDA(cudaMemsetAsync(zero.p, 0, sizeof(float) * c.d, st));
            lr = zero.as<float>();
        }
        {
            ProfScope ps(c.prof, KEEP_PROF_LOGITS, st, 2.0 * c.d * double(c.V), 4.0 * c.d * double(c.V));
            launch_logits(lr, c.unembed.as<float>(), c.d, c.V, c.logits.as<double>(), st);
        }
        KEEP_CUDA(cudaEventRecord(c.ev_b, st));
        if (out && out->last_logits)
            KEEP_CUDA(cudaMemcpyAsync(out->last_logits, c.logits.p, sizeof(double) * c.V, cudaMemcpyDeviceToHost, st));
        KEEP_CUDA(cudaStreamSynchronize(st));
        if (out) {
            float ms = 0.f;
            KEEP_CUDA(cudaEventElapsedTime(&ms, evs[0], c.ev_b));
            out->ttft_ms = ms;
            if (out->layer_ms)
                for (int l = 0; l < L; ++l) {
                    float m = 0.f;
                    KEEP_CUDA(cudaEventElapsedTime(&m, evs[l], evs[l + 1]));
                    out->layer_ms[l] = m;
                }
            if (out->final_hidden) cursor_finish(c, out->final_hidden, nullptr);
        }
    });
}

}  // extern "C"
