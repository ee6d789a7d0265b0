// engine.hpp -- the B200 KEEP prefill engine behind the C ABI (internal).
#pragma once

#include <map>
#include <memory>
#include <vector>

#include "kernels.hpp"

namespace keep_b200 {

// FAST-mode projection GEMM on the tcgen05 tensor cores:
// C[M x N] = A[M x K] (bf16 row-major) . Bt[N x K]^T (bf16, K-major rows).
// max_ctas < 148 leaves SMs free for a concurrently running selector.
void launch_gemm_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bt, int64_t ldb,
                      int M, int N, int K, const EpiArgs& epi, cudaStream_t st, int max_ctas = kNumSMs);

// FAST attention on tcgen05 (head_dim 128): stats / context / bins passes.
struct AttnTcLaunch {
    int n, T, H, d, S;        // H = this rank's heads, d = H * 128
    double inv_heads;         // 1 / (heads of the model)
    const void* q;            // [n x d] bf16 compact queries
    const void* k;            // [T x d] bf16 merged keys
    const void* v;            // [T x d] bf16 merged values
    __nv_bfloat16* vt;        // scratch [d x roundup(T, 64)]
    const int32_t* rows;
    const int32_t* row_seg;
    const int32_t* key_lo;    // nullable
    bool with_bins;
    int nsplit_a;             // stats / context splits (any cut)
    const int32_t* split_lo_a;
    const int32_t* split_hi_a;
    float* m_part;            // [nsplit_a x n x H]
    float* l_part;
    float* m_fin;             // [n x H]
    float* inv_l;
    float* o_part;            // [nsplit_a x n x d]
    __nv_bfloat16* ctx;       // [n x d]
    double* summ_raw;         // scratch [S + S*S] (raw qts, sts)
    double* summ;             // out [S + S*S] normalised summary
    const int32_t* seg_len;   // [S]
    int qlen;
    const void* chunk_tab;    // launch_chunk_table output (summary only)
    const void* zt;           // launch_zt_build output: Z^T tiles [nchunks * nb x 128] bf16
    int nb;                   // summary bins per chunk on the tensor core (16 / 32; 0 = scan bins)
};
int launch_attention_tc(const AttnTcLaunch& a, cudaStream_t st);  // returns kernels launched
// few-row layers without a summary (attn_decode.cu): single-pass split-K
// flash decoding over keys [0, kv_hi); uses q, k, v, rows, m_part, l_part,
// o_part (fp32, sized decode_splits x n x {H, d}) and ctx of the launch
bool decode_attention_fits(int n);
int decode_splits(int n_heads, int kv_hi);
int launch_attention_decode(const AttnTcLaunch& a, int kv_hi, cudaStream_t st);
// Several queries of a batch at an all-reused layer, one launch: each query's
// rows attend the shared memory sheet (rows [0, kv_mem) of k_mem / v_mem,
// read once through L2 for all of them) and then their own qlen key rows
// (rows qrow0[i] .. of k_own / v_own, own_rows rows in total).
struct DecodeMulti {
    int H = 0, d = 0, qlen = 0, kv_mem = 0, own_rows = 0;
    const void* k_mem = nullptr;
    const void* v_mem = nullptr;
    const void* k_own = nullptr;
    const void* v_own = nullptr;
    const void* q = nullptr;            // [rows x d] (pre-scaled)
    const int32_t* rows = nullptr;      // [qlen] positions kv_mem .. (the same for every query)
    __nv_bfloat16* ctx = nullptr;
    std::vector<int> qrow0, qoff;       // per query: own key row base, first q / ctx row
};
int launch_attention_decode_multi(const DecodeMulti& m, cudaStream_t st);
// per-128-key-chunk destination-segment table (32 B per chunk)
void launch_chunk_table(const int32_t* row_seg, int T, void* tab, cudaStream_t st);
// bins width for a layout (max segments touching a 128-key chunk, rounded to
// 16 / 32; 0 when some chunk has more than 32) and the Z^T indicator tiles
int summary_bins_width(const std::vector<int32_t>& row_seg);
bool bins_on_tensor_core();  // P . Z bins with P = bf16 hi + bf16 lo (default; KEEP_BINS=scan: CUDA-core scan)
void launch_zt_build(const int32_t* row_seg, int T, const void* tab, int nb, void* zt, cudaStream_t st);

// Collectives of KV-head sharding (comm.cu).  All stream-ordered on `st`.
struct Comm {
    int world = 1, rank = 0;
    virtual ~Comm() = default;
    // sum over ranks; every rank receives identical bits
    virtual void allreduce_f64(double* buf, size_t n, cudaStream_t st) = 0;
    // recv = blocks of `bytes` from every rank in rank order (send may be recv + rank*bytes)
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
    // send block q -> rank q; recv block q <- rank q
    virtual void alltoall(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
};
std::unique_ptr<Comm> make_comm(const keep_config& cfg);

struct Context;
struct Pass;
// loader.cu (K10)
void loader_begin(Context& c, Pass& p);
void loader_before_layer(Context& c, Pass& p, int l, const uint8_t* active);
void loader_after_layer(Context& c, Pass& p, int l, const uint8_t* active, double est_ms);
bool loader_covers(const Context& c, int seg, int l);  // segment's owner is host-tier and layer l not HBM-resident (loaded by K10)
void set_last_error(const std::string& msg);

// Per-phase CUDA-event timing (keep_profile_*).
struct Profiler {
    bool on = false;
    struct Rec {
        int cat;
        cudaEvent_t a, b;
        double flops, bytes;
        int kernels;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    keep_profile acc{};
    cudaEvent_t get();
    void collect();  // synchronises the recorded events
    ~Profiler();
};

struct Context;
// RAII region: events on `st` around the launches of one phase.
struct ProfScope {
    Profiler* p;
    int cat;
    cudaStream_t st;
    double flops, bytes;
    int kernels;
    cudaEvent_t a = nullptr;
    ProfScope(Profiler& prof, int c, cudaStream_t s, double fl, double by, int nk = 1);
    ~ProfScope();
};

// Device buffer with RAII.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool host = false;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release();
    void ensure(size_t nbytes);              // device, grow-only
    void alloc(size_t nbytes, bool pinned_host);
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

// PARITY projection GEMMs (gemm_oz.cu): the Ozaki int8 tensor-core GEMM from
// kOzMinRows rows, DFMA (gemm_f64acc.cu) below.  OzWork = its grow-only
// scratch (residue planes of A and B, scale exponents, Garner digits).
struct OzWork {
    DevBuf a, b, ea, eb, part;
};
constexpr int kOzMinRows = 64;
// the residual add of a cross-rank fp64 sum: x[m][n] += float(sum[m][n])
void launch_f64_resid(const double* sum, float* x, int M, int N, int64_t ldx, cudaStream_t st);
int oz_moduli();       // KEEP_OZ_MODULI (default 14)
int oz_bits(int K);    // integer bits per operand at contraction length K
bool ozaki_eligible(int M, int N, int K);
void launch_gemm_ozaki(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                       const EpiArgs& epi, cudaStream_t st, OzWork& w, int max_ctas = kNumSMs);
void launch_gemm_parity(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                        const EpiArgs& epi, cudaStream_t st, OzWork& w, bool exact = false, int max_ctas = kNumSMs);

// A KV arena: per layer, keys [rows x d] then values [rows x d].  Owner
// payloads are row ranges of an arena (a batch of canonical refreshes writes
// its merged KV straight into the arena -- no staging copy).
struct Arena {
    DevBuf buf;
    int64_t rows = 0;
    int64_t used = 0;  // rows [0, used) hold owner payloads; [used, rows) are spare (query rows of aliased layers)
    int tier = KEEP_TIER_DEVICE;
    int refs = 0;
    // pinned-host arenas: layers [mirror_from, L) also resident in HBM (the
    // capacity-bounded fast tier, keep_memory_residency); every read of those
    // layers goes to the mirror, and a write to the arena drops it
    DevBuf mirror;
    int mirror_from = 1 << 30;
    bool split = false;  // created with its resident layers in HBM only (no host copy of them)
};

struct OwnerKey {
    int kind;
    uint32_t id;
    bool operator<(const OwnerKey& o) const { return kind != o.kind ? kind < o.kind : id < o.id; }
};

struct Payload {
    std::shared_ptr<Arena> arena;
    int64_t row0 = 0, tokens = 0;
    std::vector<uint64_t> layer_version;  // per layer; 0 = absent
    std::vector<uint8_t> present;
};

// One prefill over a row space [0, T): the selective cursor (memory rows +
// query) or a batched canonical refresh (block-diagonal attention).
struct Pass {
    int T = 0, Tm = 0, qlen = 0, S = 0;
    bool with_summary = true;
    bool block_diag = false;
    std::vector<int32_t> seg_start, seg_len, row_seg;  // host copies
    std::vector<int32_t> key_lo_h;
    DevBuf d_tokens, d_row_seg, d_key_lo, d_seg_len, d_seg_start;
    // lazy summary (plan_keep, PARITY): the walk's candidates on the device, the
    // probe's scratch, and whether the probe proved the walk adds nothing this layer
    DevBuf d_walk_cand, d_probe;
    bool walk_probe = false, walk_empty = false;
    DevBuf ebin;                  // PARITY fused bins: [H x n x S] fp64 per-head segment sums
    DevBuf tp_part, tp_h;         // sharded few-row layers: fp64 partial sums [n x d], this rank's MLP slice [n x f/G]
    // compact state
    std::vector<int32_t> rows_h;  // compact -> global row, ascending
    int n = 0;
    DevBuf d_rows, d_rows_tmp, d_idx;
    DevBuf x, x_alt, xb, q, ctx, ctxb, h, hb;
    DevBuf xrecv, xrows;          // sharded: all-to-all receive [G][rows/G][dl], packed ctx rows
    bool summary_global = true;   // sharded: sum the summary over ranks this layer
    bool summary_wanted = true;   // plan_keep: only layers whose summary is read compute it
    // attention scratch
    DevBuf m_part, l_part, m_fin, l_fin, o_part, rowbin, split_lo, split_hi, attn_flag;
    int split_count = 1;
    DevBuf split_lo_b, split_hi_b;  // PARITY DMMA bins pass: its own segment-aligned splits
    DevBuf rope_tab;                // RoPE hook: (row, rows, delta) of the re-shifted cached blocks
    int split_count_b = 1;
    int64_t split_key = -1;
    DevBuf vt, split_lo_a, split_hi_a, chunk_tab, zt;  // FAST tensor-core attention
    int nb = 0;
    int split_count_a = 1;
    DevBuf seg_cbeg, seg_cend, summ, summ_raw;
    // merged KV destination per layer (device)
    std::vector<void*> kdst, vdst;
    std::vector<uint8_t> prev, dropped;
    int layer = 0;
};

// K10: layer-balanced loading of pinned-host memory KV (loader.cu).
// Items are (layer, owner) blocks exactly as the reference's workload
// (pipeline_sim.hpp:103-154); the schedule follows simulate_balanced
// (261-338) online: urgent loads of a layer before its compute, loads for
// l+1 of owners already out at l issued behind compute(l), and pre-loads of
// owners whose members all left the plan for layers >= l+2 filling the
// estimated compute window.  Copies are cudaMemcpyAsync (adjacent blocks merged) on a side
// stream (copy engines, no SMs); compute(l) waits on an event (D1).
struct Loader {
    struct Unit {
        OwnerKey key;
        int b = 0, e = 0;       // member segment positions [b, e)
        int64_t dst_row = 0;    // first merged-KV row
        int64_t tokens = 0;     // block rows
        const struct Payload* pl = nullptr;
    };
    struct Batch {
        cudaEvent_t a = nullptr, b = nullptr;
        int kind = 0, at_layer = 0;
        uint64_t bytes = 0;
        bool host = false;  // carried pinned-host blocks (H2D)
    };
    struct Rec {
        int layer, unit, batch;
        uint64_t bytes;
    };
    bool on = false;
    int L = 0;
    std::vector<Unit> units;
    std::vector<uint8_t> loaded;      // [L][units]
    std::vector<int> out_from;        // per unit: first layer all members are out (INT32_MAX: not yet)
    std::vector<uint8_t> seg_host;    // per layout segment: owner is host-tier (loaded here)
    std::vector<int> seg_mirror_from; // per layout segment: first HBM-resident layer of its owner
    std::vector<int> last_batch;      // per layer: last batch that carried one of its items (-1: none)
    std::vector<Batch> batches;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> comp_start;  // per layer, on the compute stream after the load wait
    // the realised timeline beside the loads (keep_timeline_trace): compute(l)
    // end, attention + summary done, and the walk (eval) on the selector stream
    std::vector<cudaEvent_t> comp_end, attn_end, eval_a, eval_b;
    std::vector<uint8_t> has_eval;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t t0 = nullptr;
    double bw_gbs = 50.0;             // H2D estimate (updated from finished batches)
    double bw_d2d_gbs = 1000.0;       // HBM->HBM copy-engine estimate
    bool any_host = false;
    size_t bw_seen = 0;
    ~Loader();
};

// Batched multi-query prefill: B queries over one memory
// layout.  `all` holds the concatenated compact rows of every instance (the
// projections stream each weight once per layer for all of them); views[b] is
// instance b's attention view (layout, instance-local rows, attention scratch,
// summary).  Instance b's merged KV is rows [b*Tp, b*Tp + T) of `kv`.
struct Batch {
    Pass all;
    std::vector<std::unique_ptr<Pass>> views;
    DevBuf kv;                        // [2][B*Tp][dl] merged KV of the current layer
    DevBuf tokens, iota, last_idx, last_x, logits;
    DevBuf sel_order, sel_cand, sel_ptrs, walk_host;
    DevBuf stage;                        // host memory: a ring of staged layer sheets [K|V][Tm + pad][dl]
    std::vector<cudaEvent_t> ev_load;    // per slot: sheet loaded (copy stream)
    std::vector<cudaEvent_t> ev_used;    // per slot: the sheet's readers are done (compute stream)
    ~Batch() {
        for (auto e : ev_load) if (e) cudaEventDestroy(e);
        for (auto e : ev_used) if (e) cudaEventDestroy(e);
    }
};

struct Context {
    keep_config cfg{};
    int L = 0, H = 0, d = 0, dh = 0, f = 0, V = 0;
    // KV-head sharding: this rank owns heads [R*Hl, (R+1)*Hl), i.e. the
    // q/k/v/ctx columns [R*dl, (R+1)*dl); G = 1 is the single-GPU path
    int G = 1, R = 0, Hl = 0, dl = 0;
    std::unique_ptr<Comm> comm;
    bool fast = false;
    bool exact = false;  // KEEP_NUMERICS_PARITY_EXACT: DFMA projections + reference-order scores
    double rope_theta = 0.0;  // keep_set_rope: 0 = NoPE, the reference (model.hpp:3-8)
    uint64_t hbm_budget = 0;  // keep_memory_residency: HBM capacity for pinned-host memory layers
    std::vector<std::shared_ptr<Arena>> load_hold;  // sources of in-flight asynchronous loads
    DevBuf d_live, d_next;                          // single-hop ablation: live mask in, kept mask out
    int elem = 4;  // merged-KV element bytes
    cudaStream_t s_main = nullptr, s_copy = nullptr, s_sel = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    bool weights_ready = false;
    DevBuf embed, unembed;
    std::vector<std::unique_ptr<DevBuf>> w;  // L*4 slots
    // memory tier
    std::map<OwnerKey, Payload> store;
    std::map<OwnerKey, uint64_t> current_version;
    keep_memory_stats stats{};
    // cursor
    std::unique_ptr<Pass> pf;
    std::unique_ptr<Batch> batch;   // batched multi-query prefill workspace
    std::unique_ptr<Pass> refresh;  // canonical-KV refresh workspace
    DevBuf refresh_ws;               // in-place refresh: merged KV of the refreshed owners
    DevBuf kv;  // merged KV of the cursor [L][2][T][d]
    std::vector<void*> seg_ksrc_h, seg_vsrc_h;
    DevBuf d_ksrc, d_vsrc, d_cdst, d_cn, d_bytes;
    Arena* alias_arena = nullptr;         // layout == one in-order HBM arena (all-reused layers run on it)
    std::shared_ptr<Arena> alias_hold;
    std::vector<OwnerKey> seg_owner;      // owner of each layout segment
    std::vector<const Payload*> seg_pl;   // its payload (resolved at prefill begin)
    std::vector<uint64_t> seg_cur;        // and its current version
    uint64_t store_gen = 0, seg_gen = 0;  // memory-store mutations / generation resolved
    std::vector<int64_t> seg_owner_row;   // row offset of the segment in the owner block
    // selector scratch
    DevBuf sel_order, sel_n, sel_cand;
    DevBuf logits;
    DevBuf walk_host;                     // pinned walk result (plan_keep)
    std::vector<cudaEvent_t> pk_evs;      // plan_keep layer events
    cudaEvent_t ev_sum = nullptr, ev_sel = nullptr;
    Profiler prof;
    Loader loader;
    OzWork oz;  // PARITY Ozaki GEMM scratch
    int gemm_ctas = kNumSMs;  // 147 while the selector overlaps the MLP

    void* wslot(int l, int slot) const { return w[l * 4 + slot]->p; }
};

}  // namespace keep_b200
