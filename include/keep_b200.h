/*
 * keep_b200.h -- C ABI of the B200-native KEEP per-layer memory prefill.
 *
 * The drop-in boundary for the reference's hot path.
 * Plain C types only (no torch, no C++ in the signatures); every entry point
 * returns an int status (KEEP_OK or one of the error codes below, mirroring the
 * reference's exception taxonomy, errors.hpp:8-26) and keep_last_error()
 * returns the thread-local message of the last failure.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   keep_model_init            Model::init                  include/keep/model.hpp:54-73
 *   keep_memory_put            CacheManager::put            include/keep/cache_manager.hpp:69-99
 *   keep_memory_compute        EpisodeRuntime::compute_and_put (segment_prefill /
 *                              joint full_prefill)          include/keep/harness.hpp:512-532
 *   keep_load_memory           CacheManager::load           include/keep/cache_manager.hpp:103-130
 *                              (paper: load_memory(memory_id, layer_id))
 *   keep_memory_has_current    CacheManager::has_current    include/keep/cache_manager.hpp:151-159
 *   keep_invalidate            CacheManager::invalidate     include/keep/cache_manager.hpp:163-184
 *   keep_prefill_begin         PrefillCursor::PrefillCursor include/keep/prefill.hpp:174-217
 *   keep_prefill_layer         PrefillCursor::step          include/keep/prefill.hpp:224-322
 *                              (paper: prefill_layer(input, layer_id, kv))
 *   keep_prefill_finish        PrefillCursor::finish        include/keep/prefill.hpp:324-337
 *   keep_importance_evaluation converge                     include/keep/recompute.hpp:130-138
 *                              (paper: importance_evaluation(...))
 *   keep_plan_keep             plan_keep                    include/keep/recompute.hpp:140-180
 *   keep_ratio_schedule        ratio_schedule               include/keep/recompute.hpp:33-70
 *   keep_layer_budget          layer_budget                 include/keep/recompute.hpp:73-77
 *   keep_logits                Model::logits                include/keep/model.hpp:76-85
 *   keep_divergence            divergence                   include/keep/prefill.hpp:501-531
 *
 * Threading: a context is single-threaded and stateful like the cursor and
 * the cache manager it replaces; distinct contexts may be
 * used from distinct threads.  All device work runs on the context's own
 * CUDA streams; calls return after the work they report has completed.
 *
 * Numerics (keep_config.numerics):
 *   KEEP_NUMERICS_PARITY  fp32 storage, fp64-grade accumulation on the tensor
 *                         cores: Ozaki-II int8 projections (exact integer
 *                         products of 47-bit scaled operands, one rounding to
 *                         fp32), fp64 DMMA attention / softmax / summaries.
 *                         Selections are bit-exact with the reference.
 *   KEEP_NUMERICS_PARITY_EXACT  projections bit-exact with vec_mat (DFMA in
 *                         ascending k) and scores in the reference's
 *                         dimension order: the arbiter of PARITY.
 *   KEEP_NUMERICS_FAST    bf16 operands on the sm_100a tensor cores (tcgen05)
 *                         with fp32 accumulation, fp32 residual stream, bf16
 *                         merged KV, fp32 probabilities with fp64 summary
 *                         reduction.  Selections agree with the reference
 *                         except at near-ties; see DESIGN.md.
 */
#ifndef KEEP_B200_H
#define KEEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

enum {
    KEEP_OK = 0,
    KEEP_ERR_CONFIG = 1,     /* ConfigError    */
    KEEP_ERR_INPUT = 2,      /* InputError     */
    KEEP_ERR_PLAN = 3,       /* PlanError      */
    KEEP_ERR_CACHE_MISS = 4, /* CacheMissError */
    KEEP_ERR_TRACE = 5,      /* TraceError     */
    KEEP_ERR_CUDA = 6,       /* CUDA / NCCL / out of memory */
};

/* PARITY: the reference's arithmetic (fp32 storage, fp64-grade accumulation)
 *   on the tensor cores -- Ozaki int8 projections, fp64 DMMA attention;
 * FAST: bf16 tcgen05, fp32 accumulation (selections not guaranteed);
 * PARITY_EXACT: projections bit-exact with vec_mat (DFMA, ascending k) and
 *   scores in the reference's dimension order (scalar fp64 attention). */
enum { KEEP_NUMERICS_PARITY = 0, KEEP_NUMERICS_FAST = 1, KEEP_NUMERICS_PARITY_EXACT = 2 };

/* Memory owner (OwnerRef, memory_store.hpp:61-88): a dynamic segment owns
 * per-segment blocks, a static group owns one joint block per layer. */
enum { KEEP_OWNER_SEGMENT = 0, KEEP_OWNER_GROUP = 1 };
/* Tiers: device HBM (fast) or pinned host DRAM (slow). */
enum { KEEP_TIER_DEVICE = 0, KEEP_TIER_HOST = 1 };

typedef struct {
    int32_t num_layers, num_heads, model_dim, mlp_dim, vocab_size;
    int32_t numerics;    /* KEEP_NUMERICS_* */
    uint64_t seed;       /* ModelConfig::seed */
    int32_t device;      /* CUDA ordinal */
    int32_t world_size;  /* KV-head shards G (1 = single GPU); num_heads % G == 0 */
    int32_t rank;        /* this context owns heads [rank*H/G, (rank+1)*H/G) */
    int32_t max_hops;    /* converge hop cap (BASELINE configs[3] "3-hop recompute"); 0 = the
                            reference's uncapped walk (recompute.hpp:130-138) */
    /* world_size > 1: exactly one of the following (see keep_comm_unique_id) */
    const uint8_t* nccl_id; /* 128-byte ncclUniqueId shared by all ranks (library-owned comm) */
    void* nccl_comm;        /* caller-owned ncclComm_t */
    void* loopback;         /* keep_loopback_create group: G ranks on one GPU in one process
                               (one host thread per rank; a test double for the collectives) */
} keep_config;

typedef struct {
    int32_t kind; /* KEEP_OWNER_* */
    uint32_t id;
} keep_owner;

typedef struct {
    int32_t num_segments;
    int32_t num_units;            /* 0 => one dynamic unit per segment, owner s<position> */
    const int32_t* seg_len;       /* [S] tokens per segment, >= 1 */
    const int32_t* tokens;        /* [sum seg_len] concatenated in layout order */
    const int32_t* unit_begin;    /* [num_units] first segment position of the unit */
    const int32_t* unit_end;      /* [num_units] one past the last */
    const keep_owner* unit_owner; /* [num_units] owner of the unit's cached KV */
} keep_layout;

/* Borrowed view of one (owner, layer) KV block: keys then values, each
 * [tokens x d] row-major; element type fp32 (PARITY) or bf16 (FAST).  Device
 * pointers, valid until the block is replaced or invalidated. */
typedef struct {
    void* keys;
    void* values;
    int64_t tokens;
    int32_t tier;        /* tier the block was found in before the load */
    int32_t elem_bytes;  /* 4 or 2 */
    double load_ms;      /* measured H2D time of a slow-tier load (0 for fast hits) */
    int32_t row_elems;   /* elements per row: model_dim / world_size (this rank's head columns) */
    int32_t col0;        /* first model column of the row slice */
} keep_kv_view;

typedef struct {
    uint64_t bytes_loaded_slow;
    uint64_t cache_misses;
    uint64_t tokens_invalidated;
    uint64_t blocks;
    uint64_t device_bytes;
    uint64_t host_bytes;
} keep_memory_stats;

/* Per-run outputs of keep_plan_keep.  Any pointer may be NULL. */
typedef struct {
    uint8_t* plan;          /* [L*S] plan[l*S+i] = segment position i recomputed at layer l */
    int32_t* orders;        /* [L*S] relevant_order of the walk after layer l */
    int32_t* order_len;     /* [L] walk length, -1 when the layer kept every live segment */
    int32_t* hops;          /* [L] ImportanceState::hop of that walk */
    double* summaries;      /* [L*(S+S*S)] per layer qts then sts (prefill.hpp:76-80) */
    float* final_hidden;    /* [T*d] (prefill.hpp:324-337) */
    double* last_logits;    /* [V] Model::logits of the last row (model.hpp:76-85) */
    int64_t* rows_per_layer;/* [L] N_act(l): recomputed rows (active segments + query) */
    double* layer_ms;       /* [L] device time per layer (CUDA events) */
    double ttft_ms;         /* device time begin -> last-row logits */
} keep_plan_result;

const char* keep_last_error(void);
const char* keep_version(void);

/* ---- KV-head sharding ----------------------------------
 * One context per rank.  Every rank calls the same sequence of entry points;
 * per layer the ranks all-reduce the fp64 segment summary (identical bits on
 * every rank, so importance_evaluation runs replicated), exchange attention
 * context head-sharded -> row-sharded (all-to-all) and all-gather the fp32
 * residual rows after Wo + MLP.  KV blocks, views and kv_out hold the rank's
 * head columns only (row_elems = model_dim / world_size). */
int keep_comm_unique_id(uint8_t* id_out /* 128 bytes */);
/* The partition every rank applies (host functions, no device work):
 * heads [h0, h0+hn) and model columns [c0, c0+cn) of `rank`; and this
 * rank's block [r0, r0+m) of n compact rows for Wo + MLP (equal blocks of
 * ceil(n / world) rows, the all-gather unit). */
int keep_shard_heads(int32_t num_heads, int32_t model_dim, int32_t world_size, int32_t rank,
                     int32_t* h0, int32_t* hn, int32_t* c0, int32_t* cn);
int keep_shard_rows(int64_t n, int32_t world_size, int32_t rank, int64_t* r0, int64_t* m);
int keep_loopback_create(int32_t world_size, void** group_out);
int keep_loopback_destroy(void* group);

int keep_ctx_create(const keep_config* cfg, void** ctx_out);
int keep_ctx_destroy(void* ctx);
/* Release the grow-only prefill / batch / refresh workspaces (memory store and
 * weights stay); they grow back on the next call. */
int keep_ctx_trim(void* ctx);
int keep_ctx_synchronize(void* ctx);

/* Reference-identical counter-based weights generated on the device. */
int keep_model_init(void* ctx);
/* Copy the weights back in the reference layout (fp32; oracle/keep_oracle.h). */
int keep_model_export(void* ctx, float* host_weights, uint64_t count);

/* ---- memory tier: the load_memory surface ------------------------------ */
/* keys / values: full rows [tokens x model_dim] (a sharded rank keeps its
 * head columns). */
int keep_memory_put(void* ctx, keep_owner owner, uint64_t version, int32_t layer,
                    int64_t tokens, const float* keys, const float* values, int32_t tier);
/* Canonical KV refresh on the GPU for every layer: one standalone prefill per
 * segment (owner kind SEGMENT, n_members must be 1) or one joint prefill over
 * the members (kind GROUP).  The result is stored under (owner, version). */
int keep_memory_compute(void* ctx, keep_owner owner, uint64_t version, int32_t n_members,
                        const int32_t* member_len, const int32_t* tokens, int32_t tier);
/* Batched refresh of many owners in one set of launches (same semantics). */
int keep_memory_compute_batch(void* ctx, int32_t n_owners, const keep_owner* owners,
                              const uint64_t* versions, const int32_t* owner_members,
                              const int32_t* member_len, const int32_t* tokens, int32_t tier);
int keep_load_memory(void* ctx, keep_owner owner, int32_t layer, keep_kv_view* out);
/* The asynchronous form: the slow-tier copy is enqueued on
 * the context's copy stream and the view returned at once; *done (a
 * cudaEvent_t) completes when the block is in HBM -- wait on it
 * (cudaStreamWaitEvent / keep_load_wait) before reading the view.  The event
 * is the context's: valid until its next load. */
int keep_load_memory_async(void* ctx, keep_owner owner, int32_t layer, keep_kv_view* out, void** done);
int keep_load_wait(void* ctx);
int keep_memory_has_current(void* ctx, keep_owner owner, uint64_t version, int32_t* out);
int keep_invalidate(void* ctx, keep_owner owner, uint64_t new_version, uint64_t tokens);
int keep_memory_stats_get(void* ctx, keep_memory_stats* out);
/* Drop every block, owner version and statistic: a fresh CacheManager
 * (cache_manager.hpp:62-66; harness.hpp:490-497 builds one per episode). */
int keep_memory_clear(void* ctx);
/* Capacity-bounded fast tier (CacheManager's fast_capacity_bytes,
 * cache_manager.hpp:23-35): keep the deepest layers of every pinned-host arena
 * also resident in HBM, as many as fit in hbm_budget_bytes (plans only shrink
 * with depth, so deep layers reuse the most cached KV).  Those layers are
 * then fast-tier hits and never loaded; a write to an arena drops its copy.
 * 0 releases them. */
int keep_memory_residency(void* ctx, uint64_t hbm_budget_bytes, uint64_t* resident_bytes);
/* dims[7] = {num_layers, num_heads, model_dim, mlp_dim, vocab_size, numerics, world_size} */
int keep_ctx_dims(void* ctx, int32_t* dims);
/* Copy one block back to the host as fp32 (tests): [tokens x row_elems]. */
int keep_memory_read(void* ctx, keep_owner owner, int32_t layer, float* keys, float* values);

/* ---- prefill cursor: prefill_layer ------------------------------------- */
int keep_prefill_begin(void* ctx, const keep_layout* layout, const int32_t* query,
                       int32_t query_len);
/* One layer.  active[S] host mask; summary_out (S+S*S doubles) may be NULL. */
int keep_prefill_layer(void* ctx, const uint8_t* active, double* summary_out);
/* final_hidden [T*d] fp32; kv_out per layer keys[T*dc] then values[T*dc] as
 * fp32 (converted from bf16 in FAST), dc = model_dim / world_size (the rank's
 * head columns).  Either may be NULL. */
int keep_prefill_finish(void* ctx, float* final_hidden, float* kv_out);

/* ---- selection ----------------------------------------------------------- */
int keep_importance_evaluation(void* ctx, int32_t S, const double* qts, const double* sts,
                               int64_t budget, const uint8_t* candidates, int32_t* order_out,
                               int32_t* n_out, int32_t* hops_out);
int keep_ratio_schedule(int32_t num_layers, double r_avg, double* r_out);
int64_t keep_layer_budget(double ratio, int64_t num_segments);

/* ---- the whole KEEP per-layer loop (plan_keep) on the device ------------ */
int keep_plan_keep(void* ctx, const keep_layout* layout, const int32_t* query,
                   int32_t query_len, const double* schedule, int32_t multihop,
                   keep_plan_result* out);

/* ---- batched multi-query prefill ----------------------
 * B planning queries over one memory layout, each with its own plan and
 * result exactly as keep_plan_keep(layout, queries[b]) would produce
 * (PARITY: bit-identical).  Shared work: layer 0's memory rows are computed
 * once (plan[0] is every segment for every query, and memory rows precede
 * the query); the projections of all instances run as one GEMM per layer;
 * all-reused layers of any instance read the in-order arena in place; the
 * first-token logits of all instances stream the unembedding once.
 * queries: [B x query_len]; outs: [B] (ttft_ms = the whole batch's device
 * time; layer_ms per layer of the batch).  One GPU (G = 1), HBM-resident
 * memory. */
int keep_plan_keep_batch(void* ctx, const keep_layout* layout, int32_t batch, const int32_t* queries,
                         int32_t query_len, const double* schedule, int32_t multihop, keep_plan_result* outs);
/* The same batch with given monotone plans [batch x L x S] (every segment at
 * layer 0) instead of the walks: selective_prefill (prefill.hpp:478-497) per
 * query. */
int keep_selective_prefill_batch(void* ctx, const keep_layout* layout, int32_t batch, const int32_t* queries,
                                 int32_t query_len, const uint8_t* plans, keep_plan_result* outs);

int keep_logits(void* ctx, const float* row, double* out);
/* divergence (prefill.hpp:501-531): L2 of two final rows and the symmetric
 * KL of their softmaxed logits (fp64, the reference's formula). */
int keep_divergence(void* ctx, const float* row_a, const float* row_b, double* l2, double* sym_kl);

/* ---- K10 loader trace: the realised (layer, owner) load schedule of the
 * last prefill over pinned-host owners, for the reference's timeline rules
 * (pipeline_sim.hpp:340-428: D1 loads of layer l end before compute(l); P each
 * workload item loaded once with its block bytes; S pre-loads only of owners
 * whose members all left the plan).  Times in ms from the prefill start. */
typedef struct {
    int32_t layer;        /* the item's layer */
    int32_t kind;         /* 0 urgent (before compute(layer)), 1 ahead (layer = at_layer + 1), 2 pre-load */
    int32_t at_layer;     /* issued before compute(at_layer) (urgent) or behind it */
    keep_owner owner;
    uint64_t bytes;       /* K + V block bytes of this rank */
    double batch_start_ms, batch_end_ms;  /* the copy batch that carried it */
    double compute_start_ms;              /* compute(layer) start on the compute stream */
} keep_load_record;
int keep_loader_trace(void* ctx, keep_load_record* out, int32_t cap, int32_t* n_out);

/* The realised timeline of the last keep_plan_keep over pinned-host owners as
 * the reference's Timeline (pipeline_sim.hpp:69-92), for validate_timeline
 * (340-428: R one event per resource at a time, D1, D2, P, S): kind 0 load
 * (one (layer, owner) item; a copy batch's interval is shared out to its items
 * in byte order), 1 compute(layer) on the compute stream, 2 eval(layer) = the
 * walk on the selector stream.  *attention_fraction = the smallest
 * (attention + summary done - compute start) / compute span over the walked
 * layers.  Times in ms from the prefill start. */
typedef struct {
    int32_t kind;
    int32_t layer;
    keep_owner owner; /* loads */
    uint64_t bytes;   /* loads */
    double start_ms, end_ms;
} keep_timeline_event;
int keep_timeline_trace(void* ctx, keep_timeline_event* out, int32_t cap, int32_t* n_out, double* attention_fraction);

/* ---- per-phase device timing (CUDA events on the launching streams) ----- */
enum {
    KEEP_PROF_QKV = 0,      /* gathered QKV GEMM + K/V scatter (K3)          */
    KEEP_PROF_ATTN = 1,     /* attention + segment binning (K5)              */
    KEEP_PROF_WO = 2,       /* Wo GEMM + residual (K8)                       */
    KEEP_PROF_MLP_IN = 3,   /* MLP in + ReLU (K9a)                           */
    KEEP_PROF_MLP_OUT = 4,  /* MLP out + residual (K9b)                      */
    KEEP_PROF_SUMMARY = 5,  /* row bins -> segment summary (K6)              */
    KEEP_PROF_SELECT = 6,   /* multi-hop selector (K7)                       */
    KEEP_PROF_CACHED = 7,   /* merged-KV assembly from cached blocks (K4)    */
    KEEP_PROF_COMPACT = 8,  /* active-row compaction (K2)                    */
    KEEP_PROF_EMBED = 9,    /* embedding gather (K1)                         */
    KEEP_PROF_LOGITS = 10,  /* last-row logits (K11)                         */
    KEEP_PROF_LOADER = 11,  /* host->HBM layer loads (K10)                   */
    KEEP_PROF_COMM = 12,    /* KV-head sharding collectives (NCCL)           */
    KEEP_PROF_XCHG = 13,    /* ctx pack / residual bf16 refresh around them  */
    KEEP_PROF_REFRESH = 14, /* canonical-KV refresh of updated owners (whole call) */
    KEEP_PROF_DECODE = 15,  /* few-row attention without a summary (K5d, flash decoding) */
    KEEP_PROF_COUNT = 16
};
typedef struct {
    double ms[16];          /* summed device time                          */
    double flops[16];       /* algorithmic FLOPs                           */
    double bytes[16];       /* algorithmic HBM bytes                       */
    int64_t launches[16];   /* timed regions (one per phase per layer)     */
    int64_t kernels[16];    /* kernel launches inside them                 */
} keep_profile;
int keep_profile_enable(void* ctx, int32_t on);
int keep_profile_read(void* ctx, keep_profile* out, int32_t reset);

/* ---- RoPE position re-shift (north_star subsystem 3; off by default) -----
 * The reference is NoPE (model.hpp:3-8): theta = 0 keeps it, and
 * every parity run uses 0.  theta > 0 applies rotary embeddings to q and k
 * (pairs (2j, 2j+1) per head, angle pos * theta^(-2j/dh)); canonical KV is
 * rotated at owner-local positions and a reused block's keys are re-shifted by
 * its layout offset when merged.  Single GPU, HBM-resident memory, single
 * query (keep_plan_keep / the cursor); no oracle exists for it. */
int keep_set_rope(void* ctx, double theta);

/* ---- test hook (not part of the reference surface) ----------------------
 * C[M x N] (fp32, device) = A[M x K] . Bt[N x K]^T with bf16 device operands
 * on the tcgen05 GEMM; force_bn 0 = automatic tile, 64 or 256 = forced. */
int keep_debug_gemm_bf16(const void* A, const void* Bt, float* C, int M, int N, int K, int force_bn);
/* C[M x N] (fp32, device) = A[M x K] . B[K x N] with fp32 device operands on
 * the PARITY GEMM: mode 0 automatic, 1 the Ozaki int8 tensor-core GEMM,
 * 2 the DFMA (vec_mat bit-exact) kernel. */
int keep_debug_gemm_parity(const float* A, const float* B, float* C, int M, int N, int K, int mode);
/* Test hook: y[i] = the PARITY softmax's fp64 exp (f64_exp.cuh) of x[i], device pointers. */
int keep_debug_exp_f64(const double* x, double* y, int64_t n);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* KEEP_B200_H */
