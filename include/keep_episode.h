/* keep_episode.h -- the memory control plane and episode replay (SURVEY.md
 * 8(f4)) on top of the B200 prefill engine (keep_b200.h).
 *
 * Reference interface each entry point replaces (/root/reference/proj/):
 *
 *   keep_trace_generate   generate_episode            include/keep/harness.hpp:362-413
 *   keep_store_*          MemoryStore                 include/keep/memory_store.hpp:274-496
 *                         (cluster_segments 240-272, apply_update 309-341,
 *                          advance_step 343-367, retrieve 372-418,
 *                          add_segment 420-452, state_sound 456-468)
 *   keep_run_episode      run_episode                 include/keep/harness.hpp:543-817
 *   keep_compare_csv      compare_csv                 include/keep/harness.hpp:828-871
 *   keep_report_json      report_to_json              include/keep/harness.hpp:449-484
 *
 * The store, the tier accounting (CacheManager's capacity / LRU / version
 * bookkeeping, cache_manager.hpp:60-228) and the load/compute pipeline model
 * (pipeline_sim.hpp:103-428) are host C++ bookkeeping.  Every tensor the
 * episode touches lives on the GPU: canonical KV is computed by
 * keep_memory_compute_batch into the device memory tier, plans come from
 * keep_plan_keep, selective and full prefills run through the cursor and the
 * divergence through keep_divergence.  Nothing here computes on the CPU.
 *
 * Return codes and keep_last_error() as in keep_b200.h.
 */
#ifndef KEEP_EPISODE_H
#define KEEP_EPISODE_H

#include <stdint.h>

#include "keep_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* CategorySpec (harness.hpp:38-43) */
typedef struct {
    const char* name;
    int32_t count;
    int32_t tokens_per_segment;
    double update_prob_per_step;
} keep_category;

/* EpisodeConfig (harness.hpp:53-104): store / model / cost / tier / ablation
 * flattened.  The model fields must equal the context's (keep_ctx_dims). */
enum { KEEP_GROUPING_SEMANTIC = 0, KEEP_GROUPING_FIXED = 1 };
enum { KEEP_SCHEDULE_DEFAULT = -1, KEEP_SCHEDULE_SEQUENTIAL = 0, KEEP_SCHEDULE_OVERLAP = 1,
       KEEP_SCHEDULE_BALANCED = 2 };
typedef struct {
    uint64_t seed;
    int32_t num_segments, num_steps, retrieval_k;
    double r_avg;
    int32_t query_tokens, embedding_dim, fixed_pos_edge_tokens;
    int32_t store_t, store_num_groups;
    uint64_t store_seed;            /* 0 => seed (EpisodeRuntime::store_config) */
    int32_t num_layers, num_heads, model_dim, mlp_dim, vocab_size;
    uint64_t model_seed;
    double compute_tu_per_token_per_layer, eval_tu_per_layer, attention_fraction;
    uint64_t fast_capacity_bytes, fast_bandwidth_bytes_per_tu, slow_to_fast_bandwidth_bytes_per_tu;
    int32_t n_categories;
    const keep_category* categories;
    int32_t grouping;               /* KEEP_GROUPING_* */
    int32_t multihop;               /* AblationFlags::multihop */
    int32_t balanced_loading;       /* AblationFlags::balanced_loading */
    int32_t schedule_override;      /* KEEP_SCHEDULE_* */
} keep_episode_config;

/* TraceEvent (harness.hpp:117-127).  Pointers are borrowed. */
enum { KEEP_EVENT_INIT_SEGMENT = 0, KEEP_EVENT_UPDATE = 1, KEEP_EVENT_QUERY = 2 };
typedef struct {
    int32_t type;
    int64_t step;
    uint32_t id;
    const char* category;           /* init-segment */
    int32_t n_tokens;               /* init-segment, update */
    const int32_t* tokens;
    int32_t embedding_dim;          /* init-segment */
    const double* embedding;
    uint64_t embedding_seed;        /* query */
    int32_t k;                      /* query */
} keep_trace_event;

int keep_trace_generate(const keep_episode_config* cfg, void** trace_out);
/* Copies the events; checks what trace_from_jsonl checks (harness.hpp:301-322). */
int keep_trace_create(int32_t n_events, const keep_trace_event* events, void** trace_out);
int keep_trace_size(void* trace, int32_t* n_events);
int keep_trace_event_get(void* trace, int32_t i, keep_trace_event* out);
int keep_trace_destroy(void* trace);

/* ---- MemoryStore (memory_store.hpp:274-496) ------------------------------ */
typedef struct {
    uint32_t id;
    const char* category;
    int32_t n_tokens;
    const int32_t* tokens;
    int32_t embedding_dim;
    const double* embedding;        /* unit norm */
} keep_segment;
typedef struct {                    /* StoreConfig (memory_store.hpp:47-57) */
    int32_t t, num_groups;
    uint64_t seed;
    int32_t grouping;               /* KEEP_GROUPING_* */
} keep_store_config;
int keep_store_create(int32_t n, const keep_segment* segments, const keep_store_config* cfg, void** store_out);
int keep_store_destroy(void* store);
/* groups: n_out groups; member ids concatenated into members (cap entries),
 * counts[g], state[g] (1 static), group_version[g].  Any output may be NULL. */
int keep_store_groups(void* store, int32_t* n_out, int32_t cap, uint32_t* members, int32_t* counts,
                      int32_t* state, uint64_t* group_version);
/* InvalidationRecord: owners[n] with their tokens; the segment's new version. */
int keep_store_apply_update(void* store, uint32_t id, int32_t n_tokens, const int32_t* tokens, int64_t step,
                            int32_t cap, keep_owner* owners, uint64_t* tokens_out, int32_t* n_out,
                            uint64_t* new_version);
/* GroupTransitions of this step: group ids and their new versions. */
int keep_store_advance_step(void* store, int64_t step, int32_t cap, uint32_t* groups, uint64_t* versions,
                            int32_t* n_out);
/* RetrievalSet: units in canonical order (groups by id, then segments). */
int keep_store_retrieve(void* store, const double* query_embedding, int32_t dim, int32_t k, int32_t cap,
                        keep_owner* units, int32_t* unit_segments, int32_t seg_cap, uint32_t* segments,
                        int32_t* n_units);
int keep_store_add_segment(void* store, const keep_segment* segment, int64_t step);
int keep_store_state_sound(void* store, int32_t* out);

/* ---- episode replay ------------------------------------------------------- */
/* StepReport (harness.hpp:419-433) + the measured host wall time of the
 * step's GPU work (refresh, plan, prefills, divergence). */
typedef struct {
    int64_t step;
    int64_t realized_segments;
    double ttft_tu, makespan_tu, refresh_tu, div_l2, div_kl;
    double reused_tokens, recomputed_tokens, memory_tokens;
    uint64_t invalidated_tokens_delta, bytes_loaded_slow_delta;
    int32_t num_layers;
    const int64_t* plan_sizes;      /* [num_layers], borrowed from the report */
    double wall_ms;
} keep_step_report;
/* StrategyReport aggregate (harness.hpp:435-447) */
typedef struct {
    int32_t steps;
    double mean_ttft_tu, p95_ttft_tu, mean_div_l2, mean_div_kl, reuse_ratio, mean_realized_segments;
    uint64_t invalidated_tokens, bytes_slow;
} keep_strategy_aggregate;

/* strategy: "full", "prefix", "full-reuse", "fixed-pos", "deviation", "keep"
 * (recompute.hpp:337-357).  The context's memory tier is cleared first. */
int keep_run_episode(void* ctx, void* trace, const char* strategy, const keep_episode_config* cfg,
                     void** report_out);
int keep_report_aggregate(void* report, keep_strategy_aggregate* out);
int keep_report_step(void* report, int32_t i, keep_step_report* out);
/* report_to_json text; *len = bytes needed (without the NUL). */
int keep_report_json(void* report, char* buf, uint64_t cap, uint64_t* len);
int keep_report_destroy(void* report);
/* compare_csv: one row per (strategy, sweep point); ks / rs may be empty. */
int keep_compare_csv(void* ctx, void* trace, int32_t n_strategies, const char* const* strategies,
                     const keep_episode_config* cfg, int32_t n_k, const int32_t* ks, int32_t n_r,
                     const double* rs, char* buf, uint64_t cap, uint64_t* len);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif
