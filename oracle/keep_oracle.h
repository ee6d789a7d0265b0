/*
 * keep_oracle.h -- CPU oracle API for the KEEP per-layer memory prefill.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library in
 * paper_2602_23592_b200/) may include, link or call this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it, and only as the checker or as the timed CPU baseline.
 *
 * Two implementations export this exact API with different prefixes:
 *   ko_*  oracle/keep_oracle.c   -- a plain-C restatement of the reference
 *                                   algorithm (every function cites the
 *                                   reference file:line it restates);
 *   kr_*  oracle/ref_shim.cpp    -- a thin C wrapper that calls the UNMODIFIED
 *                                   reference headers under
 *                                   /root/reference/proj/include (built into
 *                                   oracle/_ref/, never committed).
 * The restatement is pinned against the reference shim and against the golden
 * vectors in tests/golden/ (generated from the shim by
 * tests/golden/make_golden.py).
 *
 * Conventions (shared with the CUDA product so buffers can be compared):
 *  - weights: one fp32 buffer laid out as
 *      embed[V*d], unembed[d*V], then per layer l:
 *      wq[d*d], wk[d*d], wv[d*d], wo[d*d], mlp_in[d*mlp], mlp_out[mlp*d]
 *    all row-major, exactly the reference Mat layout (tensor.hpp:13-28,
 *    model.hpp:41-45).
 *  - a "problem" is a model config + a layout of S segments (concatenated
 *    tokens, per-segment lengths) + retrieval units + a query.  Unit u covers
 *    segment positions [unit_begin[u], unit_end[u]); unit_is_group[u] != 0
 *    means a static group whose canonical KV is ONE joint prefill over its
 *    members (harness.hpp:520-531), otherwise each segment of the unit has its
 *    own standalone KV (segment_prefill, prefill.hpp:472-476).  n_units == 0
 *    means one dynamic unit per segment (Layout::of, prefill.hpp:48-54).
 *  - summaries: per layer S doubles query_to_segment followed by S*S doubles
 *    segment_to_segment (row = source segment), prefill.hpp:76-80.
 *  - kv: per layer keys[T*d] then values[T*d] (merged KV, prefill.hpp:71-74).
 *  - plan: L*S bytes, plan[l*S+i] = 1 if segment position i is recomputed at
 *    layer l (RecomputePlan, prefill.hpp:91-112, by position).
 *  - return codes: 0 ok, 1 ConfigError, 2 InputError, 3 PlanError,
 *    4 CacheMissError, 5 TraceError, 9 internal (errors.hpp:8-26).
 */
#ifndef KEEP_ORACLE_H
#define KEEP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t num_layers, num_heads, model_dim, mlp_dim, vocab_size;
    int32_t pad_;
    uint64_t seed;
    int32_t num_segments;
    int32_t query_len;
    const int32_t* seg_len;      /* [S] */
    const int32_t* tokens;       /* [sum seg_len] */
    const int32_t* query;        /* [query_len] */
    int32_t num_units;           /* 0 => one dynamic unit per segment */
    int32_t pad2_;
    const int32_t* unit_begin;   /* [num_units] */
    const int32_t* unit_end;     /* [num_units] */
    const int32_t* unit_is_group;/* [num_units] */
} keep_problem;

#define KEEP_ORACLE_API(P)                                                              \
    uint64_t P##weight_count(int L, int H, int d, int mlp, int V);                      \
    int P##model_init(int L, int H, int d, int mlp, int V, uint64_t seed, float* w);   \
    int P##make_instance_layout(uint64_t seed, int S, int V, int lo, int hi, int qlen, \
                                int32_t* seg_len, int32_t* tokens, int32_t* query);    \
    int P##ratio_schedule(int L, double r_avg, double* r_out);                          \
    int64_t P##layer_budget(double ratio, int64_t S);                                   \
    int P##converge(int S, const double* qts, const double* sts, int64_t budget,        \
                    const uint8_t* candidates, int32_t* order_out, int32_t* n_out,     \
                    int32_t* hops_out);                                                 \
    int P##canonical_kv(const keep_problem* p, const float* w, float* kv_out);          \
    int P##full_prefill(const keep_problem* p, const float* w, float* final_hidden,     \
                        float* kv, double* summaries);                                  \
    int P##selective_prefill(const keep_problem* p, const float* w, const float* cached,\
                             const uint8_t* plan, float* final_hidden, float* kv,       \
                             double* summaries);                                        \
    int P##plan_keep(const keep_problem* p, const float* w, const float* cached,        \
                     const double* sched, int multihop, uint8_t* plan,                  \
                     int32_t* orders, int32_t* order_len, int32_t* hops,                \
                     double* summaries, float* final_hidden, float* kv);                \
    int P##divergence(const keep_problem* p, const float* w, const float* row_a,        \
                      const float* row_b, double* l2, double* sym_kl);                  \
    int P##logits(const keep_problem* p, const float* w, const float* row, double* out);

/* cached: the canonical KV of the memory rows, per layer keys[Tm*d] then
 * values[Tm*d] with Tm = sum(seg_len) (row r of the layout = row r here), as
 * produced by *canonical_kv.  NULL => computed internally from the units. */

KEEP_ORACLE_API(ko_)
KEEP_ORACLE_API(kr_)

/* The reference's validate_timeline (pipeline_sim.hpp:340-428) over a realised
 * timeline; kr_ only (it is the reference's own checker).  kind: 0 load,
 * 1 compute, 2 eval.  slow_bytes: [n_units x L] bytes of each unit's block in
 * the slow tier (0 = fast-resident / absent). */
typedef struct {
    int32_t kind, layer;
    int32_t owner_kind; /* 0 segment, 1 group */
    uint32_t owner_id;
    uint64_t bytes;
    double start, end;
} kr_timeline_event;
int kr_validate_timeline(int L, int S, const uint8_t* plan, const int32_t* seg_len, int query_tokens, int n_units,
                         const int32_t* unit_begin, const int32_t* unit_end, const int32_t* unit_is_group,
                         const uint32_t* unit_owner_id, const uint64_t* slow_bytes, double attention_fraction,
                         const kr_timeline_event* ev, int n_ev, char* codes_out, int cap);

const char* ko_last_error(void);
/* restatement-only extension: cap converge at max_hops hops (0 = the
 * reference's uncapped walk); see keep_oracle.c */
void ko_set_max_hops(int max_hops);
const char* kr_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
