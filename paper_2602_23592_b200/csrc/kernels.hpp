// kernels.hpp -- host-side launchers of the sm_100a kernels.
#pragma once

#include "common.cuh"

namespace keep_b200 {

// K0: counter-based weights (model.hpp:54-73, 88-94; prng.hpp:16-61).
// Element (i, j) of a named [rows x cols] tensor is the e = i*cols+j-th normal
// of Rng::stream(seed, name).  Written either fp32 row-major into a wider
// matrix (dst[i*ld + col_off + j]) or bf16 transposed (dst[(col_off+j)*ld + i]).
uint64_t fnv1a64_host(const char* s);
// [j0, j0 + jn) selects a column window (jn < 0: to the last column).
void launch_init_tensor(uint64_t seed, const char* name, int64_t rows, int64_t cols, double std_,
                        void* dst, int64_t ld, int64_t col_off, bool bf16_transposed,
                        cudaStream_t st, int64_t j0 = 0, int64_t jn = -1);

// K1: x[i] = embed[tokens[rows[i]]] (prefill.hpp:201-211).
void launch_embed(const float* embed, const int32_t* tokens, const int32_t* rows, int64_t n, int d,
                  float* x, cudaStream_t st);

// Row gather: dst[i] = src[idx[i]] (fp32 rows of width d); optional bf16 copy.
void launch_gather_rows(const float* src, const int32_t* idx, int64_t n, int d, float* dst,
                        __nv_bfloat16* dst_bf16, cudaStream_t st);
void launch_to_bf16(const float* src, int64_t n, __nv_bfloat16* dst, cudaStream_t st);

// KV-head sharding: all-to-all receive [G][cpr][dl] (block s = rank s's head
// columns of this rank's rows) -> row-major rows [m][G*dl]; es = element bytes.
void launch_pack_heads(const void* recv, int G, int cpr, int m, int dl, int es, void* rows, cudaStream_t st);

// K4: merged-KV assembly from cached blocks (prefill.hpp:255-263, 340-350).
// For entry e: copy rows [dst_row[e], dst_row[e]+nrows[e]) of K and V from
// the block pointers ksrc[e] / vsrc[e].
void launch_copy_cached(const void* const* ksrc, const void* const* vsrc, const int32_t* dst_row,
                        const int32_t* nrows, int n_entries, int64_t row_bytes, void* kdst,
                        void* vdst, int max_rows, cudaStream_t st);

// Host -> device bytes through kernel parameters (no copy engine, no host sync).
void upload_bytes(void* dst, const void* src, size_t n, cudaStream_t st);

// d0[0, bytes) = s0, d1[0, bytes) = s1 on the SMs (pointers by value).
void launch_copy2(void* d0, const void* s0, void* d1, const void* s1, int64_t bytes, cudaStream_t st);

// Batched device-to-device copy of n blocks (sizes multiples of 16 bytes).
void launch_batch_copy(const void* const* src, void* const* dst, const int64_t* bytes, int n, cudaStream_t st);

// K6: rowbins -> summary (prefill.hpp:281-288, 306-315).
// rowbin[i][j]: probability mass (head mean) of compact row i on segment j.
// seg_cbeg/seg_cend: compact row range of each segment (empty if inactive);
// query rows are [q_cbeg, q_cend).  Writes qts[S] and sts[S*S] (fp64).
template <typename TB>
void launch_summary_reduce(const TB* rowbin, int S, const int32_t* seg_cbeg, const int32_t* seg_cend,
                           const int32_t* seg_len, int q_cbeg, int q_cend, int qlen, double* summ,
                           cudaStream_t st);

// K7: converge on the device (recompute.hpp:86-138).
// Lazy summary probe (PARITY): flag[0] = 1 unless every candidate segment's keys
// provably get probability 0 from every query row in every head (s - max below
// -746 by more than the fp64 error bound of the scores), i.e. unless the
// walk's first hop might add a segment (recompute.hpp:110-121).  q: the compact
// rows [n x d] (the query rows are the last qlen), k: the layer's merged keys;
// scratch: (qlen + 1) x H uint64.
void launch_walk_probe(const float* q, const float* k, const int32_t* rows, const int32_t* row_seg,
                       const uint8_t* cand, int n, int qlen, int Tm, int H, int dh, int d, uint64_t* scratch,
                       int* flag, cudaStream_t st);
void launch_single_hop(const double* qts, const uint8_t* live, int S, int64_t budget, uint8_t* next,
                       cudaStream_t st);
void launch_select(int S, const double* qts, const double* sts, int64_t budget,
                   const uint8_t* candidates, int32_t* order, int32_t* n_out, int32_t* hops_out,
                   cudaStream_t st, int max_hops = 0);  // max_hops > 0: capped walk (BASELINE configs[3])

// K7 for a batch of queries: one walk per CTA (see select_batch_kernel).
void launch_select_batch(int S, int B, const double* const* summ, int64_t budget, const uint8_t* cand,
                         const uint8_t* run, int32_t* out, cudaStream_t st, int max_hops = 0);

// K11: Model::logits of one fp32 row, fp64 accumulation in ascending i
// (model.hpp:76-85).
void launch_logits(const float* row, const float* unembed, int d, int V, double* out,
                   cudaStream_t st);
// ... for B rows [B x d] -> out [B x V] (same arithmetic per row)
void launch_logits_multi(const float* rows, int B, const float* unembed, int d, int V, double* out, cudaStream_t st);
// K11b: divergence (prefill.hpp:501-531) of two rows given their logits;
// out[0] = L2, out[1] = symmetric KL.
void launch_divergence(const float* a, const float* b, int d, const double* la, const double* lb, int V, double* out,
                       cudaStream_t st);

// RoPE hook (off by default; the reference is NoPE): rotate q[i] and the merged
// key row rows[i] at position rows[i] - key_lo[rows[i]]; re-shift cached key
// rows (tab: per entry first row, rows, delta) by delta positions.
void launch_rope_qk(void* q, void* k, int n, const int32_t* rows, const int32_t* key_lo, int dl, int dh, double theta,
                    bool bf16, cudaStream_t st);
void launch_rope_shift(void* k, const int32_t* tab, int n_entries, int max_rows, int dl, int dh, double theta,
                       bool bf16, cudaStream_t st);

// ------------------------------------------------------------ parity GEMM --
// C = A[M x K] . B[K x N] with fp32 operands and fp64 accumulation in
// ascending k (bit-exact with vec_mat, tensor.hpp:31-41).
enum EpiKind { EPI_QKV = 0, EPI_RESID = 1, EPI_RELU = 2, EPI_STORE = 3, EPI_F64 = 4 /* out = double*: the fp64 sum itself (DFMA path) */ };
struct EpiArgs {
    int kind;
    int d;                 // model dim (QKV split)
    float* out;            // STORE / RELU: [M x N]; QKV: q [M x d]; RESID: x [M x N] (+=)
    int64_t ldo;
    void* kdst;            // QKV: merged keys [T x d] (row = rows[i])
    void* vdst;
    const int32_t* rows;   // QKV scatter rows
    __nv_bfloat16* out_bf16;  // optional bf16 mirror of the written value (FAST)
    float q_scale = 1.f;      // QKV (FAST): q is stored as bf16(q * q_scale)
};
void launch_gemm_f64acc(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                        const EpiArgs& epi, cudaStream_t st, bool exact = false);

// ------------------------------------------------------- attention family --
// Causal attention of compact rows against the merged KV of one layer, with
// normalised probabilities binned per (row, destination segment).
struct AttnArgs {
    int n;          // compact rows
    int T;          // keys
    int H, dh, d;   // heads of this rank, head dim, q/k/v/ctx row width (H * dh)
    double inv_heads;  // 1 / (heads of the model): summary bins are partial sums over this rank's heads
    const void* q;  // [n x d] compact queries (fp32 PARITY / bf16 FAST)
    const void* k;  // [T x d] merged keys
    const void* v;  // [T x d] merged values
    const int32_t* rows;     // [n] global row of compact row i
    const int32_t* row_seg;  // [T] segment of key row (-1 = query)
    const int32_t* key_lo;   // [T] first visible key of a row (nullptr = 0: causal prefix);
                             // block-diagonal contexts for canonical refresh
    bool with_bins;
    bool exact;     // PARITY_EXACT: the scalar kernels (scores in the reference's dimension order)
    int S;
    // split plan (segment-aligned key splits, computed by the host)
    int nsplit;
    const int32_t* split_lo;  // [nsplit] first key of split
    const int32_t* split_hi;  // [nsplit] one past last key
    int nsplit_b;             // the DMMA bins pass's own segment-aligned splits
    const int32_t* split_lo_b;
    const int32_t* split_hi_b;
    int rows_per_tile;
    // scratch / outputs
    double* m_part;  // [nsplit x n x H]
    double* l_part;
    double* m_fin;   // [n x H]
    double* l_fin;
    double* o_part;  // [nsplit x n x d] (only when nsplit > 1)
    float* ctx;      // [n x d] fp32 output (PARITY)
    __nv_bfloat16* ctx_bf16;  // [n x d] (FAST)
    void* rowbin;    // [n x S] fp64 (PARITY) / fp32 (FAST)
    // PARITY DMMA, bins fused into the context pass: per head, row and
    // destination segment the unnormalised sum of e = exp(s - m) over the
    // segment's keys ([H x n x S] fp64; nullptr: the separate bins pass)
    double* ebin;
    const int32_t* seg_start;  // [S] first key of each segment
    int Tm;                    // first query key (keys >= Tm have row_seg -1)
    int* flag;                 // [1] device scratch: the reference-score pass's overflow check
};
void launch_attention_parity(const AttnArgs& a, cudaStream_t st);
// PARITY on the fp64 tensor cores (attn_dmma.cu): head_dim 8 / 16 / 32 / 64 / 128,
// 64-row tiles; the split plan (split_lo / hi, nsplit) as for the SIMT kernels
bool attention_dmma_fits(int dh);
bool parity_attention_dmma(int dh);
int attention_dmma_rows_per_tile();
// summary bins fused into the warp-specialised context pass (needs AttnArgs::ebin)
bool dmma_fused_bins(int dh);
// few rows without a summary: the key-split fp64 decode kernel (its own split target)
bool attention_f64_decode(int n, int dh, bool with_bins);
void launch_attention_parity_dmma(const AttnArgs& a, cudaStream_t st);
void launch_stats_combine(const AttnArgs& a, cudaStream_t st);
void launch_ctx_combine(const AttnArgs& a, cudaStream_t st);
void launch_attention_fast(const AttnArgs& a, cudaStream_t st);

}  // namespace keep_b200
