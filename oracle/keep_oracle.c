/*
 * keep_oracle.c -- plain-C restatement of the reference KEEP prefill path.
 *
 * TEST INFRASTRUCTURE ONLY (see keep_oracle.h): the checker for the CUDA
 * product and the CPU baseline timed by bench.py.  Never linked by the product.
 *
 * Arithmetic contract restated from the reference:
 *   fp32 storage, fp64 accumulation in ascending k order, cast to fp32
 *   (tensor.hpp:31-41); fp64 attention / softmax / summaries
 *   (prefill.hpp:124-159, 266-315); fp32 residual adds (prefill.hpp:289-303).
 * Built with plain -O2 (no -ffast-math, no -march=native) so that the
 * operation sequence, and hence every rounding, equals the reference build.
 *
 * Pinned: tests/test_oracle.py checks every ko_* function against the kr_*
 * reference shim (when oracle/_ref is built) and against the committed golden
 * vectors in tests/golden/ (always).
 */
#include "keep_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* ko_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ prng -- */
/* splitmix64 step (prng.hpp:16-21): advance by the golden gamma, then mix. */
static uint64_t mix_step(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* FNV-1a over the bytes of a name (prng.hpp:23-30). */
static uint64_t fnv1a(const char* s) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= (unsigned char)*s;
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* Rng(seed) warms up with two discarded draws (prng.hpp:34-38);
 * Rng::stream xors the seed with the name hash (prng.hpp:42-45). */
static uint64_t stream_state(uint64_t seed, const char* name) {
    uint64_t s = seed ^ fnv1a(name);
    mix_step(&s);
    mix_step(&s);
    return s;
}

static double unit_draw(uint64_t* s) { /* next_double, prng.hpp:52-54 */
    return (double)(mix_step(s) >> 11) * 0x1.0p-53;
}

static double irwin_hall(uint64_t* s) { /* gaussian, prng.hpp:57-61 */
    double acc = 0.0;
    for (int i = 0; i < 12; ++i) acc += unit_draw(s);
    return acc - 6.0;
}

/* ----------------------------------------------------------------- model -- */
uint64_t ko_weight_count(int L, int H, int d, int mlp, int V) {
    (void)H;
    return 2ull * (uint64_t)V * d + (uint64_t)L * (4ull * d * d + 2ull * (uint64_t)d * mlp);
}

static int check_cfg(int L, int H, int d, int mlp, int V) { /* model.hpp:28-38 */
    if (L < 1) return fail(1, "num_layers must be positive");
    if (H < 1) return fail(1, "num_heads must be positive");
    if (d < 1) return fail(1, "model_dim must be positive");
    if (mlp < 1) return fail(1, "mlp_dim must be positive");
    if (V < 1) return fail(1, "vocab_size must be positive");
    if (d % H) return fail(1, "model_dim not divisible by num_heads");
    return 0;
}

/* One named tensor of n elements drawn as float(normal(std))
 * (model.hpp:88-94: Rng::stream(seed, name), normal = gaussian * std). */
static void init_named(uint64_t seed, const char* name, size_t n, double std_, float* out) {
    uint64_t s = stream_state(seed, name);
    for (size_t i = 0; i < n; ++i) out[i] = (float)(irwin_hall(&s) * std_);
}

int ko_model_init(int L, int H, int d, int mlp, int V, uint64_t seed, float* w) {
    int rc = check_cfg(L, H, d, mlp, V);
    if (rc) return rc;
    const double std_ = 1.0 / sqrt((double)d); /* model.hpp:56 */
    char name[64];
    init_named(seed, "embed", (size_t)V * d, std_, w);
    w += (size_t)V * d;
    init_named(seed, "unembed", (size_t)d * V, std_, w);
    w += (size_t)d * V;
    static const char* parts[6] = {"wq", "wk", "wv", "wo", "mlp_in", "mlp_out"};
    for (int l = 0; l < L; ++l) {
        for (int k = 0; k < 6; ++k) {
            size_t n = (k < 4) ? (size_t)d * d : (size_t)d * mlp;
            snprintf(name, sizeof name, "layer%d.%s", l, parts[k]);
            init_named(seed, name, n, std_, w);
            w += n;
        }
    }
    return 0;
}

/* Layout half of testutil::make_instance (tests/test_util.hpp:26-36). */
int ko_make_instance_layout(uint64_t seed, int S, int V, int lo, int hi, int qlen,
                            int32_t* seg_len, int32_t* tokens, int32_t* query) {
    uint64_t s = stream_state(seed, "instance");
    for (int i = 0; i < S; ++i) {
        int n = lo + (int)(mix_step(&s) % (uint64_t)(hi - lo + 1));
        seg_len[i] = n;
        for (int k = 0; k < n; ++k) *tokens++ = (int32_t)(mix_step(&s) % (uint64_t)V);
    }
    for (int k = 0; k < qlen; ++k) query[k] = (int32_t)(mix_step(&s) % (uint64_t)V);
    return 0;
}

/* -------------------------------------------------------------- schedule -- */
/* Geometric r[l] = g^l with g bisected (200 halvings) so mean(r) = r_avg;
 * r[0] forced to 1 (recompute.hpp:33-70). */
int ko_ratio_schedule(int L, double r_avg, double* r) {
    if (L < 1) return fail(1, "num_layers must be >= 1");
    if (L == 1) {
        r[0] = 1.0;
        return 0;
    }
    if (r_avg < 1.0 / L - 1e-9 || r_avg > 1.0 + 1e-9) return fail(1, "infeasible r_avg");
    double lo = 0.0, hi = 1.0;
    for (int it = 0; it < 200; ++it) {
        double g = 0.5 * (lo + hi), term = 1.0, sum = 0.0;
        for (int l = 0; l < L; ++l) {
            sum += term;
            term *= g;
        }
        if (sum / L < r_avg) lo = g;
        else hi = g;
    }
    double g = 0.5 * (lo + hi), term = 1.0;
    for (int l = 0; l < L; ++l) {
        r[l] = term;
        term *= g;
    }
    r[0] = 1.0;
    return 0;
}

/* budget = clamp(ceil(r*S - 1e-9), 1, S) (recompute.hpp:73-77). */
int64_t ko_layer_budget(double ratio, int64_t S) {
    int64_t b = (int64_t)ceil(ratio * (double)S - 1e-9);
    if (b > S) b = S;
    return b < 1 ? 1 : b;
}

/* -------------------------------------------------------------- selector -- */
/* converge = init_importance + propagate_hop until stable / budget / S hops
 * (recompute.hpp:86-138).  Scores of allowed, unselected positions are
 * re-derived each hop as the mean over the relevant set (summed in ascending
 * position, as std::set iterates) of segment_to_segment[m][i]; the pick is the
 * first strict maximum in ascending position among scores > 0. */
/* Optional hop cap (BASELINE configs[3] "3-hop recompute"; not in the
 * reference, whose converge runs up to S hops): the one-line restatement of
 * the capped variant is the loop bound min(S, max_hops).  0 = uncapped. */
static int g_max_hops = 0;
void ko_set_max_hops(int max_hops) { g_max_hops = max_hops; }

int ko_converge(int S, const double* qts, const double* sts, int64_t budget,
                const uint8_t* cand, int32_t* order, int32_t* n_out, int32_t* hops_out) {
    double* score = (double*)malloc(sizeof(double) * (S > 0 ? S : 1));
    uint8_t* in_r = (uint8_t*)calloc(S > 0 ? S : 1, 1);
    if (!score || !in_r) return fail(9, "oom");
    memcpy(score, qts, sizeof(double) * S);
    int n = 0, hop = 0;
    const int hop_cap = (g_max_hops > 0 && g_max_hops < S) ? g_max_hops : S;
    while ((int64_t)n < budget && hop < hop_cap) {
        if (n > 0) {
            for (int i = 0; i < S; ++i) {
                if ((cand && !cand[i]) || in_r[i]) continue;
                double acc = 0.0;
                for (int m = 0; m < S; ++m)
                    if (in_r[m]) acc += sts[(size_t)m * S + i];
                score[i] = acc / (double)n;
            }
        }
        int best = -1;
        if ((int64_t)n < budget) {
            for (int i = 0; i < S; ++i) {
                if ((cand && !cand[i]) || in_r[i]) continue;
                if (score[i] <= 0.0) continue;
                if (best < 0 || score[i] > score[best]) best = i;
            }
        }
        ++hop;
        if (best < 0) break;
        in_r[best] = 1;
        order[n++] = best;
    }
    *n_out = n;
    *hops_out = hop;
    free(score);
    free(in_r);
    return 0;
}

/* ---------------------------------------------------------------- prefill -- */
typedef struct {
    int L, H, d, f, V;
    const float *embed, *unembed;
    const float* layer; /* first layer block */
} model_view;

static model_view view_of(const keep_problem* p, const float* w) {
    model_view m;
    m.L = p->num_layers;
    m.H = p->num_heads;
    m.d = p->model_dim;
    m.f = p->mlp_dim;
    m.V = p->vocab_size;
    m.embed = w;
    m.unembed = w + (size_t)m.V * m.d;
    m.layer = m.unembed + (size_t)m.d * m.V;
    return m;
}

static const float* layer_w(const model_view* m, int l, int which) {
    const size_t dd = (size_t)m->d * m->d, df = (size_t)m->d * m->f;
    const float* base = m->layer + (size_t)l * (4 * dd + 2 * df);
    if (which < 4) return base + which * dd;
    return base + 4 * dd + (which - 4) * df;
}

/* out[n] = fp32( sum_k fp64(x[k]) * W[k][n] ), k ascending, zero x skipped
 * (tensor.hpp:31-41). */
static void row_times(const float* x, int k, const float* W, int n, float* out, double* acc) {
    for (int j = 0; j < n; ++j) acc[j] = 0.0;
    for (int i = 0; i < k; ++i) {
        const double xi = x[i];
        if (xi == 0.0) continue;
        const float* wr = W + (size_t)i * n;
        for (int j = 0; j < n; ++j) acc[j] += xi * wr[j];
    }
    for (int j = 0; j < n; ++j) out[j] = (float)acc[j];
}

/* Prefill state over one layout: the cursor of prefill.hpp:172-362 (and, with
 * every segment active and no cache, the dense pass of prefill.hpp:366-469). */
typedef struct {
    model_view m;
    int S, T, qlen, qstart;
    int *seg_start, *seg_len, *row_seg;
    float* x;                 /* [T*d] residual stream */
    uint8_t *prev, *dropped;  /* per segment */
    const float* cached;      /* flat canonical KV or NULL */
    int Tm;
    int layer;
    /* scratch */
    float *q, *ctx, *proj, *hid;
    double *acc, *prob, *scores, *qraw, *sraw, *cbuf;
} cursor;

static void cursor_free(cursor* c) {
    free(c->seg_start); free(c->seg_len); free(c->row_seg); free(c->x);
    free(c->prev); free(c->dropped); free(c->q); free(c->ctx); free(c->proj);
    free(c->hid); free(c->acc); free(c->prob); free(c->scores); free(c->qraw);
    free(c->sraw); free(c->cbuf);
}

static int cursor_open(cursor* c, const keep_problem* p, const float* w, const float* cached,
                       int with_query) {
    memset(c, 0, sizeof *c);
    int rc = check_cfg(p->num_layers, p->num_heads, p->model_dim, p->mlp_dim, p->vocab_size);
    if (rc) return rc;
    c->m = view_of(p, w);
    const int S = p->num_segments, d = c->m.d;
    if (S < 1) return fail(2, "layout is empty"); /* prefill.hpp:177 */
    c->S = S;
    c->qlen = with_query ? p->query_len : 0;
    c->seg_start = (int*)malloc(sizeof(int) * S);
    c->seg_len = (int*)malloc(sizeof(int) * S);
    int pos = 0;
    const int32_t* tok = p->tokens;
    for (int i = 0; i < S; ++i) { /* prefill.hpp:178-195 */
        if (p->seg_len[i] < 1) return fail(2, "empty segment in layout");
        for (int k = 0; k < p->seg_len[i]; ++k)
            if (tok[k] < 0 || tok[k] >= c->m.V) return fail(2, "token out of vocab range");
        tok += p->seg_len[i];
        c->seg_start[i] = pos;
        c->seg_len[i] = p->seg_len[i];
        pos += p->seg_len[i];
    }
    for (int k = 0; k < c->qlen; ++k)
        if (p->query[k] < 0 || p->query[k] >= c->m.V) return fail(2, "token out of vocab range");
    c->Tm = pos;
    c->qstart = pos;
    c->T = pos + c->qlen;
    const int T = c->T, f = c->m.f;
    c->row_seg = (int*)malloc(sizeof(int) * T);
    for (int t = 0; t < T; ++t) c->row_seg[t] = -1;
    for (int i = 0; i < S; ++i)
        for (int k = 0; k < c->seg_len[i]; ++k) c->row_seg[c->seg_start[i] + k] = i;
    c->x = (float*)malloc(sizeof(float) * (size_t)T * d);
    tok = p->tokens;
    for (int t = 0; t < c->Tm; ++t) /* embedding gather, prefill.hpp:201-211 */
        memcpy(c->x + (size_t)t * d, c->m.embed + (size_t)tok[t] * d, sizeof(float) * d);
    for (int k = 0; k < c->qlen; ++k)
        memcpy(c->x + (size_t)(c->qstart + k) * d, c->m.embed + (size_t)p->query[k] * d,
               sizeof(float) * d);
    c->prev = (uint8_t*)malloc(S);
    c->dropped = (uint8_t*)calloc(S, 1);
    memset(c->prev, 1, S);
    c->cached = cached;
    c->q = (float*)malloc(sizeof(float) * (size_t)T * d);
    c->ctx = (float*)malloc(sizeof(float) * d);
    c->proj = (float*)malloc(sizeof(float) * d);
    c->hid = (float*)malloc(sizeof(float) * f);
    c->acc = (double*)malloc(sizeof(double) * (d > f ? d : f));
    c->prob = (double*)malloc(sizeof(double) * T);
    c->scores = (double*)malloc(sizeof(double) * T);
    c->qraw = (double*)malloc(sizeof(double) * S);
    c->sraw = (double*)malloc(sizeof(double) * (size_t)S * S);
    c->cbuf = (double*)malloc(sizeof(double) * d);
    return 0;
}

/* Causal attention of row t over keys 0..t, all heads, fp64 softmax; ctx in
 * fp64 cast to fp32; prob[tau] accumulates p/H over heads in head order
 * (prefill.hpp:124-159). */
static void attend_row(cursor* c, const float* qrow, const float* K, const float* Vv, int t) {
    const int H = c->m.H, d = c->m.d, dh = d / H;
    const double scale = 1.0 / sqrt((double)dh), inv_h = 1.0 / H;
    double* s = c->scores;
    for (int h = 0; h < H; ++h) {
        const int off = h * dh;
        double mx = -1e300;
        for (int u = 0; u <= t; ++u) {
            const float* kr = K + (size_t)u * d + off;
            double dotv = 0.0;
            for (int j = 0; j < dh; ++j) dotv += (double)qrow[off + j] * kr[j];
            s[u] = dotv * scale;
            if (s[u] > mx) mx = s[u];
        }
        double sum = 0.0;
        for (int u = 0; u <= t; ++u) {
            s[u] = exp(s[u] - mx);
            sum += s[u];
        }
        const double inv = 1.0 / sum;
        double* cb = c->cbuf;
        for (int j = 0; j < dh; ++j) cb[j] = 0.0;
        for (int u = 0; u <= t; ++u) {
            const double pu = s[u] * inv;
            c->prob[u] += pu * inv_h;
            const float* vr = Vv + (size_t)u * d + off;
            for (int j = 0; j < dh; ++j) cb[j] += pu * vr[j];
        }
        for (int j = 0; j < dh; ++j) c->ctx[off + j] = (float)cb[j];
    }
}

/* One layer (PrefillCursor::step, prefill.hpp:224-322).  active[i]: segment
 * position i recomputed.  kv_out: keys[T*d], values[T*d]; summary_out: S+S*S. */
static int cursor_step(cursor* c, const uint8_t* active, float* kv_out, double* summary_out) {
    const int S = c->S, T = c->T, d = c->m.d, f = c->m.f, l = c->layer;
    if (l >= c->m.L) return fail(3, "stepped past last layer");
    for (int i = 0; i < S; ++i)
        if (active[i] && !c->prev[i]) return fail(3, "plan is not monotone across layers");
    for (int i = 0; i < S; ++i) { /* newly dropped rows are zeroed for good */
        if (!active[i] && !c->dropped[i]) {
            c->dropped[i] = 1;
            memset(c->x + (size_t)c->seg_start[i] * d, 0, sizeof(float) * (size_t)c->seg_len[i] * d);
        }
    }
    const float *wq = layer_w(&c->m, l, 0), *wk = layer_w(&c->m, l, 1), *wv = layer_w(&c->m, l, 2),
                *wo = layer_w(&c->m, l, 3), *wi = layer_w(&c->m, l, 4), *wout = layer_w(&c->m, l, 5);
    float* K = kv_out;
    float* Vv = kv_out + (size_t)T * d;
    for (int t = 0; t < T; ++t) { /* projections or cached copy, 250-264 */
        const int sg = c->row_seg[t];
        if (sg < 0 || active[sg]) {
            const float* xr = c->x + (size_t)t * d;
            row_times(xr, d, wk, d, K + (size_t)t * d, c->acc);
            row_times(xr, d, wv, d, Vv + (size_t)t * d, c->acc);
            row_times(xr, d, wq, d, c->q + (size_t)t * d, c->acc);
        } else {
            if (!c->cached) return fail(4, "no cached KV supplied");
            const float* kb = c->cached + (size_t)l * 2 * c->Tm * d;
            memcpy(K + (size_t)t * d, kb + (size_t)t * d, sizeof(float) * d);
            memcpy(Vv + (size_t)t * d, kb + (size_t)c->Tm * d + (size_t)t * d, sizeof(float) * d);
        }
    }
    for (int i = 0; i < S; ++i) c->qraw[i] = 0.0;
    memset(c->sraw, 0, sizeof(double) * (size_t)S * S);
    for (int t = 0; t < T; ++t) { /* attention, binning, Wo + residual: 274-292 */
        const int src = c->row_seg[t];
        if (!(src < 0 || active[src])) continue;
        for (int u = 0; u <= t; ++u) c->prob[u] = 0.0;
        attend_row(c, c->q + (size_t)t * d, K, Vv, t);
        for (int u = 0; u <= t; ++u) {
            const int dst = c->row_seg[u];
            if (dst < 0) continue;
            if (src < 0) c->qraw[dst] += c->prob[u];
            else if (dst != src) c->sraw[(size_t)src * S + dst] += c->prob[u];
        }
        row_times(c->ctx, d, wo, d, c->proj, c->acc);
        float* xr = c->x + (size_t)t * d;
        for (int j = 0; j < d; ++j) xr[j] += c->proj[j];
    }
    for (int t = 0; t < T; ++t) { /* ReLU MLP + residual: 295-304 */
        const int sg = c->row_seg[t];
        if (!(sg < 0 || active[sg])) continue;
        float* xr = c->x + (size_t)t * d;
        row_times(xr, d, wi, f, c->hid, c->acc);
        for (int j = 0; j < f; ++j)
            if (c->hid[j] < 0.0f) c->hid[j] = 0.0f;
        row_times(c->hid, f, wout, d, c->proj, c->acc);
        for (int j = 0; j < d; ++j) xr[j] += c->proj[j];
    }
    if (summary_out) { /* normalisation: 306-315 */
        double* qts = summary_out;
        double* sts = summary_out + S;
        for (int j = 0; j < S; ++j) qts[j] = c->qlen > 0 ? c->qraw[j] / c->qlen : 0.0;
        for (int i = 0; i < S; ++i)
            for (int j = 0; j < S; ++j)
                sts[(size_t)i * S + j] = j < i ? c->sraw[(size_t)i * S + j] / c->seg_len[i] : 0.0;
    }
    memcpy(c->prev, active, S);
    c->layer++;
    return 0;
}

/* finish (prefill.hpp:324-337): dropped rows are zero in the final hidden. */
static void cursor_finish(cursor* c, float* final_hidden) {
    if (!final_hidden) return;
    const int d = c->m.d;
    memcpy(final_hidden, c->x, sizeof(float) * (size_t)c->T * d);
    for (int i = 0; i < c->S; ++i)
        if (c->dropped[i])
            memset(final_hidden + (size_t)c->seg_start[i] * d, 0,
                   sizeof(float) * (size_t)c->seg_len[i] * d);
}

static size_t layer_kv_floats(const cursor* c) { return 2 * (size_t)c->T * c->m.d; }
static size_t summary_doubles(int S) { return (size_t)S + (size_t)S * S; }

/* Dense pass with every row computed (full_prefill, prefill.hpp:366-469). */
static int dense_pass(const keep_problem* p, const float* w, int with_query, float* final_hidden,
                      float* kv, double* summaries) {
    cursor c;
    int rc = cursor_open(&c, p, w, NULL, with_query);
    if (rc) { cursor_free(&c); return rc; }
    uint8_t* all = (uint8_t*)malloc(c.S);
    memset(all, 1, c.S);
    float* scratch = kv ? NULL : (float*)malloc(sizeof(float) * layer_kv_floats(&c));
    for (int l = 0; l < c.m.L && !rc; ++l)
        rc = cursor_step(&c, all, kv ? kv + l * layer_kv_floats(&c) : scratch,
                         summaries ? summaries + l * summary_doubles(c.S) : NULL);
    if (!rc) cursor_finish(&c, final_hidden);
    free(all);
    free(scratch);
    cursor_free(&c);
    return rc;
}

int ko_full_prefill(const keep_problem* p, const float* w, float* final_hidden, float* kv,
                    double* summaries) {
    return dense_pass(p, w, 1, final_hidden, kv, summaries);
}

/* Canonical KV of the memory rows: segment_prefill per dynamic segment
 * (prefill.hpp:472-476), one joint dense pass per static group sliced per
 * member (harness.hpp:512-532, 659-677). */
int ko_canonical_kv(const keep_problem* p, const float* w, float* out) {
    const int L = p->num_layers, d = p->model_dim, S = p->num_segments;
    int Tm = 0;
    for (int i = 0; i < S; ++i) Tm += p->seg_len[i];
    int nu = p->num_units;
    int *ub = (int*)malloc(sizeof(int) * (nu ? nu : S)), *ue = (int*)malloc(sizeof(int) * (nu ? nu : S)),
        *ug = (int*)malloc(sizeof(int) * (nu ? nu : S));
    if (nu == 0) {
        nu = S;
        for (int i = 0; i < S; ++i) { ub[i] = i; ue[i] = i + 1; ug[i] = 0; }
    } else {
        for (int u = 0; u < nu; ++u) { ub[u] = p->unit_begin[u]; ue[u] = p->unit_end[u]; ug[u] = p->unit_is_group[u]; }
    }
    int rc = 0, row0 = 0;
    const int32_t* tok = p->tokens;
    /* token offset of each segment */
    int* tok_off = (int*)malloc(sizeof(int) * (S + 1));
    tok_off[0] = 0;
    for (int i = 0; i < S; ++i) tok_off[i + 1] = tok_off[i] + p->seg_len[i];
    (void)tok;
    (void)row0;
    for (int u = 0; u < nu && !rc; ++u) {
        /* one "context" = the whole group, or one segment at a time */
        const int nctx = ug[u] ? 1 : ue[u] - ub[u];
        for (int cidx = 0; cidx < nctx && !rc; ++cidx) {
            const int b = ug[u] ? ub[u] : ub[u] + cidx;
            const int e = ug[u] ? ue[u] : b + 1;
            keep_problem sub = *p;
            sub.num_segments = e - b;
            sub.seg_len = p->seg_len + b;
            sub.tokens = p->tokens + tok_off[b];
            sub.query_len = 0;
            sub.num_units = 0;
            const int n = tok_off[e] - tok_off[b];
            float* kv = (float*)malloc(sizeof(float) * (size_t)L * 2 * n * d);
            rc = dense_pass(&sub, w, 0, NULL, kv, NULL);
            for (int l = 0; l < L && !rc; ++l) {
                float* kb = out + (size_t)l * 2 * Tm * d;
                memcpy(kb + (size_t)tok_off[b] * d, kv + (size_t)l * 2 * n * d, sizeof(float) * (size_t)n * d);
                memcpy(kb + (size_t)Tm * d + (size_t)tok_off[b] * d, kv + (size_t)l * 2 * n * d + (size_t)n * d,
                       sizeof(float) * (size_t)n * d);
            }
            free(kv);
        }
    }
    free(ub); free(ue); free(ug); free(tok_off);
    return rc;
}

static float* canonical_or(const keep_problem* p, const float* w, const float* cached, int* rc,
                           float** owned) {
    *owned = NULL;
    if (cached) return (float*)cached;
    int Tm = 0;
    for (int i = 0; i < p->num_segments; ++i) Tm += p->seg_len[i];
    *owned = (float*)malloc(sizeof(float) * (size_t)p->num_layers * 2 * Tm * p->model_dim);
    *rc = ko_canonical_kv(p, w, *owned);
    return *owned;
}

/* selective_prefill (prefill.hpp:478-497): validates the plan, then steps. */
int ko_selective_prefill(const keep_problem* p, const float* w, const float* cached,
                         const uint8_t* plan, float* final_hidden, float* kv, double* summaries) {
    const int L = p->num_layers, S = p->num_segments;
    for (int l = 0; l + 1 < L; ++l) /* is_monotone, prefill.hpp:95-104 */
        for (int i = 0; i < S; ++i)
            if (plan[(l + 1) * S + i] && !plan[l * S + i]) return fail(3, "plan is not monotone across layers");
    int rc = 0;
    float* owned;
    const float* cache = canonical_or(p, w, cached, &rc, &owned);
    if (rc) { free(owned); return rc; }
    cursor c;
    rc = cursor_open(&c, p, w, cache, 1);
    float* scratch = NULL;
    if (!rc && !kv) scratch = (float*)malloc(sizeof(float) * layer_kv_floats(&c));
    for (int l = 0; l < L && !rc; ++l)
        rc = cursor_step(&c, plan + l * S, kv ? kv + l * layer_kv_floats(&c) : scratch,
                         summaries ? summaries + l * summary_doubles(S) : NULL);
    if (!rc) cursor_finish(&c, final_hidden);
    free(scratch);
    cursor_free(&c);
    free(owned);
    return rc;
}

/* plan_keep (recompute.hpp:140-180): layer 0 all active; after step(l) the
 * budget of layer l+1 decides keep-all or converge restricted to the live set;
 * the multihop=false ablation ranks live segments by query attention with a
 * stable sort (166-176).  Outputs the realized walk per layer (order_len -1 =
 * keep-all, no walk). */
int ko_plan_keep(const keep_problem* p, const float* w, const float* cached, const double* r,
                 int multihop, uint8_t* plan, int32_t* orders, int32_t* order_len, int32_t* hops,
                 double* summaries, float* final_hidden, float* kv) {
    const int L = p->num_layers, S = p->num_segments;
    int rc = 0;
    float* owned;
    const float* cache = canonical_or(p, w, cached, &rc, &owned);
    if (rc) { free(owned); return rc; }
    cursor c;
    rc = cursor_open(&c, p, w, cache, 1);
    uint8_t* active = (uint8_t*)malloc(S);
    uint8_t* next = (uint8_t*)malloc(S);
    double* summ = (double*)malloc(sizeof(double) * summary_doubles(S));
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * S);
    float* scratch = kv ? NULL : (float*)malloc(sizeof(float) * (rc ? 1 : layer_kv_floats(&c)));
    memset(active, 1, S);
    for (int l = 0; l < L; ++l) { order_len[l] = -1; hops[l] = 0; }
    for (int l = 0; l < L && !rc; ++l) {
        memcpy(plan + l * S, active, S);
        rc = cursor_step(&c, active, kv ? kv + l * layer_kv_floats(&c) : scratch, summ);
        if (rc) break;
        if (summaries) memcpy(summaries + l * summary_doubles(S), summ, sizeof(double) * summary_doubles(S));
        if (l + 1 >= L) break;
        const int64_t budget = ko_layer_budget(r[l + 1], S);
        int64_t live = 0;
        for (int i = 0; i < S; ++i) live += active[i];
        if (budget >= live) continue;
        memset(next, 0, S);
        if (multihop) {
            int32_t n, h;
            rc = ko_converge(S, summ, summ + S, budget, active, ord, &n, &h);
            for (int k = 0; k < n; ++k) {
                next[ord[k]] = 1;
                orders[(size_t)l * S + k] = ord[k];
            }
            order_len[l] = n;
            hops[l] = h;
        } else {
            /* stable sort of live positions by qts descending (insertion sort
             * is stable and the lists are short) */
            int m = 0;
            for (int i = 0; i < S; ++i)
                if (active[i]) ord[m++] = i;
            for (int a = 1; a < m; ++a) {
                int v = ord[a], b = a - 1;
                while (b >= 0 && summ[v] > summ[ord[b]]) { ord[b + 1] = ord[b]; --b; }
                ord[b + 1] = v;
            }
            for (int k = 0; k < budget && k < m; ++k) next[ord[k]] = 1;
        }
        memcpy(active, next, S);
    }
    if (!rc) cursor_finish(&c, final_hidden);
    free(active); free(next); free(summ); free(ord); free(scratch);
    cursor_free(&c);
    free(owned);
    return rc;
}

/* Model::logits (model.hpp:76-85): fp64, i ascending. */
int ko_logits(const keep_problem* p, const float* w, const float* row, double* out) {
    model_view m = view_of(p, w);
    for (int j = 0; j < m.V; ++j) {
        double acc = 0.0;
        for (int i = 0; i < m.d; ++i) acc += (double)row[i] * m.unembed[(size_t)i * m.V + j];
        out[j] = acc;
    }
    return 0;
}

static void softmax_inplace(double* v, int n) { /* prefill.hpp:513-523 */
    double mx = v[0];
    for (int i = 0; i < n; ++i) mx = v[i] > mx ? v[i] : mx;
    double sum = 0.0;
    for (int i = 0; i < n; ++i) { v[i] = exp(v[i] - mx); sum += v[i]; }
    for (int i = 0; i < n; ++i) v[i] /= sum;
}

/* divergence on one (last) row: L2 + symmetric KL of softmax(logits)
 * (prefill.hpp:501-531). */
int ko_divergence(const keep_problem* p, const float* w, const float* a, const float* b,
                  double* l2, double* sym_kl) {
    const int d = p->model_dim, V = p->vocab_size;
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
        const double dl = (double)a[j] - b[j];
        acc += dl * dl;
    }
    *l2 = sqrt(acc);
    double* pa = (double*)malloc(sizeof(double) * V);
    double* pb = (double*)malloc(sizeof(double) * V);
    ko_logits(p, w, a, pa);
    ko_logits(p, w, b, pb);
    softmax_inplace(pa, V);
    softmax_inplace(pb, V);
    double kl = 0.0;
    for (int i = 0; i < V; ++i) kl += (pa[i] - pb[i]) * (log(pa[i]) - log(pb[i]));
    *sym_kl = kl;
    free(pa);
    free(pb);
    return 0;
}
