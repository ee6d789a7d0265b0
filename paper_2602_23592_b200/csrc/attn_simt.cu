// attn_simt.cu -- K5 causal attention + segment summary on CUDA cores.
//
// Three passes over segment-aligned key splits (the summary
// needs NORMALISED probabilities, so the softmax statistics come first):
//   1. stats   per (row tile, head, split): running max / sum of exp
//              -> combine over splits (fixed order)
//   2. context per (row tile, head, split): p = exp(s - m) * (1/l),
//              ctx = sum p v  -> combine partials over splits (fixed order)
//   3. bins    per (row tile, split), heads looped inside in head order:
//              prob_mean[key] += p / H exactly as attention_row does
//              (prefill.hpp:150-153), then per-row sums over the keys of each
//              destination segment in key order (prefill.hpp:281-288).
// Scores are recomputed bit-identically in every pass (same DFMA chain).
// PARITY instantiation: fp32 q/K/V, fp64 everything (dot in ascending
// dimension order == dot(), tensor.hpp:43-47).
// FAST instantiation (interim, CUDA cores): bf16 q/K/V, fp32 math, fp32 bins.
#include "kernels.hpp"

#include <cstring>

#include <cfloat>

namespace keep_b200 {

namespace {
constexpr int RT = 16;   // compact rows per tile
constexpr int KC = 64;   // keys per chunk
constexpr int NT = 256;  // threads
constexpr int MAXDH = 128;

template <typename T> __device__ __forceinline__ float ldf(const T* p);
template <> __device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}

template <typename A> __device__ __forceinline__ A ex(A x);
template <> __device__ __forceinline__ double ex<double>(double x) { return exp(x); }
template <> __device__ __forceinline__ float ex<float>(float x) { return __expf(x); }

// Explicitly rounded steps (no FMA contraction): the reference rounds
// s = dot * scale, then s - max, then p = e * inv, then p * inv_heads
// (prefill.hpp:140-151); at depth |s| is so large that a contracted
// s * scale - max moves exp() by orders of magnitude.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

template <typename A> __device__ __forceinline__ A neg_inf();
template <> __device__ __forceinline__ double neg_inf<double>() { return -DBL_MAX; }
template <> __device__ __forceinline__ float neg_inf<float>() { return -FLT_MAX; }

struct Tile {
    int i0, nrows, tmax, klo;
};

// rows are ascending and key_lo is non-decreasing in the row, so the tile's
// first row carries the smallest visible key
__device__ __forceinline__ Tile tile_of(const int32_t* rows, const int32_t* key_lo, int n, int tile) {
    Tile t;
    t.i0 = tile * RT;
    t.nrows = min(RT, n - t.i0);
    t.tmax = rows[t.i0 + t.nrows - 1];
    t.klo = key_lo ? key_lo[rows[t.i0]] : 0;
    return t;
}

__device__ __forceinline__ void load_rows(int* rowt, int* rowlo, const AttnArgs& a, const Tile& tl) {
    if (threadIdx.x < RT) {
        const bool ok = threadIdx.x < tl.nrows;
        const int t = ok ? a.rows[tl.i0 + threadIdx.x] : -1;
        rowt[threadIdx.x] = t;
        rowlo[threadIdx.x] = ok ? (a.key_lo ? a.key_lo[t] : 0) : 0x7fffffff;
    }
}

// Shared-memory staging of the Q head slice [RT x dh] (as ACC) and a K or V
// chunk head slice [KC x (dh+1)] fp32 (padded: conflict-free row access).
template <typename ACC>
struct Smem {
    ACC q[RT * MAXDH];
    float k[KC * (MAXDH + 1)];
    float v[KC * (MAXDH + 1)];
    ACC p[RT * KC];
    int rowt[RT];
    int rowlo[RT];
};

template <typename TQ, typename ACC>
__device__ void load_q(Smem<ACC>& sm, const TQ* q, int i0, int nrows, int d, int off, int dh) {
    for (int e = threadIdx.x; e < RT * dh; e += NT) {
        const int r = e / dh, j = e % dh;
        sm.q[r * MAXDH + j] = (r < nrows) ? ACC(ldf(q + int64_t(i0 + r) * d + off + j)) : ACC(0);
    }
}

template <typename TKV>
__device__ void load_chunk(float* dst, const TKV* src, int k0, int nk, int d, int off, int dh) {
    for (int e = threadIdx.x; e < KC * dh; e += NT) {
        const int r = e / dh, j = e % dh;
        dst[r * (MAXDH + 1) + j] = (r < nk) ? ldf(src + int64_t(k0 + r) * d + off + j) : 0.0f;
    }
}

// Scores of this thread's 4 keys for its row (thread = row r x lane c).
template <typename ACC>
__device__ __forceinline__ void scores4(const Smem<ACC>& sm, int r, int c, int dh, ACC scale, ACC s[4]) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const int key = c + 16 * kk;
        ACC acc = ACC(0);
        for (int j = 0; j < dh; ++j) acc = fma(sm.q[r * MAXDH + j], ACC(sm.k[key * (MAXDH + 1) + j]), acc);
        s[kk] = mul_rn(acc, scale);
    }
}

template <typename ACC>
__device__ __forceinline__ ACC red16_max(ACC x) {
    for (int o = 8; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o, 16));
    return x;
}
template <typename ACC>
__device__ __forceinline__ ACC red16_sum(ACC x) {
    for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o, 16);
    return x;
}

// ---------------------------------------------------------------- pass 1 --
template <typename TQ, typename TKV, typename ACC>
__global__ void __launch_bounds__(NT)
attn_stats_kernel(AttnArgs a, ACC scale) {
    extern __shared__ __align__(16) uint8_t smraw[];
    Smem<ACC>& sm = *reinterpret_cast<Smem<ACC>*>(smraw);
    const Tile tl = tile_of(a.rows, a.key_lo, a.n, blockIdx.x);
    const int h = blockIdx.y, sp = blockIdx.z;
    const int lo = max(a.split_lo[sp], tl.klo), hi = min(a.split_hi[sp], tl.tmax + 1);
    const int r = threadIdx.x / 16, c = threadIdx.x % 16;
    const int off = h * a.dh;
    load_rows(sm.rowt, sm.rowlo, a, tl);
    load_q(sm, static_cast<const TQ*>(a.q), tl.i0, tl.nrows, a.d, off, a.dh);
    ACC m = neg_inf<ACC>(), l = ACC(0);
    for (int k0 = lo; k0 < hi; k0 += KC) {
        const int nk = min(KC, hi - k0);
        __syncthreads();
        load_chunk(sm.k, static_cast<const TKV*>(a.k), k0, nk, a.d, off, a.dh);
        __syncthreads();
        ACC s[4];
        scores4(sm, r, c, a.dh, scale, s);
        const int t = sm.rowt[r], klo = sm.rowlo[r];
        ACC cm = neg_inf<ACC>();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int key = k0 + c + 16 * kk;
            if (c + 16 * kk < nk && key <= t && key >= klo) cm = max(cm, s[kk]);
        }
        cm = red16_max(cm);
        // every lane of the warp must reach the shuffles: no early continue
        const bool any = cm != neg_inf<ACC>();  // a visible key for this row in the chunk
        const ACC mn = max(m, cm);
        ACC part = ACC(0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int key = k0 + c + 16 * kk;
            if (any && c + 16 * kk < nk && key <= t && key >= klo) part += ex(sub_rn(s[kk], mn));
        }
        part = red16_sum(part);
        if (any) {
            l = (m == neg_inf<ACC>() ? ACC(0) : l * ex(sub_rn(m, mn))) + part;
            m = mn;
        }
    }
    if (c == 0 && r < tl.nrows) {
        const int64_t o = (int64_t(sp) * a.n + tl.i0 + r) * a.H + h;
        a.m_part[o] = double(m);
        a.l_part[o] = double(l);
    }
}

__global__ void stats_combine_kernel(AttnArgs a) {
    const int64_t nh = int64_t(a.n) * a.H;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nh; e += int64_t(gridDim.x) * blockDim.x) {
        double m = -DBL_MAX;
        for (int s = 0; s < a.nsplit; ++s) m = max(m, a.m_part[int64_t(s) * nh + e]);
        double l = 0.0;
        for (int s = 0; s < a.nsplit; ++s) {
            const double ms = a.m_part[int64_t(s) * nh + e];
            if (ms == -DBL_MAX) continue;
            l += a.l_part[int64_t(s) * nh + e] * exp(ms - m);
        }
        a.m_fin[e] = m;
        a.l_fin[e] = l;
    }
}

// ---------------------------------------------------------------- pass 2 --
template <typename TQ, typename TKV, typename ACC>
__global__ void __launch_bounds__(NT)
attn_ctx_kernel(AttnArgs a, ACC scale) {
    extern __shared__ __align__(16) uint8_t smraw[];
    Smem<ACC>& sm = *reinterpret_cast<Smem<ACC>*>(smraw);
    const Tile tl = tile_of(a.rows, a.key_lo, a.n, blockIdx.x);
    const int h = blockIdx.y, sp = blockIdx.z;
    const int lo = max(a.split_lo[sp], tl.klo), hi = min(a.split_hi[sp], tl.tmax + 1);
    const int r = threadIdx.x / 16, c = threadIdx.x % 16;
    const int off = h * a.dh;
    load_rows(sm.rowt, sm.rowlo, a, tl);
    load_q(sm, static_cast<const TQ*>(a.q), tl.i0, tl.nrows, a.d, off, a.dh);
    ACC mrow = ACC(0), inv = ACC(0);
    if (r < tl.nrows) {
        const int64_t o = int64_t(tl.i0 + r) * a.H + h;
        mrow = ACC(a.m_fin[o]);
        inv = ACC(1.0 / a.l_fin[o]);  // p = e * (1/sum), prefill.hpp:148-151
    }
    ACC o_acc[MAXDH / 16];
#pragma unroll
    for (int j = 0; j < MAXDH / 16; ++j) o_acc[j] = ACC(0);
    for (int k0 = lo; k0 < hi; k0 += KC) {
        const int nk = min(KC, hi - k0);
        __syncthreads();
        load_chunk(sm.k, static_cast<const TKV*>(a.k), k0, nk, a.d, off, a.dh);
        load_chunk(sm.v, static_cast<const TKV*>(a.v), k0, nk, a.d, off, a.dh);
        __syncthreads();
        ACC s[4];
        scores4(sm, r, c, a.dh, scale, s);
        const int t = sm.rowt[r], klo = sm.rowlo[r];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int key = k0 + c + 16 * kk;
            const bool ok = (c + 16 * kk < nk) && key <= t && key >= klo;
            sm.p[r * KC + c + 16 * kk] = ok ? mul_rn(ex(sub_rn(s[kk], mrow)), inv) : ACC(0);
        }
        __syncthreads();
        for (int kk = 0; kk < nk; ++kk) {
            const ACC pk = sm.p[r * KC + kk];
#pragma unroll
            for (int jj = 0; jj < MAXDH / 16; ++jj) {
                const int j = c + 16 * jj;
                if (j < a.dh) o_acc[jj] = fma(pk, ACC(sm.v[kk * (MAXDH + 1) + j]), o_acc[jj]);
            }
        }
    }
    if (r < tl.nrows) {
        const int64_t row = tl.i0 + r;
#pragma unroll
        for (int jj = 0; jj < MAXDH / 16; ++jj) {
            const int j = c + 16 * jj;
            if (j >= a.dh) continue;
            if (a.nsplit == 1) {
                if (a.ctx) a.ctx[row * a.d + off + j] = float(o_acc[jj]);
                if (a.ctx_bf16) a.ctx_bf16[row * a.d + off + j] = __float2bfloat16_rn(float(o_acc[jj]));
            } else {
                a.o_part[(int64_t(sp) * a.n + row) * a.d + off + j] = double(o_acc[jj]);
            }
        }
    }
}

__global__ void ctx_combine_kernel(AttnArgs a) {
    const int64_t nd = int64_t(a.n) * a.d;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nd; e += int64_t(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < a.nsplit; ++s) acc += a.o_part[int64_t(s) * nd + e];
        if (a.ctx) a.ctx[e] = float(acc);
        if (a.ctx_bf16) a.ctx_bf16[e] = __float2bfloat16_rn(float(acc));
    }
}

// ---------------------------------------------------------------- pass 3 --
template <typename TQ, typename TKV, typename ACC, typename TB>
__global__ void __launch_bounds__(NT)
attn_bins_kernel(AttnArgs a, ACC scale, ACC inv_heads) {
    extern __shared__ __align__(16) uint8_t smraw[];
    Smem<ACC>& sm = *reinterpret_cast<Smem<ACC>*>(smraw);
    __shared__ ACC pm[RT * KC];
    const Tile tl = tile_of(a.rows, a.key_lo, a.n, blockIdx.x);
    const int sp = blockIdx.y;
    const int lo = max(a.split_lo[sp], tl.klo), hi = min(a.split_hi[sp], tl.tmax + 1);
    if (lo >= hi) return;  // split entirely after every row of the tile
    const int r = threadIdx.x / 16, c = threadIdx.x % 16;
    load_rows(sm.rowt, sm.rowlo, a, tl);
    TB* rowbin = static_cast<TB*>(a.rowbin);
    // running bin of the row owned by thread r (< RT) across chunks
    int cur = -1;
    ACC run = ACC(0);
    for (int k0 = lo; k0 < hi; k0 += KC) {
        const int nk = min(KC, hi - k0);
        for (int e = threadIdx.x; e < RT * KC; e += NT) pm[e] = ACC(0);
        for (int h = 0; h < a.H; ++h) {
            const int off = h * a.dh;
            __syncthreads();
            load_q(sm, static_cast<const TQ*>(a.q), tl.i0, tl.nrows, a.d, off, a.dh);
            load_chunk(sm.k, static_cast<const TKV*>(a.k), k0, nk, a.d, off, a.dh);
            __syncthreads();
            ACC s[4];
            scores4(sm, r, c, a.dh, scale, s);
            const int t = sm.rowt[r], klo = sm.rowlo[r];
            if (r < tl.nrows) {
                const int64_t o = int64_t(tl.i0 + r) * a.H + h;
                const ACC mrow = ACC(a.m_fin[o]);
                const ACC inv = ACC(1.0 / a.l_fin[o]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int key = k0 + c + 16 * kk;
                    if ((c + 16 * kk < nk) && key <= t && key >= klo)
                        pm[r * KC + c + 16 * kk] = add_rn(pm[r * KC + c + 16 * kk], mul_rn(mul_rn(ex(sub_rn(s[kk], mrow)), inv), inv_heads));
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < tl.nrows) {
            const int rr = threadIdx.x;
            const int t = sm.rowt[rr];
            const int64_t rowoff = int64_t(tl.i0 + rr) * a.S;
            const int klo = sm.rowlo[rr];
            for (int kk = 0; kk < nk; ++kk) {
                const int key = k0 + kk;
                if (key > t) break;
                if (key < klo) continue;
                const int dst = a.row_seg[key];
                if (dst < 0) continue;  // mass on query tokens is not summarised (prefill.hpp:283)
                if (dst != cur) {
                    if (cur >= 0) rowbin[rowoff + cur] = TB(run);
                    cur = dst;
                    run = ACC(0);
                }
                run += pm[rr * KC + kk];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < tl.nrows && cur >= 0) rowbin[int64_t(tl.i0 + threadIdx.x) * a.S + cur] = TB(run);
}

template <typename TQ, typename TKV, typename ACC, typename TB>
void run_attention(const AttnArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    if (a.dh > MAXDH) raise(KEEP_ERR_CONFIG, "head_dim > 128 not supported");
    const int tiles = static_cast<int>(ceil_div(a.n, RT));
    const size_t smem = sizeof(Smem<ACC>);
    const ACC scale = ACC(1.0 / std::sqrt(double(a.dh)));  // prefill.hpp:129
    auto k1 = attn_stats_kernel<TQ, TKV, ACC>;
    auto k2 = attn_ctx_kernel<TQ, TKV, ACC>;
    auto k3 = attn_bins_kernel<TQ, TKV, ACC, TB>;
    KEEP_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    KEEP_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    KEEP_CUDA(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 g1(tiles, a.H, a.nsplit);
    k1<<<g1, NT, smem, st>>>(a, scale);
    KEEP_LAUNCH_CHECK();
    const int64_t nh = int64_t(a.n) * a.H;
    stats_combine_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(nh, 256), kNumSMs * 8)), 256, 0, st>>>(a);
    KEEP_LAUNCH_CHECK();
    k2<<<g1, NT, smem, st>>>(a, scale);
    KEEP_LAUNCH_CHECK();
    if (a.nsplit > 1) {
        const int64_t nd = int64_t(a.n) * a.d;
        ctx_combine_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(nd, 256), kNumSMs * 16)), 256, 0, st>>>(a);
        KEEP_LAUNCH_CHECK();
    }
    if (a.with_bins) {
        dim3 g3(tiles, a.nsplit);
        k3<<<g3, NT, smem, st>>>(a, scale, ACC(a.inv_heads));
        KEEP_LAUNCH_CHECK();
    }
}

}  // namespace

void launch_stats_combine(const AttnArgs& a, cudaStream_t st) {
    const int64_t nh = int64_t(a.n) * a.H;
    stats_combine_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(nh, 256), kNumSMs * 8)), 256, 0, st>>>(a);
    KEEP_LAUNCH_CHECK();
}

void launch_ctx_combine(const AttnArgs& a, cudaStream_t st) {
    const int64_t nd = int64_t(a.n) * a.d;
    ctx_combine_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(nd, 256), kNumSMs * 16)), 256, 0, st>>>(a);
    KEEP_LAUNCH_CHECK();
}

// KEEP_PARITY_ATTN=simt: the scalar-DFMA kernels above (A/B reference)
bool parity_attention_dmma(int dh) {
    static const bool simt = [] {
        const char* e = std::getenv("KEEP_PARITY_ATTN");
        return e && !std::strcmp(e, "simt");
    }();
    return !simt && attention_dmma_fits(dh);
}

void launch_attention_parity(const AttnArgs& a, cudaStream_t st) {
    if (!a.exact && parity_attention_dmma(a.dh)) launch_attention_parity_dmma(a, st);
    else run_attention<float, float, double, double>(a, st);
}

void launch_attention_fast(const AttnArgs& a, cudaStream_t st) {
    run_attention<__nv_bfloat16, __nv_bfloat16, float, float>(a, st);
}

}  // namespace keep_b200
