// attn_decode.cu -- K5 for the few-row layers (FAST, head_dim 128, no summary).
//
// Once the walk has ended (C3: layers 20..47) a layer computes only the query
// rows: 8 rows x H heads against the whole merged KV.  That is HBM-bound --
// every K and V byte is read once for 8 rows -- so the two-pass 128-row
// tensor-core kernel (K read twice, 120 of 128 MMA rows padding) is the wrong
// shape.  This is single-pass split-K flash decoding:
//   grid (head, key split); per CTA one producer warp streams 64-key stages of
//   K and V (four 64x64 TMA boxes, 128-byte swizzle, 3 stages, 2 CTAs / SM,
//   ~190 KB in flight per SM) and four consumer warps each take 16 keys of a
//   stage: S = Q K^T and O += P V on mma.sync m16n8k16 (bf16 in, fp32 out;
//   the 16-row tile holds the <= 16 rows, the MMA is never the bound here),
//   online softmax in the exp2 domain (q arrives pre-scaled by log2 e / sqrt dh).
//   The four warps' (m, l, O) merge in shared memory; several splits merge in
//   decode_combine.
// Algorithmic bytes per launch: 2 * kv_hi * d * 2 (K + V once) + q + ctx.
// Reference semantics: attention_row (prefill.hpp:124-159) for each row,
// keys 0..t -- the causal limit comes from the row's position.
#include <cuda_bf16.h>

#include "engine.hpp"
#include "tc_common.cuh"

namespace keep_b200 {
namespace {

using namespace tc;

constexpr int DK = 64;                  // keys per stage
constexpr int DST = 3;                  // stages
constexpr int DWARPS = 4;               // consumer warps (16 keys of each stage)
constexpr int DTHREADS = (DWARPS + 1) * 32;
constexpr int DH = 128;
constexpr int BOX_B = DK * 64 * 2;      // one TMA box: 64 keys x 64 dh (bf16) = 8 KB
constexpr int STAGE_B = 4 * BOX_B;      // K dh 0-63, K dh 64-127, V dh 0-63, V dh 64-127
constexpr int RED_OFF = DST * STAGE_B;  // barriers + per-warp row stats after the stages
constexpr int SMEM_B = 1024 + RED_OFF + 2 * DST * 8 + 3 * DWARPS * 16 * 4 + 16 * 4;

constexpr int kMaxMulti = 64;  // queries per multi-instance launch

struct DecArgs {
    int n, H, d;            // rows (<= 64: blocks of 16 on grid z), this rank's heads, row stride (= H * 128)
    int kv_hi;              // keys [0, kv_hi) are visible to some row
    int nsplit, cps;        // key splits, 64-key stages per split
    const __nv_bfloat16* q; // [n x d], pre-scaled by log2(e) / sqrt(128)
    const int32_t* rows;    // [n] ascending positions (causal limits)
    float* m_part;          // [nsplit x n x H]
    float* l_part;
    float* o_part;          // [nsplit x n x d]
    __nv_bfloat16* ctx;     // [n x d]
    // MULTI (a batch's all-reused queries, one per grid x): keys [0, kv_mem)
    // come from the shared memory sheet (mk, mv), keys [kv_mem, kv_hi) -- the
    // query's own rows -- from (mk2, mv2) at row qrow0[z] + key - kv_mem; the
    // query's q / ctx rows start at qoff[z]
    int kv_mem;
    int qrow0[kMaxMulti];
    int qoff[kMaxMulti];
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t ld_q32(const __nv_bfloat16* q, int r, int n, int64_t off) {
    return r < n ? *reinterpret_cast<const uint32_t*>(q + off) : 0u;
}

template <bool MULTI>
__global__ void __launch_bounds__(DTHREADS, 2)
attn_decode_kernel(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
                   const __grid_constant__ CUtensorMap mk2, const __grid_constant__ CUtensorMap mv2,
                   const __grid_constant__ DecArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + RED_OFF);
    uint64_t* empty = full + DST;
    float* red_m = reinterpret_cast<float*>(empty + DST);  // [DWARPS][16]
    float* red_l = red_m + DWARPS * 16;
    float* row_M = red_l + DWARPS * 16;                    // [16] merged max
    float* row_L = row_M + 16;                             // [16] merged sum

    // single: grid (head, split, 16-row block); MULTI: grid (query, head), one split
    const int h = MULTI ? blockIdx.y : blockIdx.x, sp = MULTI ? 0 : blockIdx.y;
    const int z = MULTI ? blockIdx.x : 0;
    const int r_off = MULTI ? 0 : blockIdx.z * 16;  // this CTA's block of (up to) 16 rows
    const int kv_mem = MULTI ? a.kv_mem : a.kv_hi;   // keys served by (mk, mv)
    const int nch_total = int(ceil_div(kv_mem, DK));
    const int c0 = sp * a.cps;
    const int nch_mem = MULTI ? nch_total : max(0, min(nch_total, c0 + a.cps) - c0);
    const int nch = nch_mem + (MULTI ? int(ceil_div(a.kv_hi - kv_mem, DK)) : 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < DST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], DWARPS);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == DWARPS) {  // producer
        if (lane == 0) {
            prefetch_map(&mk);
            prefetch_map(&mv);
            for (int j = 0; j < nch; ++j) {
                const int s = j % DST;
                if (j >= DST) mbar_wait(&empty[s], uint32_t((j / DST) - 1) & 1u);
                mbar_expect_tx(&full[s], STAGE_B);
                uint8_t* st = sm + s * STAGE_B;
                const bool own = MULTI && j >= nch_mem;  // the query's own key rows
                const CUtensorMap* k_map = own ? &mk2 : &mk;
                const CUtensorMap* v_map = own ? &mv2 : &mv;
                const int key = own ? a.qrow0[z] + (j - nch_mem) * DK : (c0 + j) * DK;
                tma_load_2d(st, k_map, &full[s], h * DH, key);
                tma_load_2d(st + BOX_B, k_map, &full[s], h * DH + 64, key);
                tma_load_2d(st + 2 * BOX_B, v_map, &full[s], h * DH, key);
                tma_load_2d(st + 3 * BOX_B, v_map, &full[s], h * DH + 64, key);
            }
        }
        return;
    }

    const int g = lane >> 2, i4 = lane & 3;
    const int n = min(16, a.n - r_off);  // rows of this block
    const int q_off = MULTI ? a.qoff[z] : r_off;
    const __nv_bfloat16* qblk = a.q + int64_t(q_off) * a.d;
    const int32_t* rows = a.rows + r_off;
    // Q fragments (A operand, rows g and g + 8; rows >= n are zero)
    uint32_t qa[8][4];
    {
        const int64_t b0 = int64_t(g) * a.d + h * DH + 2 * i4, b1 = int64_t(g + 8) * a.d + h * DH + 2 * i4;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            qa[ks][0] = ld_q32(qblk, g, n, b0 + ks * 16);
            qa[ks][1] = ld_q32(qblk, g + 8, n, b1 + ks * 16);
            qa[ks][2] = ld_q32(qblk, g, n, b0 + ks * 16 + 8);
            qa[ks][3] = ld_q32(qblk, g + 8, n, b1 + ks * 16 + 8);
        }
    }
    const int t0 = g < n ? rows[g] : -1, t1 = g + 8 < n ? rows[g + 8] : -1;
    const int tmin = rows[0];
    float o[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int j = 0; j < nch; ++j) {
        const int s = j % DST;
        mbar_wait(&full[s], uint32_t(j / DST) & 1u);
        const uint32_t sb = smem_u32(sm + s * STAGE_B);
        const bool own = MULTI && j >= nch_mem;
        // first key of this warp's 16, and the end of the keys its source holds
        const int kb = (own ? kv_mem + (j - nch_mem) * DK : (c0 + j) * DK) + warp * 16;
        const int klim = own ? a.kv_hi : kv_mem;
        float sc[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
            const int kr = warp * 16 + nt * 8 + (lane & 7);
#pragma unroll
            for (int kq = 0; kq < 4; ++kq) {  // 32 dh per x4: matrices dh0, +8, +16, +24
                const int half = kq >> 1, chunk = ((kq & 1) << 2) + (lane >> 3);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sb + half * BOX_B + swz(kr, chunk), b0, b1, b2, b3);
                mma16816(sc[nt], qa[2 * kq], b0, b1);
                mma16816(sc[nt], qa[2 * kq + 1], b2, b3);
            }
        }
        if (kb + 15 > tmin || kb + 15 >= klim) {  // a causal limit or the source's end inside these keys
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int key = kb + nt * 8 + 2 * i4 + e;
                    if (key > t0 || key >= klim) sc[nt][e] = -INFINITY;
                    if (key > t1 || key >= klim) sc[nt][2 + e] = -INFINITY;
                }
        }
        float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
        float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float u0 = mn0 == -INFINITY ? 0.f : mn0, u1 = mn1 == -INFINITY ? 0.f : mn1;
        const float al0 = ex2(m0 - u0), al1 = ex2(m1 - u1);
        m0 = mn0;
        m1 = mn1;
        float p[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            p[nt][0] = ex2(sc[nt][0] - u0);
            p[nt][1] = ex2(sc[nt][1] - u0);
            p[nt][2] = ex2(sc[nt][2] - u1);
            p[nt][3] = ex2(sc[nt][3] - u1);
        }
        l0 = l0 * al0 + (p[0][0] + p[0][1] + p[1][0] + p[1][1]);
        l1 = l1 * al1 + (p[0][2] + p[0][3] + p[1][2] + p[1][3]);
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
            o[nt][0] *= al0;
            o[nt][1] *= al0;
            o[nt][2] *= al1;
            o[nt][3] *= al1;
        }
        // P as the A operand of P.V (the m16n8 accumulator layout of two key
        // tiles is the m16k16 A layout)
        const uint32_t pa[4] = {pack_bf16(p[0][0], p[0][1]), pack_bf16(p[0][2], p[0][3]), pack_bf16(p[1][0], p[1][1]),
                                pack_bf16(p[1][2], p[1][3])};
        {
            const int mat = lane >> 3;
            const int kr = warp * 16 + ((mat & 1) << 3) + (lane & 7);
#pragma unroll
            for (int nd = 0; nd < 8; ++nd) {  // 16 dh per x4.trans
                const int dh = nd * 16 + ((mat >> 1) << 3);
                uint32_t v0, v1, v2, v3;
                ldsm_x4_t(sb + (2 + (dh >> 6)) * BOX_B + swz(kr, (dh & 63) >> 3), v0, v1, v2, v3);
                mma16816(o[2 * nd], pa, v0, v1);
                mma16816(o[2 * nd + 1], pa, v2, v3);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    // merge the four warps (each saw 16 of every 64 keys)
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    if (i4 == 0) {
        red_m[warp * 16 + g] = m0;
        red_m[warp * 16 + g + 8] = m1;
        red_l[warp * 16 + g] = l0;
        red_l[warp * 16 + g + 8] = l1;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // also: every stage consumed
    float M0 = -INFINITY, M1 = -INFINITY;
#pragma unroll
    for (int w = 0; w < DWARPS; ++w) {
        M0 = fmaxf(M0, red_m[w * 16 + g]);
        M1 = fmaxf(M1, red_m[w * 16 + g + 8]);
    }
    const float f0 = m0 == -INFINITY ? 0.f : ex2(m0 - M0), f1 = m1 == -INFINITY ? 0.f : ex2(m1 - M1);
    if (warp == 0 && i4 == 0) {
        float L0 = 0.f, L1 = 0.f;
#pragma unroll
        for (int w = 0; w < DWARPS; ++w) {
            const float mw0 = red_m[w * 16 + g], mw1 = red_m[w * 16 + g + 8];
            if (mw0 != -INFINITY) L0 += red_l[w * 16 + g] * ex2(mw0 - M0);
            if (mw1 != -INFINITY) L1 += red_l[w * 16 + g + 8] * ex2(mw1 - M1);
        }
        row_M[g] = M0;
        row_M[g + 8] = M1;
        row_L[g] = L0;
        row_L[g + 8] = L1;
    }
    float* ob = reinterpret_cast<float*>(sm);  // [DWARPS][16][128] over the (consumed) stages
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
        const int col = nt * 8 + 2 * i4;
        *reinterpret_cast<float2*>(ob + (warp * 16 + g) * DH + col) = make_float2(o[nt][0] * f0, o[nt][1] * f0);
        *reinterpret_cast<float2*>(ob + (warp * 16 + g + 8) * DH + col) = make_float2(o[nt][2] * f1, o[nt][3] * f1);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int tid = threadIdx.x;
    for (int e = tid; e < 16 * DH; e += DWARPS * 32) {
        const int r = e / DH, c = e % DH;
        if (r >= n) break;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < DWARPS; ++w) acc += ob[(w * 16 + r) * DH + c];
        const int64_t col = int64_t(h) * DH + c;
        const int64_t rg = q_off + r;  // row of the launch
        if (a.nsplit == 1) {
            const float L = row_L[r];
            a.ctx[rg * a.d + col] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
        } else {
            a.o_part[(int64_t(sp) * a.n + rg) * a.d + col] = acc;
            if (c == 0) {
                a.m_part[(int64_t(sp) * a.n + rg) * a.H + h] = row_M[r];
                a.l_part[(int64_t(sp) * a.n + rg) * a.H + h] = row_L[r];
            }
        }
    }
}

__global__ void decode_combine(const float* __restrict__ m_part, const float* __restrict__ l_part,
                               const float* __restrict__ o_part, int nsplit, int n, int H, int d,
                               __nv_bfloat16* __restrict__ ctx) {
    const int64_t nd = int64_t(n) * d;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nd; e += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(e / d), c = int(e % d), h = c / DH;
        float M = -INFINITY;
        for (int s = 0; s < nsplit; ++s) M = fmaxf(M, m_part[(int64_t(s) * n + r) * H + h]);
        float L = 0.f, O = 0.f;
        if (M != -INFINITY)
            for (int s = 0; s < nsplit; ++s) {
                const float ms = m_part[(int64_t(s) * n + r) * H + h];
                if (ms == -INFINITY) continue;
                const float w = ex2(ms - M);
                L += l_part[(int64_t(s) * n + r) * H + h] * w;
                O += o_part[(int64_t(s) * n + r) * d + c] * w;
            }
        ctx[e] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    }
}

}  // namespace

int decode_splits(int n_heads, int kv_hi) {
    const int nch = int(ceil_div(kv_hi, DK));
    const int slots = 2 * kNumSMs;  // two CTAs per SM
    int ns = std::max(1, std::min(slots / std::max(n_heads, 1), nch / 4));
    const int cps = int(ceil_div(nch, ns));
    return int(ceil_div(nch, cps));
}

bool decode_attention_fits(int n) { return n >= 1 && n <= 64; }

int launch_attention_decode(const AttnTcLaunch& L, int kv_hi, cudaStream_t st) {
    const int n = L.n;
    if (n == 0 || kv_hi <= 0) return 0;
    if (n > 64) raise(KEEP_ERR_CONFIG, "decode attention takes at most 64 rows");
    smem_attr(attn_decode_kernel<false>, SMEM_B);
    smem_attr(attn_decode_kernel<true>, SMEM_B);
    DecArgs a{};
    a.n = n;
    a.H = L.H;
    a.d = L.d;
    a.kv_hi = kv_hi;
    a.nsplit = decode_splits(L.H, kv_hi);
    a.cps = int(ceil_div(ceil_div(kv_hi, DK), a.nsplit));
    a.q = static_cast<const __nv_bfloat16*>(L.q);
    a.rows = L.rows;
    a.m_part = L.m_part;
    a.l_part = L.l_part;
    a.o_part = L.o_part;
    a.ctx = L.ctx;
    const CUtensorMap mk = make_map_bf16(L.k, kv_hi, L.d, L.d, DK);
    const CUtensorMap mv = make_map_bf16(L.v, kv_hi, L.d, L.d, DK);
    attn_decode_kernel<false><<<dim3(unsigned(L.H), unsigned(a.nsplit), unsigned(ceil_div(n, 16))), DTHREADS, SMEM_B,
                                st>>>(mk, mv, mk, mv, a);
    KEEP_LAUNCH_CHECK();
    if (a.nsplit == 1) return 1;
    const int64_t nd = int64_t(n) * L.d;
    decode_combine<<<unsigned(std::min<int64_t>(ceil_div(nd, 256), kNumSMs * 4)), 256, 0, st>>>(
        L.m_part, L.l_part, L.o_part, a.nsplit, n, L.H, L.d, L.ctx);
    KEEP_LAUNCH_CHECK();
    return 2;
}

int launch_attention_decode_multi(const DecodeMulti& M, cudaStream_t st) {
    const int nq = int(M.qoff.size());
    if (nq == 0) return 0;
    if (M.qlen < 1 || M.qlen > 16) raise(KEEP_ERR_CONFIG, "multi decode takes 1..16 query rows per query");
    smem_attr(attn_decode_kernel<false>, SMEM_B);
    smem_attr(attn_decode_kernel<true>, SMEM_B);
    const CUtensorMap mk = make_map_bf16(M.k_mem, M.kv_mem, M.d, M.d, DK);
    const CUtensorMap mv = make_map_bf16(M.v_mem, M.kv_mem, M.d, M.d, DK);
    const CUtensorMap mk2 = make_map_bf16(M.k_own, M.own_rows, M.d, M.d, DK);
    const CUtensorMap mv2 = make_map_bf16(M.v_own, M.own_rows, M.d, M.d, DK);
    int launched = 0;
    for (int q0 = 0; q0 < nq; q0 += kMaxMulti) {
        const int nz = std::min(kMaxMulti, nq - q0);
        DecArgs a{};
        a.n = M.qlen;
        a.H = M.H;
        a.d = M.d;
        a.kv_mem = M.kv_mem;
        a.kv_hi = M.kv_mem + M.qlen;
        a.nsplit = 1;
        a.cps = int(ceil_div(M.kv_mem, DK));
        a.q = static_cast<const __nv_bfloat16*>(M.q);
        a.rows = M.rows;
        a.ctx = M.ctx;
        for (int z = 0; z < nz; ++z) {
            a.qrow0[z] = M.qrow0[q0 + z];
            a.qoff[z] = M.qoff[q0 + z];
        }
        // queries fastest: the CTAs of one head run together and share its K / V through L2
        attn_decode_kernel<true><<<dim3(unsigned(nz), unsigned(M.H)), DTHREADS, SMEM_B, st>>>(mk, mv, mk2, mv2, a);
        KEEP_LAUNCH_CHECK();
        ++launched;
    }
    return launched;
}

}  // namespace keep_b200
