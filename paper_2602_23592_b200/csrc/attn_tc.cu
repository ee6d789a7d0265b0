// attn_tc.cu -- K5 on the tcgen05 tensor cores (FAST numerics, head_dim 128).
//
// The segment summary needs NORMALISED probabilities (prefill.hpp:138-152),
// so attention runs as two warp-specialised passes over 128-row x 128-key
// tiles, grid (row tiles, heads, key splits).  Both compute S = Q K^T with
// tcgen05.mma into TMEM (double buffered: the MMA of chunk i+1 overlaps the
// softmax of chunk i):
//
//   STATS  per-row running max / sum of exp2 (log2 domain) -> partials per
//          split, combined in split order.
//   CTX    p = exp2(s - m) / l, written as bf16 into a 128B-swizzled smem tile;
//          O += P . V with a second tcgen05.mma (V^T staged K-major); O read
//          back with tcgen05.ld.  The same fp32 p feed the segment summary
//          (prefill.hpp:266-288): each row thread sums its keys per
//          destination segment in key order (segment boundaries are the same
//          for every row of the chunk, so the branches are warp-uniform), the
//          tile's rows are reduced per source segment through shared memory,
//          and one fp64 atomic per (source, destination) pair per tile and
//          head lands in the raw summary (mass on query keys and on the row's
//          own segment is dropped, prefill.hpp:283-287).
//
// Warp roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2
// TMEM allocator, warps 4-7 softmax / summary / epilogue (thread = row = TMEM
// lane).
#include "engine.hpp"
#include "tc_common.cuh"

#include <cfloat>
#include <type_traits>

namespace keep_b200 {

using namespace tc;

namespace {

constexpr int TM = 128;  // rows per tile
constexpr int TK = 128;  // keys per chunk
constexpr int DH = 128;  // head dim (two 64-wide swizzle atoms)
constexpr int NTHR = 256;
constexpr uint32_t TILE_BYTES = TM * DH * 2;  // 32 KB: [128 x 128] bf16 as 2 boxes of 64 columns
constexpr uint32_t BOX_BYTES = TILE_BYTES / 2;
constexpr uint32_t IDESC = instr_desc(128, 128);
constexpr int PART_SEGS = 24;                 // destination segments per binning pass
constexpr int PART_STRIDE = PART_SEGS + 1;    // floats per row: slot PART_SEGS is a trash slot

enum { MODE_STATS = 0, MODE_CTX = 1, MODE_FLASH = 2 };

struct TcArgs {
    int n, T, H, d, S;
    int nsplit;
    const int32_t* split_lo;
    const int32_t* split_hi;
    const int32_t* rows;
    const int32_t* row_seg;
    const int32_t* key_lo;  // nullable (block-diagonal refresh)
    float scale_log2;       // log2(e) / sqrt(dh)
    float inv_heads;
    float* m_part;          // [nsplit][n][H] log2-domain max
    float* l_part;          // [nsplit][n][H]
    const float* m_fin;     // [n][H]
    const float* inv_l;     // [n][H] 1 / sum
    float* o_part;          // [nsplit][n][d] (nsplit > 1)
    __nv_bfloat16* ctx;     // [n][d]
    double* qts_raw;        // [S]      (nullptr: no summary)
    double* sts_raw;        // [S x S]
    const int4* chunk_tab;  // [ceil(T/128) x 2] per 128-key chunk: {d0, nseg, -, -}, {mask0..3}
    int dbg;                // A/B timing aid (KEEP_DEBUG_ATTN): 1 = bins from hi only, 2 = no P.V
    int norm_end;           // v2 without a summary: STATS finds only the max; CTX sums l and
                            // normalises O at the end (no exp in STATS)
};

template <int MODE>
struct Layout {
    static constexpr int ST = MODE == MODE_STATS ? 4 : 2;  // pipeline stages
    static constexpr uint32_t STAGE = MODE == MODE_STATS ? TILE_BYTES : 2 * TILE_BYTES;  // K (+ V^T)
    static constexpr uint32_t Q_OFF = 0;
    static constexpr uint32_t STAGE_OFF = TILE_BYTES;
    static constexpr uint32_t P_OFF = STAGE_OFF + ST * STAGE;             // CTX: one P tile
    static constexpr uint32_t PART_OFF = P_OFF + TILE_BYTES;              // CTX: 2 x partial bins [128][17] f32
    static constexpr uint32_t SEG_OFF = PART_OFF + 2 * TM * PART_STRIDE * 4;  // (unused)
    static constexpr uint32_t GRP_OFF = SEG_OFF;                          // CTX: row groups [130] + sources [129]
    static constexpr uint32_t MSK_OFF = GRP_OFF + (2 * TM + 4) * 4;       // CTX: row-group ballots [4] u32
    static constexpr uint32_t BAR_OFF = MODE == MODE_CTX ? ((MSK_OFF + 16 + 7) & ~7u) : P_OFF;
    static constexpr size_t SMEM = size_t(BAR_OFF) + 256 + 1024;
    static constexpr uint32_t TMEM_COLS = MODE == MODE_CTX ? 512 : 256;
};

// P tile 16-byte chunk (row r, keys 8*chunk16 .. +8) in the 128B-swizzled
// K-major layout TMA would produce: box = chunk16 / 8, slot = chunk16 % 8.
__device__ __forceinline__ uint32_t p_chunk_off(int r, int chunk16) {
    const int box = chunk16 >> 3, c = chunk16 & 7;
    return uint32_t(box) * BOX_BYTES + uint32_t(r >> 3) * 1024u + uint32_t(r & 7) * 128u +
           (uint32_t(c ^ (r & 7)) << 4);
}

__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int ks) {
    // k-step ks of 16 elements across the two 64-wide boxes of a tile
    return smem_desc(tile + uint32_t(ks >> 2) * BOX_BYTES + uint32_t(ks & 3) * 32u);
}

__device__ __forceinline__ void named_sync_softmax() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// one MUFU.EX2 (flush-to-zero; inputs are <= 0 after max subtraction)
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MODE>
__global__ void __launch_bounds__(NTHR, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmVt, TcArgs a) {
    using LY = Layout<MODE>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared space
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + LY::BAR_OFF);
    uint64_t* full = bar;            // [ST]
    uint64_t* empty = bar + 4;       // [ST]
    uint64_t* s_full = bar + 8;      // [2]
    uint64_t* s_empty = bar + 10;    // [2]
    uint64_t* p_full = bar + 12;
    uint64_t* p_empty = bar + 13;
    uint64_t* q_full = bar + 14;
    uint64_t* o_full = bar + 15;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.x * TM;
    const int nrows = min(TM, a.n - i0);
    const int head = blockIdx.y, sp = blockIdx.z;
    const int tmax = a.rows[i0 + nrows - 1];
    const int tklo = a.key_lo ? a.key_lo[a.rows[i0]] : 0;
    const int lo = max(a.split_lo[sp], tklo);
    const int hi = min(a.split_hi[sp], tmax + 1);
    // chunk base rounded down to 8 keys: a TMA box may only start on a
    // 16-byte boundary of the innermost dimension (the V^T loads index keys
    // there); keys below lo are masked
    const int kbase = lo & ~7;
    const int niter = hi > lo ? int(ceil_div(hi - kbase, TK)) : 0;

    if (warp == 0 && lane == 0) {
        prefetch_map(&tmQ);
        prefetch_map(&tmK);
        if (MODE == MODE_CTX) prefetch_map(&tmVt);
        for (int s = 0; s < LY::ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_empty[b], 4);
        }
        mbar_init(p_full, 4);
        mbar_init(p_empty, 1);
        mbar_init(q_full, 1);
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, LY::TMEM_COLS);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_s0 = tmem, tm_o = tmem + 256;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA
        if (lane == 0 && niter > 0) {
            mbar_expect_tx(q_full, TILE_BYTES);
            tma_load_2d(sm + LY::Q_OFF, &tmQ, q_full, head * DH, i0);
            tma_load_2d(sm + LY::Q_OFF + BOX_BYTES, &tmQ, q_full, head * DH + 64, i0);
            for (int it = 0; it < niter; ++it) {
                const int s = it % LY::ST;
                mbar_wait(&empty[s], ((it / LY::ST) & 1) ^ 1);
                uint8_t* st = sm + LY::STAGE_OFF + s * LY::STAGE;
                const int k0 = kbase + it * TK;
                mbar_expect_tx(&full[s], LY::STAGE);
                tma_load_2d(st, &tmK, &full[s], head * DH, k0);
                tma_load_2d(st + BOX_BYTES, &tmK, &full[s], head * DH + 64, k0);
                if (MODE == MODE_CTX) {
                    tma_load_2d(st + TILE_BYTES, &tmVt, &full[s], k0, head * DH);
                    tma_load_2d(st + TILE_BYTES + BOX_BYTES, &tmVt, &full[s], k0 + 64, head * DH);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA
        if (lane == 0 && niter > 0) {
            mbar_wait(q_full, 0);
            auto pv = [&](int j) {  // O += P_j . V_j  (CTX only)
                mbar_wait(p_full, j & 1);
                fence_after();
                const uint32_t pt = smem_u32(sm + LY::P_OFF);
                const uint32_t vt = smem_u32(sm + LY::STAGE_OFF + (j % LY::ST) * LY::STAGE + TILE_BYTES);
#pragma unroll
                for (int ks = 0; ks < TK / 16; ++ks)
                    umma(tm_o, desc_k(pt, ks), desc_k(vt, ks), IDESC, (j | ks) ? 1u : 0u);
                umma_commit(p_empty);
                umma_commit(&empty[j % LY::ST]);
            };
            const uint32_t qt = smem_u32(sm + LY::Q_OFF);
            for (int it = 0; it < niter; ++it) {
                const int s = it % LY::ST, b = it & 1;
                mbar_wait(&full[s], (it / LY::ST) & 1);
                mbar_wait(&s_empty[b], ((it >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t kt = smem_u32(sm + LY::STAGE_OFF + s * LY::STAGE);
#pragma unroll
                for (int ks = 0; ks < DH / 16; ++ks)
                    umma(tm_s0 + uint32_t(b * TK), desc_k(qt, ks), desc_k(kt, ks), IDESC, ks ? 1u : 0u);
                umma_commit(&s_full[b]);
                if (MODE == MODE_STATS) umma_commit(&empty[s]);
                if (MODE == MODE_CTX && it > 0) pv(it - 1);
            }
            if (MODE == MODE_CTX) {
                pv(niter - 1);
                umma_commit(o_full);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------ softmax / summary / epilogue
        const int q = warp & 3;
        const int tid = threadIdx.x - 128;
        const int r = q * 32 + lane;  // tile row == TMEM lane
        const bool rvalid = r < nrows;
        const int row = i0 + r;
        const int t = rvalid ? a.rows[row] : -1;
        const int klo = max(lo, rvalid && a.key_lo ? a.key_lo[t] : 0);  // first visible key
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const float scale = a.scale_log2;
        float m_run = -FLT_MAX, l_run = 0.f;  // STATS
        float m_row = 0.f, il_row = 0.f;      // CTX
        const bool summary = MODE == MODE_CTX && a.sts_raw != nullptr;
        float* part0 = reinterpret_cast<float*>(sm + LY::PART_OFF);
        int32_t* grp = reinterpret_cast<int32_t*>(sm + LY::GRP_OFF);  // [0]=count, then group row starts
        int32_t* gsrc_s = grp + TM + 2;                                 // source segment of each group
        uint32_t* bmask = reinterpret_cast<uint32_t*>(sm + LY::MSK_OFF);
        int pbuf = 0;
        int src = -1;  // this row's source segment (-1: query row)
        if (MODE == MODE_CTX) {
            if (rvalid) {
                m_row = a.m_fin[int64_t(row) * a.H + head];
                il_row = a.inv_l[int64_t(row) * a.H + head];
                src = a.row_seg[t];
            }
            if (summary) {
                // row groups of equal source segment (rows of a segment are contiguous)
                const int prev = (r > 0 && rvalid) ? a.row_seg[a.rows[row - 1]] : INT32_MIN;
                const bool start = rvalid && (r == 0 || prev != src);
                const uint32_t bal = __ballot_sync(0xffffffffu, start);
                if (lane == 0) bmask[q] = bal;
                named_sync_softmax();
                if (tid == 0) {
                    int ng = 0;
                    for (int w = 0; w < 4; ++w)
                        for (uint32_t m = bmask[w]; m; m &= m - 1) grp[1 + ng++] = w * 32 + __ffs(m) - 1;
                    grp[1 + ng] = nrows;
                    grp[0] = ng;
                }
                named_sync_softmax();
                for (int g = tid; g < grp[0]; g += 128) gsrc_s[g] = a.row_seg[a.rows[i0 + grp[1 + g]]];
                named_sync_softmax();
            }
        }
        for (int it = 0; it < niter; ++it) {
            const int b = it & 1;
            const int k0 = kbase + it * TK;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            fence_after();
            uint32_t sv[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tm_s0 + lane_base + uint32_t(b * TK + c * 32), sv[c]);
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
            // keys of this chunk visible to this row: [kv0, kv1)
            // (max: a row that ends before this key split sees an empty range,
            // not a wrapped unsigned one)
            const int kv0 = klo - k0, kv1 = max(kv0, min(hi, t + 1) - k0);
            // fully visible chunk for every row of the warp: no per-key masks
            const bool full_chunk = __all_sync(0xffffffffu, kv0 <= 0 && kv1 >= TK);
            if (MODE == MODE_STATS) {
                float cm = -FLT_MAX;
                if (full_chunk) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float v = __uint_as_float(sv[c][j]) * scale;
                            sv[c][j] = __float_as_uint(v);
                            cm = fmaxf(cm, v);
                        }
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const bool ok = unsigned(c * 32 + j - kv0) < unsigned(kv1 - kv0);
                            const float v = ok ? __uint_as_float(sv[c][j]) * scale : -FLT_MAX;
                            sv[c][j] = __float_as_uint(v);
                            cm = fmaxf(cm, v);
                        }
                }
                if (cm > -FLT_MAX) {
                    const float mn = fmaxf(m_run, cm);
                    float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            ps0 += ex2(__uint_as_float(sv[c][j]) - mn);
                            ps1 += ex2(__uint_as_float(sv[c][j + 1]) - mn);
                        }
                    l_run = (m_run > -FLT_MAX ? l_run * ex2(m_run - mn) : 0.f) + (ps0 + ps1);
                    m_run = mn;
                }
            } else {
                // normalised probabilities (fp32, kept in sv for the summary)
                if (full_chunk) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            sv[c][j] = __float_as_uint(ex2(fmaf(__uint_as_float(sv[c][j]), scale, -m_row)) * il_row);
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const bool ok = unsigned(c * 32 + j - kv0) < unsigned(kv1 - kv0);
                            const float p = ex2(fmaf(__uint_as_float(sv[c][j]), scale, -m_row)) * il_row;
                            sv[c][j] = __float_as_uint(ok ? p : 0.f);
                        }
                }
                mbar_wait(p_empty, (it & 1) ^ 1);
                uint8_t* pt = sm + LY::P_OFF;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const uint32_t* v = &sv[c][g * 8];
                        const uint4 w4 = make_uint4(pack_bf16(__uint_as_float(v[0]), __uint_as_float(v[1])),
                                                    pack_bf16(__uint_as_float(v[2]), __uint_as_float(v[3])),
                                                    pack_bf16(__uint_as_float(v[4]), __uint_as_float(v[5])),
                                                    pack_bf16(__uint_as_float(v[6]), __uint_as_float(v[7])));
                        *reinterpret_cast<uint4*>(pt + p_chunk_off(r, c * 4 + g)) = w4;
                    }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full);

                if (summary) {
                    // per-chunk segment table (prefill constant): flush j of the
                    // boundary bits closes destination segment d0 + j
                    const int4 hdr = a.chunk_tab[2 * (k0 / TK)];
                    const int4 msk = a.chunk_tab[2 * (k0 / TK) + 1];
                    const int d0 = hdr.x, nseg = hdr.y;
                    const uint32_t mw[4] = {uint32_t(msk.x), uint32_t(msk.y), uint32_t(msk.z), uint32_t(msk.w)};
                    for (int pass = 0; pass * PART_SEGS < nseg; ++pass) {
                        const int jlo = pass * PART_SEGS, jhi = min(nseg, jlo + PART_SEGS);
                        float* part = part0 + pbuf * (TM * PART_STRIDE);
                        float* prow = part + r * PART_STRIDE;
                        // own segment (dropped) as a local flush index: stored to the trash slot
                        const int own = src - d0 - jlo;
                        float run = 0.f;
                        int j = -jlo;  // local index of the next flush
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint32_t mword = mw[c];
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) {
                                run += __uint_as_float(sv[c][jj]);
                                const uint32_t bit = (mword >> jj) & 1u;
                                // branch-free: predicated store, index clamped to the trash slot
                                const unsigned idx = (unsigned(j) < unsigned(PART_SEGS) && j != own) ? unsigned(j)
                                                                                                       : unsigned(PART_SEGS);
                                if (bit) prow[idx] = run;
                                run = bit ? 0.f : run;
                                j += int(bit);
                            }
                        }
                        // segments closed in this pass that were the row's own: write 0
                        if (unsigned(own) < unsigned(PART_SEGS) && own < jhi - jlo) prow[own] = 0.f;
                        // one barrier per pass: the other buffer's reduction (previous
                        // pass) finished before anyone got here
                        named_sync_softmax();
                        const int ng = grp[0], nj = jhi - jlo;
                        for (int e = tid; e < ng * nj; e += 128) {
                            const int g = e / nj, jj = e % nj;
                            const int rb = grp[1 + g], re = grp[2 + g];
                            float acc = 0.f;
                            for (int rr = rb; rr < re; ++rr) acc += part[rr * PART_STRIDE + jj];
                            if (acc != 0.f) {
                                const int gs = gsrc_s[g];
                                const int dst = d0 + jlo + jj;
                                double* tgt = gs < 0 ? a.qts_raw + dst : a.sts_raw + int64_t(gs) * a.S + dst;
                                atomicAdd(tgt, double(acc) * double(a.inv_heads));
                            }
                        }
                        pbuf ^= 1;
                    }
                }
            }
        }
        // ---------------------------------------------------------- outputs
        if (MODE == MODE_STATS && rvalid) {
            const int64_t o = (int64_t(sp) * a.n + row) * a.H + head;
            a.m_part[o] = m_run;
            a.l_part[o] = l_run;
        } else if (MODE == MODE_CTX) {
            if (niter > 0) {
                mbar_wait(o_full, 0);
                fence_after();
            }
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t ov[32];
                if (niter > 0) {
                    tmem_ld32(tm_o + lane_base + uint32_t(c * 32), ov);
                } else {
                    for (int e = 0; e < 32; ++e) ov[e] = 0u;
                }
                if (!rvalid) continue;
                if (a.nsplit == 1) {
                    uint4* dst = reinterpret_cast<uint4*>(a.ctx + int64_t(row) * a.d + head * DH + c * 32);
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        dst[g] = make_uint4(pack_bf16(__uint_as_float(ov[g * 8 + 0]), __uint_as_float(ov[g * 8 + 1])),
                                            pack_bf16(__uint_as_float(ov[g * 8 + 2]), __uint_as_float(ov[g * 8 + 3])),
                                            pack_bf16(__uint_as_float(ov[g * 8 + 4]), __uint_as_float(ov[g * 8 + 5])),
                                            pack_bf16(__uint_as_float(ov[g * 8 + 6]), __uint_as_float(ov[g * 8 + 7])));
                } else {
                    float4* dst =
                        reinterpret_cast<float4*>(a.o_part + (int64_t(sp) * a.n + row) * a.d + head * DH + c * 32);
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        dst[g] = make_float4(__uint_as_float(ov[4 * g]), __uint_as_float(ov[4 * g + 1]),
                                             __uint_as_float(ov[4 * g + 2]), __uint_as_float(ov[4 * g + 3]));
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        tmem_dealloc(tmem, LY::TMEM_COLS);
    }
}

// ===================================================================== v2 ==
// 608 threads: warp 0 TMA (Q, K), warp 1 MMA issuer, warp 2 TMEM allocator
// and TMA (V, Z), warps 3..18 softmax in two TEAMS of eight warps.  Team t
// owns the chunks it = t (mod 2) -- exactly the chunks whose scores land in
// TMEM buffer S[t] -- so while one team waits for its scores to stream out of
// TMEM (tcgen05.ld, ~64 B/clk/SM) the other team computes on the chunk it has
// already read: TMEM reads, MUFU and the tensor pipe overlap across chunks.
// Within a team, warp w serves TMEM lanes 32(w%4).. (rows) and key half
// h = ((w-3)/4) & 1 of the chunk (64 keys).
//
// CTX: p = exp2(s*scale - m - log2 l) (fp32) is split into hi = bf16(p) and
// lo = bf16(p - hi), written back into the TMEM columns of S[t] (half h: hi
// at 64h..64h+31, lo at 64h+32..64h+63) and read by tcgen05.mma as the A
// operand (TS form):
//   O    += hi . V                (P.V; V is the MN-major B operand read
//                                  straight from the merged KV)
//   BINS  = hi . Z + lo . Z       (segment summary with 16 bits of p: the
//                                  precision the reference's near-tied
//                                  selections need)
// Z is the one-hot key -> destination-segment indicator of the chunk
// (prefill constant, zt_build_kernel); query keys have no column (their mass
// is dropped, prefill.hpp:283).  The owning team flushes a chunk's bins two of
// its chunks later (TMEM buffer 2*(j&1) + ((j>>1)&1)): own segment zeroed
// (prefill.hpp:284), rows reduced per source segment through shared memory,
// one fp64 atomic per (source, destination) pair.
constexpr int NTEAM = 2;
constexpr int KH = TK / 2;            // keys per warp (key half)
constexpr int NTHR2 = 96 + NTEAM * 256;
constexpr uint32_t BINS_COL = 384;    // TMEM: S 0..255, O 256..383, bins 384..

// Two TMA rings: K (STATS 4 stages, CTX 3 or 2) freed after Q.K^T, and (CTX)
// V + Z (2 stages) freed after P.V.
template <int MODE, int NB>
struct Layout2 {
    static constexpr int ST = MODE == MODE_STATS ? 4 : (NB <= 16 ? 3 : 2);  // K stages
    static constexpr int NH = NB / 2;                 // bins columns per key half
    static constexpr uint32_t ZB = NB * 128 * 2;      // Z^T tile [NB x 128] bf16 (2 boxes of NB x 64)
    static constexpr uint32_t STAGE = TILE_BYTES;     // K stage
    static constexpr uint32_t VSTAGE = TILE_BYTES + (MODE == MODE_CTX ? ZB : 0);
    static constexpr uint32_t Q_OFF = 0;
    static constexpr uint32_t STAGE_OFF = TILE_BYTES;
    static constexpr uint32_t VSTAGE_OFF = STAGE_OFF + ST * STAGE;
    static constexpr uint32_t PART_OFF = VSTAGE_OFF + (MODE != MODE_STATS ? 2 * VSTAGE : 0);
    // STATS: (m, l) of the 3 other (team, half) partials; CTX: bins partials [team][half][128][NH];
    // FLASH: chunk maxima [2][team][half][128] then the epilogue's l [team][half][128] and m [team][128]
    static constexpr uint32_t PART_BYTES =
        MODE == MODE_STATS ? 3 * TM * 2 * 4 : (MODE == MODE_CTX ? NTEAM * 2 * TM * NH * 4 : 14 * TM * 4);
    static constexpr uint32_t GRP_OFF = PART_OFF + PART_BYTES;  // CTX: groups [130] + sources [130]
    static constexpr uint32_t MSK_OFF = GRP_OFF + (2 * TM + 4) * 4;
    static constexpr uint32_t BAR_OFF = (MSK_OFF + 16 + 7) & ~7u;
    static constexpr size_t SMEM = size_t(BAR_OFF) + 256 + 1024;
    static constexpr uint32_t TMEM_COLS = MODE != MODE_STATS ? 512 : 256;
};
static_assert(Layout2<MODE_FLASH, 16>::SMEM <= 232448, "FLASH v2 smem");
static_assert(Layout2<MODE_CTX, 32>::SMEM <= 232448, "CTX v2 smem (NB 32)");
static_assert(Layout2<MODE_CTX, 16>::SMEM <= 232448, "CTX v2 smem (NB 16)");
static_assert(Layout2<MODE_STATS, 16>::SMEM <= 232448, "STATS v2 smem");
static_assert(BINS_COL + 4 * 32 <= 512, "bins buffers");

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// MN-major 128B-swizzled B operand (V as [keys x dh], dh contiguous): 64-wide
// dh chunks 16 KB apart (LBO), 8-key row groups 1024 B apart (SBO); a K=16
// step starts 2 row groups (2048 B) further.
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t(BOX_BYTES >> 4) << 16;  // leading byte offset: next 64 dh columns
    d |= uint64_t(1024 >> 4) << 32;       // stride byte offset: next 8 keys
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
constexpr uint32_t IDESC_VMN = instr_desc(128, 128) | (1u << 16);  // B MN-major

__device__ __forceinline__ int bins_buf(int j) { return 2 * (j & 1) + ((j >> 1) & 1); }

template <int MODE, int NB>
__global__ void __launch_bounds__(NTHR2, 1)
attn_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmZ, TcArgs a) {
    using LY = Layout2<MODE, NB>;
    constexpr uint32_t IDESC_B = instr_desc(128, NB);
    constexpr int NH = LY::NH;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared space
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + LY::BAR_OFF);
    uint64_t* full = bar;            // [ST] K ring
    uint64_t* empty = bar + 4;       // [ST]
    uint64_t* s_full = bar + 8;      // [2] per S buffer (= per team)
    uint64_t* s_empty = bar + 10;    // [2] (STATS)
    uint64_t* p_full = bar + 12;     // [2] (CTX)
    uint64_t* q_full = bar + 14;
    uint64_t* o_full = bar + 15;
    uint64_t* vfull = bar + 16;      // [2] V ring (CTX)
    uint64_t* vempty = bar + 18;     // [2]
    uint64_t* bins_full = bar + 20;  // [4]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 24);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.x * TM;
    const int nrows = min(TM, a.n - i0);
    const int head = blockIdx.y, sp = blockIdx.z;
    const int tmax = a.rows[i0 + nrows - 1];
    const int tklo = a.key_lo ? a.key_lo[a.rows[i0]] : 0;
    const int lo = max(a.split_lo[sp], tklo);
    const int hi = min(a.split_hi[sp], tmax + 1);
    const int kbase = lo & ~7;
    const int niter = hi > lo ? int(ceil_div(hi - kbase, TK)) : 0;
    const bool bins = MODE == MODE_CTX && a.sts_raw != nullptr;

    if (warp == 0 && lane == 0) {
        prefetch_map(&tmQ);
        prefetch_map(&tmK);
        if (MODE != MODE_STATS) prefetch_map(&tmV);
        if (bins) prefetch_map(&tmZ);
        for (int s = 0; s < LY::ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_empty[b], 8);
            mbar_init(&p_full[b], 8);
            mbar_init(&vfull[b], 1);
            mbar_init(&vempty[b], 1);
        }
        for (int b = 0; b < 4; ++b) mbar_init(&bins_full[b], 1);
        mbar_init(q_full, 1);
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, LY::TMEM_COLS);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_s0 = tmem, tm_o = tmem + 256, tm_b = tmem + BINS_COL;

    if (warp == 0) {
        // ------------------------------------------------------- TMA: Q, K
        if (lane == 0 && niter > 0) {
            mbar_expect_tx(q_full, TILE_BYTES);
            tma_load_2d(sm + LY::Q_OFF, &tmQ, q_full, head * DH, i0);
            tma_load_2d(sm + LY::Q_OFF + BOX_BYTES, &tmQ, q_full, head * DH + 64, i0);
            for (int it = 0; it < niter; ++it) {
                const int s = it % LY::ST;
                mbar_wait(&empty[s], ((it / LY::ST) & 1) ^ 1);
                uint8_t* st = sm + LY::STAGE_OFF + s * LY::STAGE;
                const int k0 = kbase + it * TK;
                mbar_expect_tx(&full[s], TILE_BYTES);
                tma_load_2d(st, &tmK, &full[s], head * DH, k0);
                tma_load_2d(st + BOX_BYTES, &tmK, &full[s], head * DH + 64, k0);
            }
        }
    } else if (warp == 2) {
        // ------------------------------------ TMA: V, Z (CTX; after the alloc)
        if (MODE != MODE_STATS && lane == 0 && niter > 0) {
            for (int it = 0; it < niter; ++it) {
                const int s = it & 1;
                mbar_wait(&vempty[s], ((it >> 1) & 1) ^ 1);
                uint8_t* st = sm + LY::VSTAGE_OFF + s * LY::VSTAGE;
                const int k0 = kbase + it * TK;
                mbar_expect_tx(&vfull[s], bins ? LY::VSTAGE : TILE_BYTES);
                // V rows straight from the merged KV ([keys x dh] tile, dh
                // contiguous): the MN-major B operand of P.V, no transpose
                tma_load_2d(st, &tmV, &vfull[s], head * DH, k0);
                tma_load_2d(st + BOX_BYTES, &tmV, &vfull[s], head * DH + 64, k0);
                if (bins) {
                    const int zrow = (k0 / TK) * NB;
                    tma_load_2d(st + TILE_BYTES, &tmZ, &vfull[s], 0, zrow);
                    tma_load_2d(st + TILE_BYTES + LY::ZB / 2, &tmZ, &vfull[s], 64, zrow);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA
        // The whole warp walks the schedule (waits, descriptors: warp-uniform
        // values in uniform registers) and one elected lane issues each group
        // of tcgen05.mma / commits -- no per-instruction divergence loop.
        if (niter > 0) {
            mbar_wait(q_full, 0);
            const uint32_t qt = smem_u32(sm + LY::Q_OFF);
            const uint64_t qd = smem_desc(qt);
            // k-step ks of 16 elements across the two 64-wide boxes of a tile:
            // + ((ks >> 2) * BOX_BYTES + (ks & 3) * 32) in the 16-byte address field
            auto koff = [](int ks) { return uint64_t(((ks >> 2) * BOX_BYTES + (ks & 3) * 32) >> 4); };
            // CTX: O += hi_j . V_j ; BINS[bins_buf(j)] = hi_j . Z_j + lo_j . Z_j,
            // P(j) in S[j&1]: half h's hi at columns 64h..64h+31, lo at +32
            auto pv = [&](int j) {
                mbar_wait(&p_full[j & 1], (j >> 1) & 1);
                mbar_wait(&vfull[j & 1], (j >> 1) & 1);
                fence_after();
                const uint32_t pb = tm_s0 + uint32_t((j & 1) * TK);
                const uint32_t vt = smem_u32(sm + LY::VSTAGE_OFF + (j & 1) * LY::VSTAGE);
                const uint64_t vd = desc_mn(vt);
                // FLASH: one O accumulator per team (columns 256 + 128 team),
                // each started by the team's first chunk
                const uint32_t to = MODE == MODE_FLASH ? tm_o + uint32_t((j & 1) * 128) : tm_o;
                const int jacc = MODE == MODE_FLASH ? (j >> 1) : j;
                if (elect_one()) {
                    if (a.dbg != 2)
#pragma unroll
                        for (int ks = 0; ks < TK / 16; ++ks)
                            umma_ts(to, pb + uint32_t(64 * (ks >> 2) + 8 * (ks & 3)), vd + uint64_t(ks) * 128u,
                                    IDESC_VMN, (jacc | ks) ? 1u : 0u);
                    if (bins) {
                        const uint32_t zt = vt + TILE_BYTES;
                        const uint64_t zd = smem_desc(zt);
                        const uint32_t tb = tm_b + uint32_t(bins_buf(j) * NB);
                        const int nplo = a.dbg == 1 ? 1 : 2;
#pragma unroll
                        for (int plo = 0; plo < 2; ++plo)
                            if (plo < nplo)
#pragma unroll
                                for (int ks = 0; ks < TK / 16; ++ks)
                                    umma_ts(tb, pb + uint32_t(64 * (ks >> 2) + 32 * plo + 8 * (ks & 3)),
                                            zd + uint64_t(((ks >> 2) * (LY::ZB / 2) + (ks & 3) * 32) >> 4), IDESC_B,
                                            (plo | ks) ? 1u : 0u);
                        umma_commit(&bins_full[bins_buf(j)]);
                    }
                    umma_commit(&vempty[j & 1]);
                }
                __syncwarp();
            };
            for (int it = 0; it < niter; ++it) {
                const int s = it % LY::ST, b = it & 1;
                mbar_wait(&full[s], (it / LY::ST) & 1);
                // CTX: S[b] held P(it-2), consumed by MMAs issued earlier (issue order)
                if (MODE == MODE_STATS) mbar_wait(&s_empty[b], ((it >> 1) & 1) ^ 1);
                fence_after();
                const uint64_t kd = smem_desc(smem_u32(sm + LY::STAGE_OFF + s * LY::STAGE));
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < DH / 16; ++ks)
                        umma(tm_s0 + uint32_t(b * TK), qd + koff(ks), kd + koff(ks), IDESC, ks ? 1u : 0u);
                    umma_commit(&s_full[b]);
                    umma_commit(&empty[s]);
                }
                __syncwarp();
                if (MODE != MODE_STATS && it > 0) pv(it - 1);
            }
            if (MODE != MODE_STATS) {
                pv(niter - 1);
                if (elect_one()) umma_commit(o_full);
                __syncwarp();
            }
        }
    } else if (warp >= 3) {
        // ------------------------------------------ softmax / summary / epilogue
        const int q = warp & 3;
        const int team = (warp - 3) >> 3;     // owns chunks it = team (mod 2) and S[team]
        const int half = ((warp - 3) >> 2) & 1;
        const int tid = threadIdx.x - 96;     // 0..511
        const int htid = tid & 127;           // within (team, half)
        const int r = q * 32 + lane;          // tile row == TMEM lane
        const bool rvalid = r < nrows;
        const int row = i0 + r;
        const int t = rvalid ? a.rows[row] : -1;
        const int klo = max(lo, rvalid && a.key_lo ? a.key_lo[t] : 0);
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const float scale = a.scale_log2;
        const int c0 = half * KH;             // first key column of this warp in a chunk
        float m_run = -FLT_MAX, l_run = 0.f;  // STATS
        float lsum = 0.f;                     // CTX with norm_end / FLASH: this warp's part of l
        float fm = -INFINITY;                 // FLASH: running max of the team's rows (exp2 domain)
        bool o_started = false;               // FLASH: this team's O has been written by a P.V
        float* part = reinterpret_cast<float*>(sm + LY::PART_OFF);
        int32_t* grp = reinterpret_cast<int32_t*>(sm + LY::GRP_OFF);
        int32_t* gsrc_s = grp + TM + 2;
        uint32_t* bmask = reinterpret_cast<uint32_t*>(sm + LY::MSK_OFF);
        int src = -1;
        float m_eff = 0.f;  // CTX: m + log2(l): p = exp2(s*scale - m_eff)
        if (MODE == MODE_CTX) {
            if (rvalid) {
                const float m_row = a.m_fin[int64_t(row) * a.H + head];
                const float il_row = a.inv_l[int64_t(row) * a.H + head];
                src = a.row_seg[t];
                m_eff = a.norm_end ? m_row : (il_row > 0.f ? m_row - __log2f(il_row) : INFINITY);
            }
            if (bins) {
                const int prev = (r > 0 && rvalid) ? a.row_seg[a.rows[row - 1]] : INT32_MIN;
                const bool start = rvalid && (r == 0 || prev != src);
                const uint32_t bal = __ballot_sync(0xffffffffu, start);
                if (tid < 128 && lane == 0) bmask[q] = bal;  // (warps 3..6 cover q = 3, 0, 1, 2)
                named_sync(1, NTEAM * 256);
                if (tid == 0) {
                    int ng = 0;
                    for (int w = 0; w < 4; ++w)
                        for (uint32_t m = bmask[w]; m; m &= m - 1) grp[1 + ng++] = w * 32 + __ffs(m) - 1;
                    grp[1 + ng] = nrows;
                    grp[0] = ng;
                }
                named_sync(1, NTEAM * 256);
                for (int g = tid; g < grp[0]; g += NTEAM * 256) gsrc_s[g] = a.row_seg[a.rows[i0 + grp[1 + g]]];
                named_sync(1, NTEAM * 256);
            }
        }
        // bins of chunk j (this team's, complete in TMEM buffer bins_buf(j)):
        // own segment zeroed, rows reduced per source segment, one fp64 atomic
        // per pair; the (team, half) group reduces bins columns [half*NH, +NH)
        const int ngrp = bins ? grp[0] : 0;
        const int bar_id = 2 + team * 2 + half;
        float* gp = part + (team * 2 + half) * (TM * NH);
        auto flush_bins = [&](int j) {
            mbar_wait(&bins_full[bins_buf(j)], (j >> 2) & 1);
            fence_after();
            const int k0 = kbase + j * TK;
            const int4 hdr = __ldg(&a.chunk_tab[2 * (k0 / TK)]);
            const int d0 = hdr.x, nseg = hdr.y;
            const int jb = half * NH;           // first bins column of this group
            const int nj = min(NH, nseg - jb);  // (uniform across the group)
            if (nj > 0) {
                uint32_t bv[NH];
                if constexpr (NH == 16) tmem_ld16(tm_b + lane_base + uint32_t(bins_buf(j) * NB + jb), bv);
                else tmem_ld8(tm_b + lane_base + uint32_t(bins_buf(j) * NB + jb), bv);
                const int own = src - d0 - jb;
#pragma unroll
                for (int c = 0; c < NH; ++c) gp[r * NH + (c ^ (r & (NH - 1)))] = (c == own) ? 0.f : __uint_as_float(bv[c]);
            }
            fence_before();
            named_sync(bar_id, 128);
            if (nj > 0) {
                constexpr int LNH = NH == 16 ? 4 : 3;
                for (int e = htid; e < (ngrp << LNH); e += 128) {
                    const int g = e >> LNH, c = e & (NH - 1);
                    if (c >= nj) continue;
                    const int rb = grp[1 + g], re = grp[2 + g];
                    float acc = 0.f;
                    for (int rr = rb; rr < re; ++rr) acc += gp[rr * NH + (c ^ (rr & (NH - 1)))];
                    if (acc != 0.f) {
                        const int gs = gsrc_s[g];
                        const int dst = d0 + jb + c;
                        double* tgt = gs < 0 ? a.qts_raw + dst : a.sts_raw + int64_t(gs) * a.S + dst;
                        atomicAdd(tgt, double(acc) * double(a.inv_heads));
                    }
                }
            }
            named_sync(bar_id, 128);  // the partials are rewritten by the next flush
        };
        const int b = team;
        // a warp whose 32 rows are all padding (few-row tiles: the deep layers'
        // query) skips the scores entirely -- its P rows only feed accumulator
        // rows that are never stored -- and just keeps the barriers moving
        const bool wvalid = __any_sync(0xffffffffu, rvalid);
        for (int it = team; it < niter; it += NTEAM) {
            const int k0 = kbase + it * TK;
            mbar_wait(&s_full[b], (it >> 1) & 1);
            fence_after();
            if (!wvalid) {
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(MODE == MODE_STATS ? &s_empty[b] : &p_full[b]);
                if (MODE == MODE_CTX && bins && it >= 2) flush_bins(it - 2);
                continue;
            }
            uint32_t sv[2][32];
            tmem_ld32x2(tm_s0 + lane_base + uint32_t(b * TK + c0), sv[0], sv[1]);
            if (MODE == MODE_STATS) {
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[b]);
            }
            // visible keys of this half; a row that ends before this key split
            // sees an empty range (max), never a wrapped unsigned one
            const int kv0 = klo - k0 - c0, kv1 = max(kv0, min(hi, t + 1) - k0 - c0);
            const bool full_half = __all_sync(0xffffffffu, kv0 <= 0 && kv1 >= KH);
            if (MODE == MODE_STATS) {
                // max on the raw scores (scale > 0), then exp2(s*scale - m):
                // FMNMX + FFMA + MUFU + FADD per score.  Masked chunks take a
                // separate instantiation so full chunks carry no predicated work.
                auto stats = [&](auto masked) {
                    float cmr = -INFINITY;
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            if constexpr (decltype(masked)::value)
                                if (unsigned(c * 32 + jj - kv0) >= unsigned(kv1 - kv0))
                                    sv[c][jj] = __float_as_uint(-INFINITY);
                            cmr = fmaxf(cmr, __uint_as_float(sv[c][jj]));
                        }
                    if (cmr > -INFINITY && a.norm_end) {
                        m_run = fmaxf(m_run, cmr * scale);  // max only: the CTX pass sums l
                    } else if (cmr > -INFINITY) {
                        const float mn = fmaxf(m_run, cmr * scale);
                        float ps0 = 0.f, ps1 = 0.f, ps2 = 0.f, ps3 = 0.f;
#pragma unroll
                        for (int c = 0; c < 2; ++c)
#pragma unroll
                            for (int jj = 0; jj < 32; jj += 4) {
                                ps0 += ex2(fmaf(__uint_as_float(sv[c][jj]), scale, -mn));
                                ps1 += ex2(fmaf(__uint_as_float(sv[c][jj + 1]), scale, -mn));
                                ps2 += ex2(fmaf(__uint_as_float(sv[c][jj + 2]), scale, -mn));
                                ps3 += ex2(fmaf(__uint_as_float(sv[c][jj + 3]), scale, -mn));
                            }
                        l_run = (m_run > -FLT_MAX ? l_run * ex2(m_run - mn) : 0.f) + ((ps0 + ps1) + (ps2 + ps3));
                        m_run = mn;
                    }
                };
                if (full_half) stats(std::false_type{});
                else stats(std::true_type{});
            } else if (MODE == MODE_FLASH) {
                // single pass (no summary): running max per row shared by the
                // two key halves of the team, lazy rescale of the team's O
                // (only when the max grows by more than 2^8): P <= 256.  When
                // S[b] of chunk `it` is full, every MMA issued before Q.K^T(it)
                // is complete -- P.V(it-2), the last one into O[b] -- and
                // P.V(it) waits for p_full: O[b] is quiescent here.
                // (two interleaved max chains: half the dependent latency)
                float cm = -INFINITY, cm2 = -INFINITY;
                if (full_half) {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int jj = 0; jj < 32; jj += 2) {
                            cm = fmaxf(cm, __uint_as_float(sv[c][jj]));
                            cm2 = fmaxf(cm2, __uint_as_float(sv[c][jj + 1]));
                        }
                } else {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int jj = 0; jj < 32; jj += 2) {
                            if (unsigned(c * 32 + jj - kv0) < unsigned(kv1 - kv0)) cm = fmaxf(cm, __uint_as_float(sv[c][jj]));
                            if (unsigned(c * 32 + jj + 1 - kv0) < unsigned(kv1 - kv0))
                                cm2 = fmaxf(cm2, __uint_as_float(sv[c][jj + 1]));
                        }
                }
                cm = fmaxf(cm, cm2);
                float* xm = part + ((((it >> 1) & 1) * NTEAM + team) * 2) * TM;  // [parity][team][half][TM]
                xm[half * TM + r] = cm;
                named_sync(2 + team * 4 + q, 64);  // the two key halves of rows 32q.. in this team
                cm = fmaxf(cm, xm[(half ^ 1) * TM + r]);
                const float m_new = fmaxf(fm, cm);
                const bool resc = m_new > fm + 8.f;  // (fm = -inf, m_new finite: the first keys)
                const float al = resc ? ex2(fm - m_new) : 1.f;
                if (resc) {
                    fm = m_new;
                    lsum *= al;
                }
                m_eff = fm == -INFINITY ? 0.f : fm;
                const uint32_t tp = tm_s0 + lane_base + uint32_t(b * TK + half * 64);
                // packed fp32x2 arithmetic (FADD2): half the subtract / sum instructions
                float2 ls2 = make_float2(0.f, 0.f);
                const float2 negm = make_float2(-m_eff, -m_eff);
                auto make_p = [&](auto masked, int c) {
                    uint32_t hv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int kk = 32 * c + 2 * i;
                        const float2 x = __fadd2_rn(make_float2(__uint_as_float(sv[c][2 * i]),
                                                                __uint_as_float(sv[c][2 * i + 1])), negm);
                        float p0 = ex2(x.x);
                        float p1 = ex2(x.y);
                        if constexpr (decltype(masked)::value) {
                            p0 = unsigned(kk - kv0) < unsigned(kv1 - kv0) ? p0 : 0.f;
                            p1 = unsigned(kk + 1 - kv0) < unsigned(kv1 - kv0) ? p1 : 0.f;
                        }
                        hv[i] = pack_bf16(p0, p1);
                        ls2 = __fadd2_rn(ls2, make_float2(p0, p1));
                    }
                    tmem_st16(tp + uint32_t(16 * c), hv);
                };
                if (full_half) {
                    make_p(std::false_type{}, 0);
                    make_p(std::false_type{}, 1);
                } else {
                    make_p(std::true_type{}, 0);
                    make_p(std::true_type{}, 1);
                }
                lsum += ls2.x + ls2.y;
                if (o_started && __any_sync(0xffffffffu, resc)) {
                    const uint32_t to = tm_o + lane_base + uint32_t(b * 128 + half * 64);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t ov[32];
                        tmem_ld32(to + uint32_t(32 * c), ov);
#pragma unroll
                        for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * al);
                        tmem_st32(to + uint32_t(32 * c), ov);
                    }
                }
                o_started = true;
                tmem_wait_st();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[b]);
            } else {
                // p, then P = hi + lo back into S[b] (this half's 64 columns),
                // 32 keys at a time so the split stays in registers
                const uint32_t tp = tm_s0 + lane_base + uint32_t(b * TK + half * 64);
                // (without a summary only hi feeds P.V: lo is neither formed nor stored)
                auto make_p = [&](auto masked, auto with_lo, int c) {
                    uint32_t hv[16], lv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int kk = 32 * c + 2 * i;
                        float p0 = ex2(fmaf(__uint_as_float(sv[c][2 * i]), scale, -m_eff));
                        float p1 = ex2(fmaf(__uint_as_float(sv[c][2 * i + 1]), scale, -m_eff));
                        if constexpr (decltype(masked)::value) {
                            p0 = unsigned(kk - kv0) < unsigned(kv1 - kv0) ? p0 : 0.f;
                            p1 = unsigned(kk + 1 - kv0) < unsigned(kv1 - kv0) ? p1 : 0.f;
                        }
                        const uint32_t h = pack_bf16(p0, p1);
                        hv[i] = h;
                        if constexpr (decltype(with_lo)::value)
                            lv[i] = pack_bf16(p0 - __uint_as_float(h << 16), p1 - __uint_as_float(h & 0xffff0000u));
                        else
                            lsum += p0 + p1;
                    }
                    tmem_st16(tp + uint32_t(16 * c), hv);
                    if constexpr (decltype(with_lo)::value) tmem_st16(tp + uint32_t(32 + 16 * c), lv);
                };
                if (bins) {
                    if (full_half) {
                        make_p(std::false_type{}, std::true_type{}, 0);
                        make_p(std::false_type{}, std::true_type{}, 1);
                    } else {
                        make_p(std::true_type{}, std::true_type{}, 0);
                        make_p(std::true_type{}, std::true_type{}, 1);
                    }
                } else {
                    if (full_half) {
                        make_p(std::false_type{}, std::false_type{}, 0);
                        make_p(std::false_type{}, std::false_type{}, 1);
                    } else {
                        make_p(std::true_type{}, std::false_type{}, 0);
                        make_p(std::true_type{}, std::false_type{}, 1);
                    }
                }
                tmem_wait_st();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[b]);
                if (bins && it >= 2) flush_bins(it - 2);
            }
        }
        // ---------------------------------------------------------- outputs
        if (MODE == MODE_STATS) {
            // combine the 4 (team, half) partials in a fixed order
            float* ml = part;
            const int gidx = team * 2 + half;
            if (gidx > 0) {
                ml[((gidx - 1) * TM + r) * 2] = m_run;
                ml[((gidx - 1) * TM + r) * 2 + 1] = l_run;
            }
            named_sync(1, NTEAM * 256);
            if (gidx == 0 && rvalid) {
                float m = m_run;
                for (int g = 1; g < 4; ++g) m = fmaxf(m, ml[((g - 1) * TM + r) * 2]);
                float l = m_run > -FLT_MAX ? l_run * ex2(m_run - m) : 0.f;
                for (int g = 1; g < 4; ++g) {
                    const float mg = ml[((g - 1) * TM + r) * 2], lg = ml[((g - 1) * TM + r) * 2 + 1];
                    if (mg > -FLT_MAX) l += lg * ex2(mg - m);
                }
                const int64_t o = (int64_t(sp) * a.n + row) * a.H + head;
                a.m_part[o] = m;
                a.l_part[o] = l;
            }
        } else if (MODE == MODE_FLASH) {
            if (niter > 0) {
                mbar_wait(o_full, 0);
                fence_after();
            }
            // merge the two teams: O = O0 2^(m0 - M) + O1 2^(m1 - M), l alike
            float* lp = part + 8 * TM;   // [team][half][TM]
            float* mp = part + 12 * TM;  // [team][TM]
            lp[(team * 2 + half) * TM + r] = lsum;
            if (half == 0) mp[team * TM + r] = fm;
            named_sync(1, NTEAM * 256);
            const float m0 = mp[r], m1 = mp[TM + r];
            const float M = fmaxf(m0, m1);
            const float f0 = m0 == -INFINITY ? 0.f : ex2(m0 - M), f1 = m1 == -INFINITY ? 0.f : ex2(m1 - M);
            const float L = (lp[r] + lp[TM + r]) * f0 + (lp[2 * TM + r] + lp[3 * TM + r]) * f1;
            const int oc = 32 * (team * 2 + half);
            uint32_t ov[32];
            if (niter > 0) {
                uint32_t o1[32];
                tmem_ld32(tm_o + lane_base + uint32_t(oc), ov);
                tmem_ld32(tm_o + lane_base + uint32_t(128 + oc), o1);
                // (a team without chunks, or whose rows saw no key, has f = 0
                // and an O that was never written)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    ov[e] = __float_as_uint((f0 != 0.f ? __uint_as_float(ov[e]) * f0 : 0.f) +
                                            (f1 != 0.f ? __uint_as_float(o1[e]) * f1 : 0.f));
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = 0u;
            }
            if (rvalid) {
                const int col = head * DH + oc;
                if (a.nsplit == 1) {
                    const float il = L > 0.f ? 1.f / L : 0.f;
                    uint4* dst = reinterpret_cast<uint4*>(a.ctx + int64_t(row) * a.d + col);
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        dst[g] = make_uint4(
                            pack_bf16(__uint_as_float(ov[g * 8 + 0]) * il, __uint_as_float(ov[g * 8 + 1]) * il),
                            pack_bf16(__uint_as_float(ov[g * 8 + 2]) * il, __uint_as_float(ov[g * 8 + 3]) * il),
                            pack_bf16(__uint_as_float(ov[g * 8 + 4]) * il, __uint_as_float(ov[g * 8 + 5]) * il),
                            pack_bf16(__uint_as_float(ov[g * 8 + 6]) * il, __uint_as_float(ov[g * 8 + 7]) * il));
                } else {
                    float4* dst = reinterpret_cast<float4*>(a.o_part + (int64_t(sp) * a.n + row) * a.d + col);
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        dst[g] = make_float4(__uint_as_float(ov[4 * g]), __uint_as_float(ov[4 * g + 1]),
                                             __uint_as_float(ov[4 * g + 2]), __uint_as_float(ov[4 * g + 3]));
                    if (team == 0 && half == 0) {
                        const int64_t o = (int64_t(sp) * a.n + row) * a.H + head;
                        a.m_part[o] = M;
                        a.l_part[o] = L;
                    }
                }
            }
        } else {
            if (niter > 0) {
                mbar_wait(o_full, 0);
                fence_after();
                // this team's last chunk (its lag-2 flushes covered the rest)
                const int last = ((niter - 1 - team) >= 0) ? niter - 1 - ((niter - 1 - team) & 1) : -1;
                if (bins && last >= 0) flush_bins(last);
            }
            // norm_end: l of each row = the 4 (team, half) partials, fixed order
            float o_scale = 1.f, l_row = 0.f;
            if (a.norm_end) {
                float* lp = part;  // [4][128] (the bins partials are unused without a summary)
                lp[(team * 2 + half) * TM + r] = lsum;
                named_sync(1, NTEAM * 256);
                l_row = ((lp[r] + lp[TM + r]) + lp[2 * TM + r]) + lp[3 * TM + r];
                o_scale = (a.nsplit == 1 && l_row > 0.f) ? 1.f / l_row : 1.f;
                if (a.nsplit > 1 && rvalid && team == 0 && half == 0)
                    a.l_part[(int64_t(sp) * a.n + row) * a.H + head] = l_row;
            }
            // O columns [32 g, 32 g + 32), g = 2 team + half
            const int oc = 32 * (team * 2 + half);
            uint32_t ov[32];
            if (niter > 0) {
                tmem_ld32(tm_o + lane_base + uint32_t(oc), ov);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = 0u;
            }
            if (o_scale != 1.f)
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * o_scale);
            if (rvalid) {
                const int col = head * DH + oc;
                if (a.nsplit == 1) {
                    uint4* dst = reinterpret_cast<uint4*>(a.ctx + int64_t(row) * a.d + col);
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        dst[g] = make_uint4(pack_bf16(__uint_as_float(ov[g * 8 + 0]), __uint_as_float(ov[g * 8 + 1])),
                                            pack_bf16(__uint_as_float(ov[g * 8 + 2]), __uint_as_float(ov[g * 8 + 3])),
                                            pack_bf16(__uint_as_float(ov[g * 8 + 4]), __uint_as_float(ov[g * 8 + 5])),
                                            pack_bf16(__uint_as_float(ov[g * 8 + 6]), __uint_as_float(ov[g * 8 + 7])));
                } else {
                    float4* dst = reinterpret_cast<float4*>(a.o_part + (int64_t(sp) * a.n + row) * a.d + col);
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        dst[g] = make_float4(__uint_as_float(ov[4 * g]), __uint_as_float(ov[4 * g + 1]),
                                             __uint_as_float(ov[4 * g + 2]), __uint_as_float(ov[4 * g + 3]));
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        tmem_dealloc(tmem, LY::TMEM_COLS);
    }
}

// Z^T tiles of the segment summary: for 128-key chunk c, row j of tile c is
// the indicator of the keys of destination segment d0(c) + j (bf16 0/1);
// rows >= nseg(c) and query keys are zero.  Prefill constant.
__global__ void zt_build_kernel(const int32_t* __restrict__ row_seg, int T, const int4* __restrict__ tab, int NB,
                                int nchunks, __nv_bfloat16* __restrict__ zt) {
    const int64_t total = int64_t(nchunks) * NB * TK;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int k = int(e % TK);
        const int64_t rj = e / TK;
        const int j = int(rj % NB), c = int(rj / NB);
        const int key = c * TK + k;
        const int4 hdr = tab[2 * c];
        const int sk = key < T ? row_seg[key] : -1;
        zt[e] = __float2bfloat16_rn((sk >= 0 && j < hdr.y && sk == hdr.x + j) ? 1.f : 0.f);
    }
}

// m = max_s m_s, l = sum_s l_s 2^(m_s - m)  (split order fixed); inv_l = 1/l
__global__ void tc_stats_combine(const float* __restrict__ mp, const float* __restrict__ lp, int nsplit,
                                 int64_t nh, float* __restrict__ m_fin, float* __restrict__ inv_l) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nh; e += int64_t(gridDim.x) * blockDim.x) {
        float m = -FLT_MAX;
        for (int s = 0; s < nsplit; ++s) m = fmaxf(m, mp[s * nh + e]);
        float l = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float ms = mp[s * nh + e];
            if (ms > -FLT_MAX) l += lp[s * nh + e] * exp2f(ms - m);
        }
        m_fin[e] = m;
        inv_l[e] = l > 0.f ? 1.f / l : 0.f;
    }
}

// FLASH splits: each split's (m, l, O) relative to its own max
__global__ void tc_flash_combine(const float* __restrict__ m_part, const float* __restrict__ l_part,
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

// lp != nullptr (norm_end): the partials are unnormalised with one global max,
// ctx = sum_s O_s / sum_s l_s
__global__ void tc_ctx_combine(const float* __restrict__ op, int nsplit, int64_t nd, __nv_bfloat16* __restrict__ ctx,
                               const float* __restrict__ lp, int d, int H, int64_t nh) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nd; e += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int s = 0; s < nsplit; ++s) acc += op[s * nd + e];
        if (lp) {
            const int64_t rh = (e / d) * H + (e % d) / DH;
            float l = 0.f;
            for (int s = 0; s < nsplit; ++s) l += lp[s * nh + rh];
            acc = l > 0.f ? acc / l : 0.f;
        }
        ctx[e] = __float2bfloat16_rn(acc);
    }
}

// Per 128-key chunk c: the destination segments whose last key (or the chunk
// end) falls inside the chunk, as a boundary bit mask, plus the first such
// segment.  Depends only on the layout, so it is built once per prefill.
__global__ void chunk_table_kernel(const int32_t* __restrict__ row_seg, int T, int nchunks, int4* __restrict__ tab) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    uint32_t m[4] = {0, 0, 0, 0};
    int d0 = -1, nseg = 0;
    for (int k = 0; k < TK; ++k) {
        const int key = c * TK + k;
        const int sk = key < T ? row_seg[key] : -1;
        const int sn = (k + 1 < TK && key + 1 < T) ? row_seg[key + 1] : -2;
        if (sk >= 0 && sn != sk) {
            m[k >> 5] |= 1u << (k & 31);
            if (d0 < 0) d0 = sk;
            ++nseg;
        }
    }
    tab[2 * c] = make_int4(d0 < 0 ? 0 : d0, nseg, 0, 0);
    tab[2 * c + 1] = make_int4(int(m[0]), int(m[1]), int(m[2]), int(m[3]));
}

// raw summary -> AttentionSummary: qts/qlen, sts[i][j]/seg_len[i] for j < i
// (prefill.hpp:306-315)
__global__ void summary_normalize(const double* __restrict__ qraw, const double* __restrict__ sraw, int S,
                                  const int32_t* __restrict__ seg_len, int qlen, double* __restrict__ summ) {
    const int i = int(blockIdx.y) - 1;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S; j += gridDim.x * blockDim.x) {
        if (i < 0) summ[j] = qlen > 0 ? qraw[j] / double(qlen) : 0.0;
        else summ[S + int64_t(i) * S + j] = j < i ? sraw[int64_t(i) * S + j] / double(seg_len[i]) : 0.0;
    }
}

// V [T x d] -> V^T [d x ldt] (bf16), 64x64 tiles through shared memory;
// padding keys [T, ldt) are written as zero.
__global__ void transpose_bf16(const __nv_bfloat16* __restrict__ v, int T, int d, int64_t ldt,
                               __nv_bfloat16* __restrict__ vt) {
    __shared__ __nv_bfloat16 tile[64][66];
    const int t0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
        const int r = e / 64, c = e % 64;
        tile[r][c] = (t0 + r < T) ? v[int64_t(t0 + r) * d + c0 + c] : __float2bfloat16_rn(0.f);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
        const int r = e / 64, c = e % 64;  // out row c0+r, col t0+c
        vt[int64_t(c0 + r) * ldt + t0 + c] = tile[c][r];
    }
}

template <int MODE>
void launch_mode(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& vt, const TcArgs& a, dim3 grid,
                 cudaStream_t st) {
    using LY = Layout<MODE>;
    smem_attr(attn_tc_kernel<MODE>, int(LY::SMEM));
    attn_tc_kernel<MODE><<<grid, NTHR, LY::SMEM, st>>>(q, k, vt, a);
    KEEP_LAUNCH_CHECK();
}

static_assert(Layout<MODE_CTX>::SMEM <= 232448, "CTX smem");

template <int MODE, int NB>
void launch_mode2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& vt, const CUtensorMap& z,
                  const TcArgs& a, dim3 grid, cudaStream_t st) {
    using LY = Layout2<MODE, NB>;
    smem_attr(attn_tc2_kernel<MODE, NB>, int(LY::SMEM));
    attn_tc2_kernel<MODE, NB><<<grid, NTHR2, LY::SMEM, st>>>(q, k, vt, z, a);
    KEEP_LAUNCH_CHECK();
}

bool flash_enabled() {  // KEEP_ATTN_FLASH=0: the two-pass form also without a summary (A/B)
    static const bool v = [] {
        const char* e = std::getenv("KEEP_ATTN_FLASH");
        return !(e && *e == '0');
    }();
    return v;
}

bool force_v1() {
    static const bool v = [] {
        const char* e = std::getenv("KEEP_ATTN_V1");
        return e && *e == '1';
    }();
    return v;
}

}  // namespace

void launch_chunk_table(const int32_t* row_seg, int T, void* tab, cudaStream_t st) {
    const int nchunks = int(ceil_div(T, TK));
    chunk_table_kernel<<<unsigned(ceil_div(nchunks, 128)), 128, 0, st>>>(row_seg, T, nchunks, static_cast<int4*>(tab));
    KEEP_LAUNCH_CHECK();
}

// Summary bins on the tensor core (default) or, with KEEP_BINS=scan, the
// CUDA-core scan (A/B reference for the tensor-core path).
bool bins_on_tensor_core() {
    static const bool v = [] {
        const char* e = std::getenv("KEEP_BINS");
        return !(e && std::string(e) == "scan");
    }();
    return v;
}

int summary_bins_width(const std::vector<int32_t>& row_seg) {
    const int T = int(row_seg.size());
    int mx = 0;
    for (int c0 = 0; c0 < T; c0 += TK) {
        int n = 0, prev = INT32_MIN;
        for (int k = c0; k < std::min(T, c0 + TK); ++k)
            if (row_seg[k] >= 0 && row_seg[k] != prev) {
                ++n;
                prev = row_seg[k];
            }
        mx = std::max(mx, n);
    }
    if (force_v1()) return 0;
    return mx <= 16 ? 16 : mx <= 32 ? 32 : 0;
}

void launch_zt_build(const int32_t* row_seg, int T, const void* tab, int nb, void* zt, cudaStream_t st) {
    const int nchunks = int(ceil_div(T, TK));
    const int64_t total = int64_t(nchunks) * nb * TK;
    zt_build_kernel<<<unsigned(std::min<int64_t>(ceil_div(total, 256), kNumSMs * 8)), 256, 0, st>>>(
        row_seg, T, static_cast<const int4*>(tab), nb, nchunks, static_cast<__nv_bfloat16*>(zt));
    KEEP_LAUNCH_CHECK();
}

// Host driver of the two passes (see file comment).
int launch_attention_tc(const AttnTcLaunch& L, cudaStream_t st) {
    const int n = L.n, T = L.T, H = L.H, d = L.d;
    if (n == 0) return 0;
    int launched = 0;
    const int tiles = int(ceil_div(n, TM));
    const bool v2 = !force_v1() && (!L.with_bins || (L.nb > 0 && bins_on_tensor_core()));
    const CUtensorMap mq = make_map_bf16(L.q, n, d, d, 128);
    const CUtensorMap mk = make_map_bf16(L.k, T, d, d, 128);
    CUtensorMap mv;
    if (v2) {
        mv = make_map_bf16(L.v, T, d, d, 128);  // V as stored: MN-major B operand
    } else {
        // v1: V^T for the P.V operand (K-major over keys); inner extent padded
        // to a multiple of 64 keys so TMA boxes never straddle a ragged edge
        const int64_t ldt = ceil_div(T, 64) * 64;
        dim3 g(unsigned(ceil_div(T, 64)), unsigned(d / 64));
        transpose_bf16<<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(L.v), T, d, ldt, L.vt);
        KEEP_LAUNCH_CHECK();
        ++launched;
        mv = make_map_bf16(L.vt, d, ldt, ldt, 128);
    }

    TcArgs a{};
    a.n = n;
    a.T = T;
    a.H = H;
    a.d = d;
    a.S = L.S;
    a.rows = L.rows;
    a.row_seg = L.row_seg;
    a.key_lo = L.key_lo;
    // q arrives pre-scaled by log2(e)/sqrt(dh) (QKV epilogue, before its bf16
    // rounding): the scores are already in the exp2 domain, so both passes
    // subtract the row max from the SAME fp32 value.  Folding the scale into an
    // fma here instead would make the max element's exponent the rounding
    // error of s*scale -- up to ulp(m)/2, i.e. 2^30+ once deep-layer logits
    // reach 1e9 -- and blow p far above 1.
    a.scale_log2 = 1.f;
    a.inv_heads = float(L.inv_heads);
    a.m_part = L.m_part;
    a.l_part = L.l_part;
    a.m_fin = L.m_fin;
    a.inv_l = L.inv_l;
    a.o_part = L.o_part;
    a.ctx = L.ctx;
    a.nsplit = L.nsplit_a;
    a.split_lo = L.split_lo_a;
    a.split_hi = L.split_hi_a;
    a.qts_raw = L.with_bins ? L.summ_raw : nullptr;
    a.sts_raw = L.with_bins ? L.summ_raw + L.S : nullptr;
    a.chunk_tab = reinterpret_cast<const int4*>(L.chunk_tab);
    if (L.with_bins)
        KEEP_CUDA(cudaMemsetAsync(L.summ_raw, 0, sizeof(double) * (size_t(L.S) + size_t(L.S) * L.S), st));

    // v2 (384 threads, summary bins on the tensor core) unless the layout has
    // more than 32 segments in some 128-key chunk (then the v1 scan bins)
    const dim3 grid(tiles, H, a.nsplit);
    {
        // without a summary the v2 passes need no normalised p: max-only STATS,
        // l summed by the CTX pass
        const char* e = std::getenv("KEEP_DEBUG_NO_BINS");
        const bool no_bins = !L.with_bins || (e && *e == '1');
        a.norm_end = (v2 && no_bins) ? 1 : 0;
    }
    {
        const char* e = std::getenv("KEEP_DEBUG_ATTN");
        a.dbg = e ? std::atoi(e) : 0;
    }
    if (v2 && a.norm_end && flash_enabled()) {
        // no summary: single pass with online softmax (no STATS pass, K read once)
        launch_mode2<MODE_FLASH, 16>(mq, mk, mv, mq, a, grid, st);
        ++launched;
        if (a.nsplit > 1) {
            const int64_t nd = int64_t(n) * d;
            tc_flash_combine<<<unsigned(std::min<int64_t>(ceil_div(nd, 256), kNumSMs * 16)), 256, 0, st>>>(
                L.m_part, L.l_part, L.o_part, a.nsplit, n, H, d, L.ctx);
            KEEP_LAUNCH_CHECK();
            ++launched;
        }
        return launched;
    }
    if (v2) { launch_mode2<MODE_STATS, 16>(mq, mk, mv, mq, a, grid, st); ++launched; }
    else { launch_mode<MODE_STATS>(mq, mk, mv, a, grid, st); ++launched; }
    const int64_t nh = int64_t(n) * H;
    tc_stats_combine<<<unsigned(std::min<int64_t>(ceil_div(nh, 256), kNumSMs * 8)), 256, 0, st>>>(
        L.m_part, L.l_part, a.nsplit, nh, L.m_fin, L.inv_l);
    KEEP_LAUNCH_CHECK();
        ++launched;
    static const bool dbg_no_bins = [] {  // A/B timing aid: KEEP_DEBUG_NO_BINS=1 drops the summary
        const char* e = std::getenv("KEEP_DEBUG_NO_BINS");
        return e && *e == '1';
    }();
    if (v2 && dbg_no_bins) a.sts_raw = nullptr;
    {
        const char* e = std::getenv("KEEP_DEBUG_ATTN");
        a.dbg = e ? std::atoi(e) : 0;
    }

    if (v2) {
        if (L.with_bins && !dbg_no_bins) {
            const int nchunks = int(ceil_div(T, TK));
            {
            const CUtensorMap mz = make_map_bf16(L.zt, int64_t(nchunks) * L.nb, TK, TK, L.nb);
            if (L.nb == 16) { launch_mode2<MODE_CTX, 16>(mq, mk, mv, mz, a, grid, st); ++launched; }
            else { launch_mode2<MODE_CTX, 32>(mq, mk, mv, mz, a, grid, st); ++launched; }
            }
        } else {
            { launch_mode2<MODE_CTX, 16>(mq, mk, mv, mq, a, grid, st); ++launched; }
        }
    } else {
        launch_mode<MODE_CTX>(mq, mk, mv, a, grid, st);
        ++launched;
    }
    if (a.nsplit > 1) {
        const int64_t nd = int64_t(n) * d;
        tc_ctx_combine<<<unsigned(std::min<int64_t>(ceil_div(nd, 256), kNumSMs * 16)), 256, 0, st>>>(
            L.o_part, a.nsplit, nd, L.ctx, a.norm_end ? L.l_part : nullptr, d, H, int64_t(n) * H);
        KEEP_LAUNCH_CHECK();
        ++launched;
    }
    if (L.with_bins) {
        dim3 g(unsigned(ceil_div(L.S, 256)), unsigned(L.S + 1));
        summary_normalize<<<g, 256, 0, st>>>(L.summ_raw, L.summ_raw + L.S, L.S, L.seg_len, L.qlen, L.summ);
        KEEP_LAUNCH_CHECK();
        ++launched;
    }
    return launched;
}

}  // namespace keep_b200
