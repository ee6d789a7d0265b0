// gemm_oz.cu -- PARITY projection GEMM on the int8 tensor cores (Ozaki scheme).
//
//   C[M x N] = A[M x K] . B[K x N]     fp32 operands, fp64-grade accumulation
//
// The reference computes every projection with fp32 storage and an fp64
// accumulator (vec_mat, tensor.hpp:31-41).  DFMA on the CUDA cores does that
// at ~14 TFLOP/s (gemm_f64acc.cu).  Here the same product runs on the
// 5th-generation tensor cores in exact integer arithmetic:
//
//  * every row of A is scaled by a power of two 2^ea[m] so its largest
//    element lies in [32, 64), and split into s signed 8-bit digits
//        x * 2^ea = d0 + d1 / 256 + ... + d_{s-1} / 256^(s-1) + r,
//    d0 in [-65, 65], d_p in [-128, 127] (split_digits), |r| <= 2^-(8s-7);
//    every column of B likewise with 2^eb[n] (oz_split_rows / oz_split_cols);
//  * x.w = sum_{p,q} d_p e_q 256^-(p+q).  Level k collects the digit pairs
//    with p + q = k (k < s, the standard triangular truncation); one level
//    is an int8 GEMM with K' = (k+1) K accumulated EXACTLY in int32 TMEM
//    (tcgen05.mma kind::i8; |d_p e_q| <= 2^14, so (k+1) K <= 2^17 keeps the
//    sum below 2^31 -- longer levels are split into several units);
//  * the levels are combined in fp64 in Horner order from the smallest
//    (P = D_{s-1}; P = D_k + P / 256; ...), then scaled by 2^-(ea+eb) and
//    rounded once to fp32 -- the reference's "fp64 accumulate, cast" with an
//    error of ~2^-(8s-10) of max|x| max|w| per product instead of 2^-53.
//
// That is the same grade as the fp64 re-ordering the PARITY attention already
// has (any fp64 order reproduced every plan); the int8
// tensor cores do it at ~4.5 POPS against ~40 TFLOP/s of DFMA.
//
// Kernel structure = gemm_tc.cu's (persistent, warp-specialised, TMA ring,
// double-buffered TMEM accumulators, 128 x 256 tiles), with a work unit =
// (tile, level unit) and an epilogue that keeps the fp64 Horner partial of
// its tile in a per-CTA scratch (L2-resident: 256 KB x 148 CTAs).
#include <cstring>

#include "engine.hpp"
#include "tc_common.cuh"

namespace keep_b200 {

namespace {

using namespace tc;

constexpr int OBM = 128, OBN = 256, OBK = 128;  // OBK bytes = int8 elements per stage
constexpr int OSTAGES = 4;
constexpr int OTHREADS = 256;
constexpr int OGM = 16;
constexpr int kMaxUnits = 32;
constexpr uint32_t OA_BYTES = OBM * OBK, OB_BYTES = OBN * OBK, OSTAGE = OA_BYTES + OB_BYTES;
constexpr size_t OSMEM = size_t(OSTAGES) * OSTAGE + 1024 + 256;

// kind::i8 instruction descriptor: D s32, A / B signed 8-bit, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

// A unit: digit pairs (p, k - p) for p in [pb, pe) of level k, one int32
// accumulation.  op: 0 P = D; 1 P = D + P/256 (next level); 2 P = P + D (same level).
struct OzUnit {
    int8_t k, pb, pe, op;
};
struct OzPlan {
    int nunits;
    OzUnit u[kMaxUnits];
};

__device__ __forceinline__ void otile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
    const int band = t / (OGM * tiles_n);
    const int m0 = band * OGM;
    const int gm = min(OGM, tiles_m - m0);
    const int r = t - band * OGM * tiles_n;
    mb = m0 + r % gm;
    nb = r / gm;
}

__device__ __forceinline__ void epi_store32(const EpiArgs& e, int m, int n, int N, const float (&v)[32]) {
    switch (e.kind) {
        case EPI_QKV: {
            const int d = e.d;
            float* dst;
            if (n < d) dst = e.out + int64_t(m) * e.ldo + n;
            else if (n < 2 * d) dst = static_cast<float*>(e.kdst) + int64_t(e.rows[m]) * d + (n - d);
            else dst = static_cast<float*>(e.vdst) + int64_t(e.rows[m]) * d + (n - 2 * d);
            // a 32-column chunk never straddles the q / k / v boundary (d % 32 == 0)
#pragma unroll
            for (int q = 0; q < 8; ++q)
                reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            break;
        }
        case EPI_RESID: {
            float4* x = reinterpret_cast<float4*>(e.out + int64_t(m) * e.ldo + n);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float4 t = x[q];
                t.x += v[4 * q];
                t.y += v[4 * q + 1];
                t.z += v[4 * q + 2];
                t.w += v[4 * q + 3];
                x[q] = t;
            }
            break;
        }
        case EPI_RELU: {
            float4* o = reinterpret_cast<float4*>(e.out + int64_t(m) * e.ldo + n);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                o[q] = make_float4(fmaxf(v[4 * q], 0.f), fmaxf(v[4 * q + 1], 0.f), fmaxf(v[4 * q + 2], 0.f),
                                   fmaxf(v[4 * q + 3], 0.f));
            break;
        }
        default: {
            float4* o = reinterpret_cast<float4*>(e.out + int64_t(m) * e.ldo + n);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
    (void)N;
}

__global__ void __launch_bounds__(OTHREADS, 1)
gemm_oz_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
               int Mp, int Np, const __grid_constant__ OzPlan plan, const int* __restrict__ ea,
               const int* __restrict__ eb, double* __restrict__ scratch, EpiArgs epi) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + OSTAGES * OSTAGE);
    uint64_t* empty = full + OSTAGES;
    uint64_t* tfull = empty + OSTAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_m = int(ceil_div(M, OBM)), tiles_n = int(ceil_div(N, OBN));
    const int ntiles = tiles_m * tiles_n;
    const int kblocks = int(ceil_div(K, OBK));
    const int U = plan.nunits;

    if (warp == 0 && lane == 0) {
        prefetch_map(&tmA);
        prefetch_map(&tmB);
        for (int s = 0; s < OSTAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mb, nb;
                otile_coords(t, tiles_m, tiles_n, mb, nb);
                for (int u = 0; u < U; ++u) {
                    const OzUnit un = plan.u[u];
                    for (int p = un.pb; p < un.pe; ++p) {
                        const int q = un.k - p;
                        for (int kb = 0; kb < kblocks; ++kb) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            uint8_t* sa = smem + stage * OSTAGE;
                            mbar_expect_tx(&full[stage], OSTAGE);
                            tma_load_2d(sa, &tmA, &full[stage], kb * OBK, p * Mp + mb * OBM);
                            tma_load_2d(sa + OA_BYTES, &tmB, &full[stage], kb * OBK, q * Np + nb * OBN);
                            if (++stage == OSTAGES) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer
        constexpr uint32_t idesc = idesc_i8(OBM, OBN);
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int u = 0; u < U; ++u, ++it) {
                const OzUnit un = plan.u[u];
                const int acc = it & 1;
                mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t tmem_d = tmem_base + uint32_t(acc * OBN);
                bool first = true;
                for (int p = un.pb; p < un.pe; ++p) {
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&full[stage], phase);
                        fence_after();
                        const uint32_t sa = smem_u32(smem + stage * OSTAGE);
                        const uint64_t ad = smem_desc(sa), bd = smem_desc(sa + OA_BYTES);
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < OBK / 32; ++k)  // 32 int8 = 32 bytes per MMA
                                umma_i8(tmem_d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                        (first && k == 0) ? 0u : 1u);
                            umma_commit(&empty[stage]);
                        }
                        __syncwarp();
                        first = false;
                        if (++stage == OSTAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                if (elect_one()) umma_commit(&tfull[acc]);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue: fp64 Horner over the levels
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;  // tile row = TMEM lane
        double* P = scratch + size_t(blockIdx.x) * OBM * OBN;  // [col][row]
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int mb, nb;
            otile_coords(t, tiles_m, tiles_n, mb, nb);
            const int m = mb * OBM + r;
            const bool mok = m < M;
            const int eam = mok ? ea[m] : 0;
            for (int u = 0; u < U; ++u, ++it) {
                const int op = plan.u[u].op;
                const bool last = u == U - 1;
                const int acc = it & 1;
                mbar_wait(&tfull[acc], (it >> 1) & 1);
                fence_after();
#pragma unroll 1
                for (int ch = 0; ch < OBN / 32; ++ch) {
                    uint32_t d[32];
                    tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * OBN + ch * 32), d);
                    const int n0 = nb * OBN + ch * 32;
                    if (n0 >= N) continue;
                    double* pc = P + size_t(ch * 32) * OBM + r;
                    if (!last) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const double dv = double(int(d[j]));
                            double pv;
                            if (op == 0) pv = dv;
                            else if (op == 1) pv = fma(pc[j * OBM], 0.00390625, dv);
                            else pv = pc[j * OBM] + dv;
                            pc[j * OBM] = pv;
                        }
                    } else if (mok) {
                        float v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const double dv = double(int(d[j]));
                            double pv;
                            if (op == 0) pv = dv;
                            else if (op == 1) pv = fma(pc[j * OBM], 0.00390625, dv);
                            else pv = pc[j * OBM] + dv;
                            const int n = n0 + j;
                            const int e = eam + (n < N ? eb[n] : 0);
                            v[j] = float(ldexp(pv, -e));
                        }
                        epi_store32(epi, m, n0, N, v);
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------- splits --
// x * 2^e with max |x| * 2^e in [32, 64): e = 6 - exponent(max) (frexp).
__device__ __forceinline__ int scale_exp(float amax) {
    if (!(amax > 0.f)) return 0;
    int ex;
    frexpf(amax, &ex);
    return 6 - ex;
}

// s base-256 digits of v = x 2^e (|v| < 64), most significant first:
//   d_p = floor(v_p + 1/2),  v_{p+1} = 256 (v_p - d_p)     (exact in fp64)
// leaves d_p in [-128, 128]; a digit of 128 becomes -128 with a carry of one
// into the digit above (128 / 256^p = 1 / 256^(p-1) - 128 / 256^p), so every
// digit fits int8: d_0 in [-65, 65], d_p in [-128, 127].
__device__ __forceinline__ void split_digits(double v, int s, int (&dd)[8]) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        if (p < s) {
            const double f = floor(v + 0.5);
            dd[p] = int(f);
            v = (v - f) * 256.0;
        } else {
            dd[p] = 0;
        }
    }
#pragma unroll
    for (int p = 7; p >= 1; --p)
        if (dd[p] == 128) {
            dd[p] = -128;
            dd[p - 1] += 1;
        }
}

// A rows -> out[p][m][0..Kp) int8 digits + ea[m]; one warp per row.
__global__ void oz_split_rows_kernel(const float* __restrict__ A, int64_t lda, int M, int K, int Kp, int s, int Mp,
                                     int8_t* __restrict__ out, int* __restrict__ ea) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= M) return;
    const float* a = A + int64_t(warp) * lda;
    float mx = 0.f;
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(a[k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int e = scale_exp(mx);
    if (lane == 0) ea[warp] = e;
    const size_t plane = size_t(Mp) * Kp;
    int8_t* o = out + size_t(warp) * Kp;
    for (int k0 = lane * 4; k0 < Kp; k0 += 128) {
        int dd[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i) split_digits(ldexp(double((k0 + i < K) ? a[k0 + i] : 0.f), e), s, dd[i]);
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            if (p >= s) break;
            char4 dg;
            dg.x = int8_t(dd[0][p]);
            dg.y = int8_t(dd[1][p]);
            dg.z = int8_t(dd[2][p]);
            dg.w = int8_t(dd[3][p]);
            *reinterpret_cast<char4*>(o + p * plane + k0) = dg;
        }
    }
}

// column max |B[k][n]| over k: fp32 bit patterns of non-negative values order
// like the values, so an integer atomicMax reduces them exactly
__global__ void oz_colmax_kernel(const float* __restrict__ B, int64_t ldb, int K, int N, int krows,
                                 unsigned* __restrict__ cmax) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int k0 = blockIdx.y * krows, k1 = min(K, k0 + krows);
    float mx = 0.f;
    for (int k = k0; k < k1; ++k) mx = fmaxf(mx, fabsf(B[int64_t(k) * ldb + n]));
    atomicMax(cmax + n, __float_as_uint(mx));
}

// B [K x N] row-major -> out[q][n][0..Kp) int8 digits (transposed, K-major) +
// eb[n].  Tile 128 k x 32 n through shared memory.
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const float* __restrict__ B, int64_t ldb, int K, int N,
                                                            int Kp, int s, int Np, const unsigned* __restrict__ cmax,
                                                            int8_t* __restrict__ out, int* __restrict__ eb) {
    __shared__ int8_t sd[8][32][128 + 16];
    const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 128;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
    const int n = n0 + tx;
    const int e = n < N ? scale_exp(__uint_as_float(cmax[n])) : 0;
    if (blockIdx.y == 0 && ty == 0 && n < N) eb[n] = e;
    for (int kk = ty; kk < 128; kk += 8) {
        const int k = k0 + kk;
        const float x = (k < K && n < N) ? B[int64_t(k) * ldb + n] : 0.f;
        int dd[8];
        split_digits(ldexp(double(x), e), s, dd);
#pragma unroll
        for (int p = 0; p < 8; ++p)
            if (p < s) sd[p][tx][kk] = int8_t(dd[p]);
    }
    __syncthreads();
    // write rows (q, n): 128 contiguous bytes = 8 x 16 B
    const size_t plane = size_t(Np) * Kp;
    for (int idx = threadIdx.x; idx < s * 32 * 8; idx += 256) {
        const int q = idx / 256, rem = idx % 256, nn = rem / 8, c = rem % 8;
        if (n0 + nn >= N || k0 + c * 16 >= Kp) continue;
        const int4 v = *reinterpret_cast<const int4*>(&sd[q][nn][c * 16]);
        *reinterpret_cast<int4*>(out + q * plane + size_t(n0 + nn) * Kp + k0 + c * 16) = v;
    }
}

CUtensorMap make_map_i8(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    CUtensorMap tm;
    const cuuint64_t gdim[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t gstride[1] = {cuuint64_t(ld)};
    const cuuint32_t box[2] = {cuuint32_t(OBK), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), gdim, gstride, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(KEEP_ERR_CUDA, "cuTensorMapEncodeTiled (int8) failed: " + std::to_string(int(r)));
    return tm;
}

OzPlan make_plan(int s, int K) {
    // int32 safety: a unit sums pairs * K products of magnitude <= 2^14
    const int max_pairs = std::max(1, int((int64_t(1) << 17) / std::max(K, 1)));
    if (max_pairs < 1) raise(KEEP_ERR_CONFIG, "Ozaki GEMM: K too large");
    OzPlan pl{};
    pl.nunits = 0;
    for (int k = s - 1; k >= 0; --k) {
        const int np = k + 1;  // pairs (p, k - p), p = 0..k
        for (int pb = 0; pb < np; pb += max_pairs) {
            if (pl.nunits >= kMaxUnits) raise(KEEP_ERR_CONFIG, "Ozaki GEMM: too many level units");
            OzUnit& u = pl.u[pl.nunits];
            u.k = int8_t(k);
            u.pb = int8_t(pb);
            u.pe = int8_t(std::min(np, pb + max_pairs));
            u.op = int8_t(pl.nunits == 0 ? 0 : (pb == 0 ? 1 : 2));
            ++pl.nunits;
        }
    }
    return pl;
}

}  // namespace

int oz_slices() {
    static const int s = [] {
        const char* e = std::getenv("KEEP_OZ_SLICES");
        const int v = e ? std::atoi(e) : 7;
        return std::min(8, std::max(2, v));
    }();
    return s;
}

// KEEP_PARITY_GEMM=dfma|ozaki|auto (default auto: Ozaki from kOzMinRows rows)
int parity_gemm_mode() {
    static const int m = [] {
        const char* e = std::getenv("KEEP_PARITY_GEMM");
        if (!e) return 0;
        if (!std::strcmp(e, "dfma")) return 2;
        if (!std::strcmp(e, "ozaki")) return 1;
        return 0;
    }();
    return m;
}

bool ozaki_eligible(int M, int N, int K) {
    return K % 16 == 0 && N % 32 == 0 && (parity_gemm_mode() == 1 || (parity_gemm_mode() == 0 && M >= kOzMinRows));
}

void launch_gemm_ozaki(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                       const EpiArgs& epi, cudaStream_t st, OzWork& w, int max_ctas) {
    if (M == 0 || N == 0) return;
    const int s = oz_slices();
    const int Mp = int(ceil_div(M, OBM) * OBM), Np = int(ceil_div(N, OBN) * OBN);
    const int Kp = int(ceil_div(K, 16) * 16);
    w.a.ensure(size_t(s) * Mp * Kp);
    w.b.ensure(size_t(s) * Np * Kp);
    w.ea.ensure(sizeof(int) * size_t(Mp));
    w.eb.ensure(sizeof(int) * size_t(Np) + sizeof(unsigned) * size_t(N));
    int* eb = w.eb.as<int>();
    unsigned* cmax = reinterpret_cast<unsigned*>(eb + Np);
    // digits of A (rows) and B (columns)
    oz_split_rows_kernel<<<unsigned(ceil_div(M, 8)), 256, 0, st>>>(A, lda, M, K, Kp, s, Mp, w.a.as<int8_t>(),
                                                                    w.ea.as<int>());
    KEEP_LAUNCH_CHECK();
    KEEP_CUDA(cudaMemsetAsync(cmax, 0, sizeof(unsigned) * size_t(N), st));
    const int ksplit = int(std::min<int64_t>(64, ceil_div(K, 64)));
    const int krows = int(ceil_div(K, ksplit));
    oz_colmax_kernel<<<dim3(unsigned(ceil_div(N, 256)), unsigned(ksplit)), 256, 0, st>>>(B, ldb, K, N, krows, cmax);
    KEEP_LAUNCH_CHECK();
    oz_split_cols_kernel<<<dim3(unsigned(ceil_div(N, 32)), unsigned(ceil_div(Kp, 128))), 256, 0, st>>>(
        B, ldb, K, N, Kp, s, Np, cmax, w.b.as<int8_t>(), eb);
    KEEP_LAUNCH_CHECK();
    // the GEMM
    smem_attr(gemm_oz_kernel, int(OSMEM));
    const OzPlan plan = make_plan(s, K);
    const CUtensorMap ta = make_map_i8(w.a.p, int64_t(s) * Mp, K, Kp, OBM);
    const CUtensorMap tb = make_map_i8(w.b.p, int64_t(s) * Np, K, Kp, OBN);
    const int ntiles = int(ceil_div(M, OBM) * ceil_div(N, OBN));
    const int grid = std::min(ntiles, std::max(1, std::min(max_ctas, kNumSMs)));
    w.part.ensure(sizeof(double) * size_t(grid) * OBM * OBN);
    gemm_oz_kernel<<<grid, OTHREADS, OSMEM, st>>>(ta, tb, M, N, K, Mp, Np, plan, w.ea.as<int>(), eb,
                                                  w.part.as<double>(), epi);
    KEEP_LAUNCH_CHECK();
}

void launch_gemm_parity(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                        const EpiArgs& epi, cudaStream_t st, OzWork& w, bool exact, int max_ctas) {
    if (!exact && ozaki_eligible(M, N, K) && (epi.kind != EPI_QKV || epi.d % 32 == 0)) launch_gemm_ozaki(A, lda, B, ldb, M, N, K, epi, st, w, max_ctas);
    else launch_gemm_f64acc(A, lda, B, ldb, M, N, K, epi, st);
}

}  // namespace keep_b200

// Test hook: C = A . B on device pointers (fp32 [M x K] . [K x N] -> fp32),
// mode 0 auto, 1 Ozaki, 2 DFMA.
extern "C" int keep_debug_gemm_parity(const float* A, const float* B, float* Cout, int M, int N, int K, int mode) {
    try {
        keep_b200::EpiArgs e{keep_b200::EPI_STORE, 0, Cout, N, nullptr, nullptr, nullptr, nullptr};
        thread_local keep_b200::OzWork w;
        if (mode == 1 || (mode == 0 && keep_b200::ozaki_eligible(M, N, K)))
            keep_b200::launch_gemm_ozaki(A, K, B, N, M, N, K, e, 0, w, keep_b200::kNumSMs);
        else
            keep_b200::launch_gemm_f64acc(A, K, B, N, M, N, K, e, 0);
        return cudaDeviceSynchronize() == cudaSuccess ? 0 : KEEP_ERR_CUDA;
    } catch (const keep_b200::KeepError& e) {
        return e.code;
    }
}
