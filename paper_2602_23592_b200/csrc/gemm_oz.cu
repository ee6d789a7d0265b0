// gemm_oz.cu -- PARITY projection GEMM on the int8 tensor cores (Ozaki scheme
// II: integer residues and the Chinese remainder theorem).
//
//   C[M x N] = A[M x K] . B[K x N]     fp32 operands, fp64-grade accumulation
//
// The reference computes every projection with fp32 storage and an fp64
// accumulator (vec_mat, tensor.hpp:31-41).  DFMA on the CUDA cores does that
// at ~14 TFLOP/s (gemm_f64acc.cu).  Here the same product runs on the
// 5th-generation tensor cores in exact integer arithmetic:
//
//  * every row of A is scaled by a power of two 2^ea[m] so its largest
//    element lies in [2^(b-1), 2^b), and rounded to an integer A' (exact for
//    every element within b - 24 binades of the row maximum, else an error of
//    at most 2^-b of it); every column of B likewise (2^eb[n], B');
//  * the integer product X = A'.B' (|X| <= K 2^2b) is computed modulo n
//    pairwise-coprime moduli m_i <= 256 (kModuli): one int8 GEMM per modulus
//    on the symmetric residues of A' and B' (|r| <= 128), accumulated EXACTLY
//    in int32 TMEM (tcgen05.mma kind::i8; K 2^14 < 2^31);
//  * X is rebuilt from its residues by Garner's algorithm -- mixed-radix
//    digits v_i, computed tile by tile as the residues arrive (v_i needs
//    v_0..v_{i-1}, kept as int8 in a per-CTA scratch): v_i = (r_i - sum_j v_j
//    (W_j mod m_i)) (W_i^-1 mod m_i) mod m_i, the sum exact in int32 with
//    four digits per dp4a, the two reductions in exact fp32 -- and Horner in
//    fp64 from the top digit (X = v_0 + m_0 (v_1 + m_1 (...))), then scaled
//    by 2^-(ea+eb) and rounded once to fp32: the reference's "fp64
//    accumulate, cast".  (The sequential form, u dependent fp32 steps per
//    digit, left the tensor pipe idle ~25% of the time at 14 moduli.)
//
// b is the largest integer with K 2^2b < M/4 (M = prod m_i), so the symmetric
// CRT range holds X with margin: with the default 14 moduli (110 bits) b = 47
// at K <= 16384, an input error of 2^-47 of the row/column maximum per
// operand -- the grade of the reference's own fp64 accumulation over
// K ~ 10^4 terms (any fp64 order reproduced every plan).
// The previous form of this kernel (Ozaki scheme I: 7 int8 digits per
// operand, 28 digit-pair GEMMs) had the same grade at twice the tensor work.
//
// Kernel structure = gemm_tc.cu's (persistent, warp-specialised, TMA ring,
// double-buffered TMEM accumulators, 128 x 256 tiles), with a work unit =
// (tile, modulus) and eight epilogue warps doing the Garner steps.
#include <cmath>
#include <cstring>

#include "engine.hpp"
#include "tc_common.cuh"

namespace keep_b200 {

namespace {

using namespace tc;

constexpr int OBM = 128, OBN = 256, OBK = 128;  // OBK bytes = int8 elements per stage
constexpr int OSTAGES = 4;
constexpr int OEPI = 8;                         // epilogue warps (2 per TMEM lane quarter)
constexpr int OTHREADS = (4 + OEPI) * 32;
constexpr int OGM = 16;
constexpr int kMaxModuli = 16;
constexpr uint32_t OA_BYTES = OBM * OBK, OB_BYTES = OBN * OBK, OSTAGE = OA_BYTES + OB_BYTES;
constexpr size_t OSMEM = size_t(OSTAGES) * OSTAGE + 1024 + 256;
// pairwise coprime, descending from 256 (greedy)
constexpr int kModuliAll[kMaxModuli] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};

// the modulus tables (kernel parameter: constant bank)
struct OzCrt {
    int n;                      // moduli used
    int gm;                     // tile raster: bands of gm row tiles (KEEP_OZ_GM, default OGM)
    int mi[kMaxModuli];         // m_i
    float mf[kMaxModuli];       // m_i
    float rcp[kMaxModuli];      // 1 / m_i (fp32)
    double md[kMaxModuli];      // m_i
    double rcpd[kMaxModuli];    // 1 / m_i (fp64)
    int dpk[kMaxModuli][kMaxModuli / 4];  // byte k of dpk[u][g] = W_{4g+k} mod m_u, symmetric (0 for 4g+k >= u)
    int dcorr[kMaxModuli];              // 128 sum_j (W_j mod m_u): the digits' +128 bias through the dot product
    float winv[kMaxModuli];             // W_u^-1 mod m_u (symmetric), W_u = m_0 ... m_{u-1}
};

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

// ---- CTA-pair (cta_group::2) primitives: a 256 x 256 tile over two SMs of a
// TPC.  Each CTA stages its 128 rows of A and 128 of the 256 rows of B; the
// leader (cluster rank 0) issues one M = 256 MMA over both CTAs' smem, each CTA
// holding its 128 accumulator rows in its own TMEM.  Per k-step an SM reads
// 32 KB instead of 48 KB (ncu: the single-CTA kernel's TMA stream was
// ~15 TB/s across the chip at 63% tensor-pipe activity).
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_rank0(uint32_t saddr) {  // the leader's copy of a smem address
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's smem, completing bytes on the LEADER's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* tm, uint32_t bar_leader, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar_leader), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
// MMA completion -> the mbarrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}
constexpr int OSTAGES2 = 6;                            // pair: 32 KB stages
constexpr uint32_t OB2_BYTES = 128 * OBK, OSTAGE2 = OA_BYTES + OB2_BYTES;
constexpr size_t OSMEM2 = size_t(OSTAGES2) * OSTAGE2 + 1024 + 256;

__device__ __forceinline__ void otile_coords(int t, int tiles_m, int tiles_n, int ogm, int& mb, int& nb) {
    const int band = t / (ogm * tiles_n);
    const int m0 = band * ogm;
    const int gm = min(ogm, tiles_m - m0);
    const int r = t - band * ogm * tiles_n;
    mb = m0 + r % gm;
    nb = r / gm;
}

__device__ __forceinline__ void epi_store32(const EpiArgs& e, int m, int n, const float (&v)[32]) {
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
}

// Small exact integer arithmetic in fp32 without the conversion pipe:
// rounding to an integer by the 1.5 * 2^23 magic constant (round to nearest
// even, exact for |x| < 2^22), digits stored biased by 128 and widened with a
// byte permute into the mantissa of 2^23.
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr float kByteBias = 8388736.0f;  // 2^23 + 128

// x - m rint(x / m) for an exactly representable fp32 integer x (|x| < 2^22):
// the symmetric residue (canonical for odd m; +-m/2 both possible for even m)
__device__ __forceinline__ float redm(float x, float m, float rc) {
    const float q = fmaf(x, rc, kMagic) - kMagic;
    return fmaf(-q, m, x);
}

// sum of the four products of the unsigned bytes of a and the signed bytes of b, plus c
__device__ __forceinline__ int dp4a_us(uint32_t a, int b, int c) {
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// byte b of w (a digit v + 128) -> 2^23 + 128 + v as fp32
__device__ __forceinline__ float byte_biased(uint32_t w, int b) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, uint32_t(b) | 0x7650u));
}
template <bool PAIR>
__global__ void __launch_bounds__(OTHREADS, 1)
gemm_oz_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
               int Mp, int Np, const __grid_constant__ OzCrt crt, const int* __restrict__ ea,
               const int* __restrict__ eb, uint32_t* __restrict__ scratch, EpiArgs epi) {
    constexpr int NST = PAIR ? OSTAGES2 : OSTAGES;
    constexpr uint32_t STAGE = PAIR ? OSTAGE2 : OSTAGE;
    constexpr int TM = PAIR ? 2 * OBM : OBM;  // tile rows (over the pair)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = PAIR ? int(cluster_rank()) : 0;
    const int cid = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);      // cluster (tile walker) index
    const int ncl = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
    const int tiles_m = int(ceil_div(M, TM)), tiles_n = int(ceil_div(N, OBN));
    const int ntiles = tiles_m * tiles_n;
    const int kblocks = int(ceil_div(K, OBK));
    const int U = crt.n;

    if (warp == 0 && lane == 0) {
        prefetch_map(&tmA);
        prefetch_map(&tmB);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], PAIR ? 2 * OEPI : OEPI);  // pair: both CTAs' epilogues free the leader's buffer
        }
        fence_barrier_init();
    }
    if constexpr (PAIR) cluster_sync_all();  // barriers initialised in both CTAs before any remote use
    if (warp == 2) {
        if constexpr (PAIR) tmem_alloc_pair(tmem_slot, 512);
        else tmem_alloc(tmem_slot, 512);
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer: residue planes u of A and B
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                int mb, nb;
                otile_coords(t, tiles_m, tiles_n, crt.gm, mb, nb);
                for (int u = 0; u < U; ++u) {
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * STAGE;
                        if constexpr (PAIR) {
                            // both CTAs' bytes complete on the leader's barrier
                            const uint32_t fl = map_to_rank0(smem_u32(&full[stage]));
                            if (rank == 0) mbar_expect_tx(&full[stage], 2 * STAGE);
                            tma_load_2d_pair(sa, &tmA, fl, kb * OBK, u * Mp + mb * TM + rank * OBM);
                            tma_load_2d_pair(sa + OA_BYTES, &tmB, fl, kb * OBK, u * Np + nb * OBN + rank * (OBN / 2));
                        } else {
                            mbar_expect_tx(&full[stage], STAGE);
                            tma_load_2d(sa, &tmA, &full[stage], kb * OBK, u * Mp + mb * OBM);
                            tma_load_2d(sa + OA_BYTES, &tmB, &full[stage], kb * OBK, u * Np + nb * OBN);
                        }
                        if (++stage == NST) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer: one exact int32 GEMM per modulus
        if (!PAIR || rank == 0) {
            constexpr uint32_t idesc = idesc_i8(TM, OBN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                for (int u = 0; u < U; ++u, ++it) {
                    const int acc = it & 1;
                    mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                    fence_after();
                    const uint32_t tmem_d = tmem_base + uint32_t(acc * OBN);
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&full[stage], phase);
                        fence_after();
                        const uint32_t sa = smem_u32(smem + stage * STAGE);
                        const uint64_t ad = smem_desc(sa), bd = smem_desc(sa + OA_BYTES);
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < OBK / 32; ++k) {  // 32 int8 = 32 bytes per MMA
                                if constexpr (PAIR)
                                    umma_i8_pair(tmem_d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                                 (kb == 0 && k == 0) ? 0u : 1u);
                                else
                                    umma_i8(tmem_d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                            (kb == 0 && k == 0) ? 0u : 1u);
                            }
                            if constexpr (PAIR) umma_commit_pair(&empty[stage]);
                            else umma_commit(&empty[stage]);
                        }
                        __syncwarp();
                        if (++stage == NST) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    if (elect_one()) {
                        if constexpr (PAIR) umma_commit_pair(&tfull[acc]);
                        else umma_commit(&tfull[acc]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue: Garner digits, fp64 Horner on the last modulus
        const int q4 = warp & 3;                 // TMEM lane quarter
        const int ch0 = ((warp - 4) >> 2) * (OBN / 32 / 2);  // this warp's four 32-column chunks
        const int r = q4 * 32 + lane;            // tile row = TMEM lane
        // digits v_j of this CTA's tile: [j][OBN / 4 column quads][OBM rows] x char4
        uint32_t* vs = scratch + size_t(blockIdx.x) * kMaxModuli * (OBN / 4) * OBM + r;
        const uint32_t tempty_leader0 = PAIR ? map_to_rank0(smem_u32(&tempty[0])) : 0u;
        int it = 0;
        for (int t = cid; t < ntiles; t += ncl) {
            int mb, nb;
            otile_coords(t, tiles_m, tiles_n, crt.gm, mb, nb);
            const int m = mb * TM + rank * OBM + r;
            const bool mok = m < M;
            const int eam = mok ? ea[m] : 0;
            for (int u = 0; u < U; ++u, ++it) {
                const bool last = u == U - 1;
                const int acc = it & 1;
                const float mf = crt.mf[u], rc = crt.rcp[u];
                const int mi = crt.mi[u];
                mbar_wait(&tfull[acc], (it >> 1) & 1);
                fence_after();
#pragma unroll 1
                for (int ch = ch0; ch < ch0 + OBN / 32 / 2; ++ch) {
                    uint32_t d[32];
                    tmem_ld32(tmem_base + (uint32_t(q4 * 32) << 16) + uint32_t(acc * OBN + ch * 32), d);
                    const int n0 = nb * OBN + ch * 32;
                    if (n0 >= N) continue;
                    float tv[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        // |acc| <= K 2^14 < 2^28: the fp32 quotient is within one of exact
                        const int a = int(d[j]);
                        const int q = __float_as_int(fmaf(float(a), rc, kMagic)) - __float_as_int(kMagic);
                        const int rr = a - q * mi;  // |rr| < 2m
                        tv[j] = redm(__int_as_float(0x4B400000 + rr) - kMagic, mf, rc);
                    }
                    if (u == 0) {  // m_0 = 256 is even: +128 -> -128
#pragma unroll
                        for (int j = 0; j < 32; ++j) tv[j] = tv[j] >= 0.5f * mf ? tv[j] - mf : tv[j];
                    }
                    uint32_t* vq = vs + size_t(ch * 8) * OBM;
                    auto ld8 = [&](uint32_t(&w)[8], int jm) {
#pragma unroll
                        for (int g = 0; g < 8; ++g) w[g] = vq[(size_t(jm) * (OBN / 4) + g) * OBM];
                    };
                    // Garner as one dot product: with W_j = m_0 ... m_{j-1},
                    //   v_u = (r_u - sum_{j<u} v_j (W_j mod m_u)) (W_u^-1 mod m_u)  mod m_u,
                    // the sum exact in int32: four digits per dp4a (the stored digits are v + 128, unsigned;
                    // the constants W_j mod m_u symmetric, signed; crt.dcorr[u] removes the bias), after a
                    // 4 x 4 byte transpose of four digit words (digit-major, 4 columns each) into four
                    // column words (4 digits each).  Two fp32 reductions per element instead of u
                    // dependent steps.
                    if (u > 0) {
                        const int G = (u + 3) >> 2;  // digit groups 4g .. 4g+3 holding v_0 .. v_{u-1}
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf) {  // 16 columns = 4 column quads at a time
                            uint32_t wd[kMaxModuli][4];
#pragma unroll
                            for (int j = 0; j < kMaxModuli; ++j)
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    wd[j][q] = (j < u) ? vq[(size_t(j) * (OBN / 4) + hf * 4 + q) * OBM] : 0u;
                            int s[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j) s[j] = -crt.dcorr[u];
#pragma unroll
                            for (int g = 0; g < kMaxModuli / 4; ++g)
                                if (g < G) {
                                    const int dk = crt.dpk[u][g];
#pragma unroll
                                    for (int q = 0; q < 4; ++q) {
                                        const uint32_t a = wd[4 * g][q], b = wd[4 * g + 1][q], c = wd[4 * g + 2][q],
                                                       e = wd[4 * g + 3][q];
                                        const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
                                        const uint32_t t2 = __byte_perm(c, e, 0x5140), t3 = __byte_perm(c, e, 0x7362);
                                        s[4 * q] = dp4a_us(__byte_perm(t0, t2, 0x5410), dk, s[4 * q]);
                                        s[4 * q + 1] = dp4a_us(__byte_perm(t0, t2, 0x7632), dk, s[4 * q + 1]);
                                        s[4 * q + 2] = dp4a_us(__byte_perm(t1, t3, 0x5410), dk, s[4 * q + 2]);
                                        s[4 * q + 3] = dp4a_us(__byte_perm(t1, t3, 0x7632), dk, s[4 * q + 3]);
                                    }
                                }
                            const float wi = crt.winv[u];
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                float& x = tv[hf * 16 + j];  // |r_u - s| < 2^19: redm stays canonical (odd m_u)
                                x = redm(redm(x - float(s[j]), mf, rc) * wi, mf, rc);
                            }
                        }
                    }
                    uint32_t w0[8], w1[8], w2[8];
                    if (!last) {
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            uint32_t b[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) b[k] = uint32_t(__float_as_int(tv[4 * g + k] + kByteBias)) & 0xffu;
                            vq[(size_t(u) * (OBN / 4) + g) * OBM] = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
                        }
                    } else if (mok) {
                        // X = v_0 + m_0 (v_1 + m_1 (... + m_{U-2} v_{U-1})), exact while |partial| < 2^53
                        double P[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) P[j] = double(tv[j]);
                        auto hstep = [&](const uint32_t(&w)[8], int jm) {
                            const double mdj = crt.md[jm];
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                P[j] = fma(P[j], mdj,
                                           __hiloint2double(0x43300000, __byte_perm(w[j >> 2], 0u, uint32_t(j & 3) | 0x4440u)) -
                                               4503599627370624.0);  // (2^52 + 128 + v) - (2^52 + 128)
                        };
                        // digits u-1 .. 0, two ahead
                        if (u > 0) ld8(w0, u - 1);
                        if (u > 1) ld8(w1, u - 2);
#pragma unroll 1
                        for (int k = 0; k < u; k += 3) {
                            if (k + 2 < u) ld8(w2, u - 3 - k);
                            hstep(w0, u - 1 - k);
                            if (k + 1 >= u) break;
                            if (k + 3 < u) ld8(w0, u - 4 - k);
                            hstep(w1, u - 2 - k);
                            if (k + 2 >= u) break;
                            if (k + 4 < u) ld8(w1, u - 5 - k);
                            hstep(w2, u - 3 - k);
                        }
                        float v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int n = n0 + j;
                            const int e = eam + (n < N ? eb[n] : 0);  // |e| < 1000: 2^-e is a normal double
                            v[j] = float(P[j] * __longlong_as_double(int64_t(1023 - e) << 52));
                        }
                        epi_store32(epi, m, n0, v);
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR) mbar_arrive_cluster(tempty_leader0 + uint32_t(acc * sizeof(uint64_t)));
                    else mbar_arrive(&tempty[acc]);
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync_all();  // the peer's TMEM is the leader's MMA target until the end
    if (warp == 2) {
        fence_after();
        if constexpr (PAIR) tmem_dealloc_pair(tmem_base, 512);
        else tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------- splits --
// x 2^e with max |x| 2^e in [2^(b-1), 2^b): e = b - exponent(max) (frexp).
__device__ __forceinline__ int scale_exp(float amax, int bits) {
    if (!(amax > 0.f)) return 0;
    int ex;
    frexpf(amax, &ex);
    return bits - ex;
}

// X = rint(x 2^e) (|X| < 2^51) held as b = 1.5 * 2^52 + X: b - 1.5 * 2^52 is X
// exactly, and the low word of b is X mod 2^32 (b's mantissa is 2^51 + X)
struct OzInt {
    double b;
};
constexpr double kM52 = 6755399441055744.0;  // 1.5 * 2^52
__device__ __forceinline__ OzInt oz_int(float x, double pw) {
    return {fma(double(x), pw, kM52)};  // x 2^e is exact: one rounding, to nearest even
}

// symmetric residue of X modulo m_i: q = rint(X / m) from one fma against the
// 1.5 * 2^52 magic constant (X * (1/m) is within 2^-13 of X / m, which is at
// least 1/(2m) from a half-integer for odd m, so the residue is canonical),
// read as q mod 2^32 from its low word; then r = X - q m in wrapping int32
// arithmetic (|r| < m).  m_0 = 256: the low byte of X (+128 -> -128).
__device__ __forceinline__ uint32_t residue_word(const OzInt& X, const OzCrt& c, int i) {  // residue in the low byte
    const int lo = __double2loint(X.b);
    if (i == 0) return uint32_t(lo);
    const int q = __double2loint(fma(X.b - kM52, c.rcpd[i], kM52));
    return uint32_t(lo - q * c.mi[i]);
}

// A rows -> out[i][m][0..Kp) int8 residues of A' = rint(A 2^ea) + ea[m]; one warp per row.
__global__ void oz_split_rows_kernel(const float* __restrict__ A, int64_t lda, int M, int K, int Kp, int bits,
                                     int Mp, const __grid_constant__ OzCrt crt, int8_t* __restrict__ out,
                                     int* __restrict__ ea) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= M) return;
    const float* a = A + int64_t(warp) * lda;
    float mx = 0.f;
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(a[k]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int e = scale_exp(mx, bits);
    if (lane == 0) ea[warp] = e;
    const double pw = ldexp(1.0, e);
    const size_t plane = size_t(Mp) * Kp;
    int8_t* o = out + size_t(warp) * Kp;
    for (int k0 = lane * 4; k0 < Kp; k0 += 128) {
        OzInt X[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) X[q] = oz_int((k0 + q < K) ? a[k0 + q] : 0.f, pw);
        for (int i = 0; i < crt.n; ++i) {
            const uint32_t p01 = __byte_perm(residue_word(X[0], crt, i), residue_word(X[1], crt, i), 0x0040);
            const uint32_t p23 = __byte_perm(residue_word(X[2], crt, i), residue_word(X[3], crt, i), 0x0040);
            *reinterpret_cast<uint32_t*>(o + i * plane + k0) = __byte_perm(p01, p23, 0x5410);
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

// B [K x N] row-major -> out[i][n][0..Kp) int8 residues of B' = rint(B 2^eb)
// (transposed, K-major) + eb[n].  Tile 128 k x 32 n through shared memory,
// eight moduli at a time; a thread holds 4 consecutive k of its column (4
// groups), so one modulus' residues leave as four 4-byte smem stores.
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const float* __restrict__ B, int64_t ldb, int K, int N,
                                                            int Kp, int bits, int Np,
                                                            const __grid_constant__ OzCrt crt,
                                                            const unsigned* __restrict__ cmax,
                                                            int8_t* __restrict__ out, int* __restrict__ eb) {
    __shared__ __align__(16) int8_t sd[8][32][128 + 16];
    const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 128;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
    const int n = n0 + tx;
    const int e = n < N ? scale_exp(__uint_as_float(cmax[n]), bits) : 0;
    if (blockIdx.y == 0 && ty == 0 && n < N) eb[n] = e;
    const double pw = ldexp(1.0, e);
    OzInt X[16];  // [g][j]: k = k0 + 32 g + 4 ty + j
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int k = k0 + 32 * (q >> 2) + 4 * ty + (q & 3);
        X[q] = oz_int((k < K && n < N) ? B[int64_t(k) * ldb + n] : 0.f, pw);
    }
    const size_t plane = size_t(Np) * Kp;
    for (int g0 = 0; g0 < crt.n; g0 += 8) {
        const int gn = min(8, crt.n - g0);
        for (int i = 0; i < gn; ++i) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    OzInt x = X[4 * g + j];
                    asm("" : "+d"(x.b));  // recomputed per modulus, not hoisted into more registers
                    w[j] = residue_word(x, crt, g0 + i);
                }
                *reinterpret_cast<uint32_t*>(&sd[i][tx][32 * g + 4 * ty]) =
                    __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
            }
        }
        __syncthreads();
        // write rows (i, n): 128 contiguous bytes = 8 x 16 B
        for (int idx = threadIdx.x; idx < gn * 32 * 8; idx += 256) {
            const int i = idx / 256, rem = idx % 256, nn = rem / 8, c = rem % 8;
            if (n0 + nn >= N || k0 + c * 16 >= Kp) continue;
            const int4 v = *reinterpret_cast<const int4*>(&sd[i][nn][c * 16]);
            *reinterpret_cast<int4*>(out + (g0 + i) * plane + size_t(n0 + nn) * Kp + k0 + c * 16) = v;
        }
        __syncthreads();
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

int mod_inverse(int a, int m) {
    a %= m;
    for (int x = 1; x < m; ++x)
        if ((a * x) % m == 1) return x;
    raise(KEEP_ERR_CONFIG, "Ozaki GEMM: moduli are not coprime");
    return 0;
}

const OzCrt& crt_tables() {
    static const OzCrt c = [] {
        OzCrt t{};
        t.n = oz_moduli();
        const char* g = std::getenv("KEEP_OZ_GM");
        t.gm = g ? std::max(1, std::atoi(g)) : OGM;
        for (int i = 0; i < t.n; ++i) {
            t.mi[i] = kModuliAll[i];
            t.mf[i] = float(kModuliAll[i]);
            t.rcp[i] = 1.f / float(kModuliAll[i]);
            t.md[i] = double(kModuliAll[i]);
            t.rcpd[i] = 1.0 / double(kModuliAll[i]);
            // W_j mod m_i (j < i) and W_i^-1 mod m_i, as symmetric residues
            const int mi = kModuliAll[i];
            auto sym = [mi](long long a) {
                const int r = int(((a % mi) + mi) % mi);
                return r > mi / 2 ? r - mi : r;
            };
            long long w = 1;
            for (int j = 0; j < i; ++j) {
                const int dj = sym(w);
                t.dpk[i][j / 4] = int(uint32_t(t.dpk[i][j / 4]) | ((uint32_t(dj) & 0xffu) << (8 * (j % 4))));
                t.dcorr[i] += 128 * dj;
                w = (w * kModuliAll[j]) % mi;
            }
            t.winv[i] = i == 0 ? 1.f : float(sym(mod_inverse(int(w), mi)));
        }
        return t;
    }();
    return c;
}

}  // namespace

int oz_moduli() {
    static const int s = [] {
        const char* e = std::getenv("KEEP_OZ_MODULI");
        const int v = e ? std::atoi(e) : 14;
        return std::min(kMaxModuli, std::max(8, v));
    }();
    return s;
}

int oz_bits(int K) {
    double lm = 0.0;
    for (int i = 0; i < oz_moduli(); ++i) lm += std::log2(double(kModuliAll[i]));
    // K 2^2b <= M / 4: the symmetric range (-M/2, M/2) holds every product sum
    // with a margin for the non-canonical top digit
    return int(std::floor((lm - 2.0 - std::log2(double(std::max(K, 1)))) / 2.0));
}

// KEEP_OZ_PAIR=0: the single-CTA kernel only (A/B knob)
bool oz_pair_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KEEP_OZ_PAIR");
        return !(e && *e == '0');
    }();
    return on;
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
    return K % 16 == 0 && N % 32 == 0 && K <= (1 << 17) &&
           (parity_gemm_mode() == 1 || (parity_gemm_mode() == 0 && M >= kOzMinRows));
}

void launch_gemm_ozaki(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                       const EpiArgs& epi, cudaStream_t st, OzWork& w, int max_ctas) {
    if (M == 0 || N == 0) return;
    const OzCrt& crt = crt_tables();
    const int s = crt.n;
    const int bits = oz_bits(K);
    if (bits < 30) raise(KEEP_ERR_CONFIG, "Ozaki GEMM: too few moduli for K = " + std::to_string(K));
    // CTA pairs when the 256-row tiles still fill the machine
    const int ntiles2 = int(ceil_div(M, 2 * OBM) * ceil_div(N, OBN));
    const int maxc = std::max(1, std::min(max_ctas, kNumSMs));
    const bool pair = oz_pair_enabled() && maxc >= 2 && 2 * ntiles2 >= maxc;
    const int Mp = int(ceil_div(M, 2 * OBM) * 2 * OBM), Np = int(ceil_div(N, OBN) * OBN);
    const int Kp = int(ceil_div(K, 16) * 16);
    w.a.ensure(size_t(s) * Mp * Kp);
    w.b.ensure(size_t(s) * Np * Kp);
    w.ea.ensure(sizeof(int) * size_t(Mp));
    w.eb.ensure(sizeof(int) * size_t(Np) + sizeof(unsigned) * size_t(N));
    int* eb = w.eb.as<int>();
    unsigned* cmax = reinterpret_cast<unsigned*>(eb + Np);
    // residues of A (rows) and B (columns)
    oz_split_rows_kernel<<<unsigned(ceil_div(M, 8)), 256, 0, st>>>(A, lda, M, K, Kp, bits, Mp, crt,
                                                                    w.a.as<int8_t>(), w.ea.as<int>());
    KEEP_LAUNCH_CHECK();
    KEEP_CUDA(cudaMemsetAsync(cmax, 0, sizeof(unsigned) * size_t(N), st));
    const int ksplit = int(std::min<int64_t>(64, ceil_div(K, 64)));
    const int krows = int(ceil_div(K, ksplit));
    oz_colmax_kernel<<<dim3(unsigned(ceil_div(N, 256)), unsigned(ksplit)), 256, 0, st>>>(B, ldb, K, N, krows, cmax);
    KEEP_LAUNCH_CHECK();
    oz_split_cols_kernel<<<dim3(unsigned(ceil_div(N, 32)), unsigned(ceil_div(Kp, 128))), 256, 0, st>>>(
        B, ldb, K, N, Kp, bits, Np, crt, cmax, w.b.as<int8_t>(), eb);
    KEEP_LAUNCH_CHECK();
    // the GEMM
    const CUtensorMap ta = make_map_i8(w.a.p, int64_t(s) * Mp, K, Kp, OBM);
    if (pair) {
        const CUtensorMap tb = make_map_i8(w.b.p, int64_t(s) * Np, K, Kp, OBN / 2);
        const int grid = std::min(2 * ntiles2, maxc & ~1);
        w.part.ensure(sizeof(uint32_t) * size_t(grid) * kMaxModuli * (OBN / 4) * OBM);
        smem_attr(gemm_oz_kernel<true>, int(OSMEM2));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(OTHREADS);
        cfg.dynamicSmemBytes = OSMEM2;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        KEEP_CUDA(cudaLaunchKernelEx(&cfg, gemm_oz_kernel<true>, ta, tb, M, N, K, Mp, Np, crt, w.ea.as<int>(),
                                     static_cast<const int*>(eb), w.part.as<uint32_t>(), epi));
        KEEP_LAUNCH_CHECK();
        return;
    }
    smem_attr(gemm_oz_kernel<false>, int(OSMEM));
    const CUtensorMap tb = make_map_i8(w.b.p, int64_t(s) * Np, K, Kp, OBN);
    const int ntiles = int(ceil_div(M, OBM) * ceil_div(N, OBN));
    const int grid = std::min(ntiles, maxc);
    w.part.ensure(sizeof(uint32_t) * size_t(grid) * kMaxModuli * (OBN / 4) * OBM);
    gemm_oz_kernel<false><<<grid, OTHREADS, OSMEM, st>>>(ta, tb, M, N, K, Mp, Np, crt, w.ea.as<int>(), eb,
                                                         w.part.as<uint32_t>(), epi);
    KEEP_LAUNCH_CHECK();
}

void launch_gemm_parity(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                        const EpiArgs& epi, cudaStream_t st, OzWork& w, bool exact, int max_ctas) {
    if (!exact && ozaki_eligible(M, N, K) && (epi.kind != EPI_QKV || epi.d % 32 == 0)) launch_gemm_ozaki(A, lda, B, ldb, M, N, K, epi, st, w, max_ctas);
    else launch_gemm_f64acc(A, lda, B, ldb, M, N, K, epi, st, exact);
}

}  // namespace keep_b200

// Test hook: C = A . B on device pointers (fp32 [M x K] . [K x N] -> fp32),
// mode 0 auto, 1 Ozaki, 2 DFMA one k chain per output (PARITY_EXACT: vec_mat's
// order), 3 DFMA with the few-row split-K (PARITY).
extern "C" int keep_debug_gemm_parity(const float* A, const float* B, float* Cout, int M, int N, int K, int mode) {
    try {
        keep_b200::EpiArgs e{keep_b200::EPI_STORE, 0, Cout, N, nullptr, nullptr, nullptr, nullptr};
        thread_local keep_b200::OzWork w;
        if (mode == 1 || (mode == 0 && keep_b200::ozaki_eligible(M, N, K)))
            keep_b200::launch_gemm_ozaki(A, K, B, N, M, N, K, e, 0, w, keep_b200::kNumSMs);
        else
            keep_b200::launch_gemm_f64acc(A, K, B, N, M, N, K, e, 0, mode == 2);
        return cudaDeviceSynchronize() == cudaSuccess ? 0 : KEEP_ERR_CUDA;
    } catch (const keep_b200::KeepError& e) {
        return e.code;
    }
}
