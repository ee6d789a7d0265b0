// gemm_tc.cu -- FAST-mode projection GEMM on the 5th-generation tensor cores.
//
//   C[M x N] = A[M x K] . Bt[N x K]^T      bf16 operands, fp32 accumulation
//
// A = compact activations (row-major, K-major), Bt = transposed weights
// (K-major rows).  One persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer   (one elected lane; cp.async.bulk.tensor into a
//                               STAGES-deep ring of 128B-swizzled tiles)
//   warp 1      MMA issuer     (one lane; tcgen05.mma.cta_group::1.kind::f16,
//                               128 x BN x 16 per instruction, accumulators in
//                               TMEM, double buffered so the epilogue of tile
//                               i overlaps the main loop of tile i+1)
//   warp 2      TMEM allocator
//   warps 4..7  epilogue       (tcgen05.ld 32x32b -> registers -> fused op)
// Fused epilogues: QKV split with K/V rows scattered into
// the merged KV cache at their global row (gathered recompute), fp32 residual
// add with a bf16 mirror for the next GEMM, ReLU to bf16, plain fp32 store.
// Tiles are rasterised in bands of GM m-blocks so a band of A and a window of
// weight columns stay L2-resident (126 MB) while 148 CTAs sweep them.
#include <map>
#include <mutex>
#include <unordered_map>

#include "engine.hpp"
#include "tc_common.cuh"

namespace keep_b200 {

namespace tc {
// ------------------------------------------------------------ tensor maps --
EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            raise(KEEP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

// 2-D bf16 tensor [rows x cols] (row stride ld elements), box BK x box_rows,
// 128-byte swizzle; out-of-bounds rows read as zero.
CUtensorMap make_map_bf16(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    // memoised: a map is a pure function of its arguments, and the engine
    // re-uses the same weight / workspace buffers every layer and every prefill
    struct Key {
        const void* p;
        int64_t r, c, ld;
        int b;
        bool operator==(const Key& o) const { return p == o.p && r == o.r && c == o.c && ld == o.ld && b == o.b; }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            return std::hash<const void*>()(k.p) ^ (size_t(k.r) * 0x9e3779b97f4a7c15ull) ^ (size_t(k.c) << 17) ^
                   (size_t(k.ld) << 7) ^ size_t(k.b);
        }
    };
    thread_local std::unordered_map<Key, CUtensorMap, Hash> memo;
    const Key key{ptr, rows, cols, ld, box_rows};
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    if (memo.size() > 8192) memo.clear();
    CUtensorMap tm;
    const cuuint64_t gdim[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t gstride[1] = {cuuint64_t(ld * 2)};
    const cuuint32_t box[2] = {cuuint32_t(64), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstride, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(KEEP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    memo.emplace(key, tm);
    return tm;
}

}  // namespace tc

namespace {

constexpr int BM = 128, BK = 64, UMMA_K = 16, GM = 16;
constexpr int kThreads = 256;

using namespace tc;

// Store 32 consecutive values of one row starting at column n.
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
    uint4* o = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        o[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                          pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}

__device__ __forceinline__ void epilogue_chunk(const EpiArgs& e, int m, int n, float (&v)[32]) {
    switch (e.kind) {
        case EPI_QKV: {
            const int d = e.d;
            if (n < d) {
                if (e.q_scale != 1.f) {
#pragma unroll
                    for (int q = 0; q < 32; ++q) v[q] *= e.q_scale;
                }
                store_bf16x32(e.out_bf16 + int64_t(m) * d + n, v);
            } else if (n < 2 * d) {
                store_bf16x32(static_cast<__nv_bfloat16*>(e.kdst) + int64_t(e.rows[m]) * d + (n - d), v);
            } else {
                store_bf16x32(static_cast<__nv_bfloat16*>(e.vdst) + int64_t(e.rows[m]) * d + (n - 2 * d), v);
            }
            break;
        }
        case EPI_RESID: {
            float4* x = reinterpret_cast<float4*>(e.out + int64_t(m) * e.ldo + n);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float4 t = x[q];
                t.x += v[4 * q + 0];
                t.y += v[4 * q + 1];
                t.z += v[4 * q + 2];
                t.w += v[4 * q + 3];
                x[q] = t;
                v[4 * q + 0] = t.x;
                v[4 * q + 1] = t.y;
                v[4 * q + 2] = t.z;
                v[4 * q + 3] = t.w;
            }
            if (e.out_bf16) store_bf16x32(e.out_bf16 + int64_t(m) * e.ldo + n, v);
            break;
        }
        case EPI_RELU: {
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = v[q] < 0.f ? 0.f : v[q];
            store_bf16x32(e.out_bf16 + int64_t(m) * e.ldo + n, v);
            break;
        }
        default: {
            float4* o = reinterpret_cast<float4*>(e.out + int64_t(m) * e.ldo + n);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
    }
}

// AR = rows of A staged per k-block.  Small-M GEMMs (the deep layers, where
// only the query rows are recomputed) stage just AR = 32 rows: the M = 128
// MMA reads the rest of its A window from whatever follows in shared memory
// (those accumulator rows are never stored), so the weight stream -- the
// whole cost at small M -- runs through a deep ring of small stages.
template <int BN, int AR = BM>
struct Cfg {
    static constexpr uint32_t A_BYTES = AR * BK * 2;
    static constexpr uint32_t B_BYTES = BN * BK * 2;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = AR < BM ? int((192u * 1024u) / STAGE_BYTES) : (BN == 256 ? 4 : 8);
    static constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    // (+16 KB: the M = 128 window of the last stage's A must stay in bounds)
    static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + (AR < BM ? BM * BK * 2 : 0) + 1024 + 256;
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
    const int band = t / (GM * tiles_n);
    const int m0 = band * GM;
    const int gm = min(GM, tiles_m - m0);
    const int r = t - band * GM * tiles_n;
    mb = m0 + r % gm;
    nb = r / gm;
}

template <int BN, int AR>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
               EpiArgs epi, int ksplit, float* __restrict__ acc_out) {
    using CF = Cfg<BN, AR>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared space
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::STAGES * CF::STAGE_BYTES + (AR < BM ? BM * BK * 2 : 0));
    uint64_t* empty = full + CF::STAGES;
    uint64_t* tfull = empty + CF::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_m = int(ceil_div(M, BM)), tiles_n = int(ceil_div(N, BN));
    // split-K (small M): work unit t = (tile, k-slice); the slices' partial
    // sums meet in acc_out through fp32 reductions, finalised by a separate pass
    const int ntiles = tiles_m * tiles_n * ksplit, kblocks_all = K / BK;
    const int kper = int(ceil_div(kblocks_all, ksplit));

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        for (int s = 0; s < CF::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(CF::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
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
                const int ks = t % ksplit;
                tile_coords(t / ksplit, tiles_m, tiles_n, mb, nb);
                const int kb0 = ks * kper, kb1 = min(kblocks_all, kb0 + kper);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * CF::STAGE_BYTES;
                    mbar_expect_tx(&full[stage], CF::STAGE_BYTES);
                    tma_load_2d(sa, &tmA, &full[stage], kb * BK, mb * BM);
                    tma_load_2d(sa + CF::A_BYTES, &tmB, &full[stage], kb * BK, nb * BN);
                    if (++stage == CF::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // ---------------- MMA issuer: the warp walks the schedule, one elected lane issues
            constexpr uint32_t idesc = instr_desc(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait(&tempty[acc], aphase ^ 1);  // epilogue drained this accumulator
                fence_after();
                const uint32_t tmem_d = tmem_base + uint32_t(acc * BN);
                const int ks = t % ksplit;
                const int kb0 = ks * kper, kb1 = min(kblocks_all, kb0 + kper);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    const uint32_t sa = smem_u32(smem + stage * CF::STAGE_BYTES);
                    const uint64_t ad = smem_desc(sa), bd = smem_desc(sa + CF::A_BYTES);
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < BK / UMMA_K; ++k) {
                            // advance 16 bf16 = 32 bytes along K inside the swizzle atom
                            umma(tmem_d, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb > kb0 || k) ? 1u : 0u);
                        }
                        umma_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
                    }
                    __syncwarp();
                    if (++stage == CF::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (elect_one()) umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
                __syncwarp();
            }
        }
    } else if (warp >= 4) {  // ---------------- epilogue warps
        const int q = warp & 3;  // TMEM lanes 32q..32q+31
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            int mb, nb;
            tile_coords(t / ksplit, tiles_m, tiles_n, mb, nb);
            const int acc = it & 1;
            mbar_wait(&tfull[acc], (it >> 1) & 1);
            fence_after();
            const int m = mb * BM + q * 32 + lane;
#pragma unroll 1
            for (int ch = 0; ch < BN / 32; ++ch) {
                uint32_t r[32];
                tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + ch * 32), r);
                const int n = nb * BN + ch * 32;
                if (m < M && n < N) {
                    if (ksplit > 1) {
                        float* o = acc_out + int64_t(m) * N + n;
#pragma unroll
                        for (int j = 0; j < 32; ++j) atomicAdd(o + j, __uint_as_float(r[j]));
                    } else {
                        float v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                        epilogue_chunk(epi, m, n, v);
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::TMEM_COLS)
                     : "memory");
    }
}

// split-K finalisation: the fused epilogue over the reduced fp32 tile
// (it leaves the workspace zeroed for the next split-K GEMM)
__global__ void splitk_epilogue_kernel(float* __restrict__ acc, int M, int N, EpiArgs epi) {
    const int chunks = N / 32;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < M * chunks; e += gridDim.x * blockDim.x) {
        const int m = e / chunks, n = (e % chunks) * 32;
        float v[32];
        float4* src = reinterpret_cast<float4*>(acc + int64_t(m) * N + n);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 x = src[q];
            src[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
        epilogue_chunk(epi, m, n, v);
    }
}

// ------------------------------------------------------------ skinny GEMM --
// M <= 16 rows (the layers after the walk compute only the query rows): the
// GEMM is a weight stream, HBM-bound at 2*N*K bytes.  Persistent CTAs walk a
// contiguous range of (64-row n-block, 256-wide k-stage) units; a producer warp
// TMA-loads each stage (B: four 64x64 boxes, A: four 16x64 boxes, 40 KB) into
// a 4-deep ring and four consumer warps each multiply one 64-wide k slice on
// mma.sync m16n8k16 (the MMA is never the bound at 16 rows).  Partial sums
// go to the fp32 split-K workspace with vector reductions whenever a CTA
// leaves an n-block; splitk_epilogue_kernel applies the fused epilogue.
constexpr int SK_ST = 4;
constexpr int SK_BOXB = 64 * 64 * 2;  // B box: 64 n x 64 k
constexpr int SK_THREADS = 5 * 32;
template <int MT>  // m16 tiles: M <= 16 * MT
struct SkCfg {
    static constexpr int BOXA = 16 * MT * 64 * 2;  // A box: 16 MT rows x 64 k
    static constexpr int STAGE = 4 * SK_BOXB + 4 * BOXA;
    static constexpr int SMEM = 1024 + SK_ST * STAGE + 2 * SK_ST * 8;
};

template <int MT>
__global__ void __launch_bounds__(SK_THREADS, 1)
gemm_skinny_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M, int N,
                   int K, float* __restrict__ acc) {
    using SC = SkCfg<MT>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + SK_ST * SC::STAGE);
    uint64_t* empty = full + SK_ST;
    const int nb_count = int(ceil_div(N, 64)), ks_count = int(ceil_div(K, 256));
    const int64_t units = int64_t(nb_count) * ks_count;
    const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SK_ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 4) {
        if (lane == 0) {
            prefetch_map(&ta);
            prefetch_map(&tb);
            for (int64_t u = u0; u < u1; ++u) {
                const int j = int(u - u0), s = j % SK_ST;
                if (j >= SK_ST) mbar_wait(&empty[s], uint32_t(j / SK_ST - 1) & 1u);
                mbar_expect_tx(&full[s], SC::STAGE);
                const int nb = int(u / ks_count), k0 = int(u % ks_count) * 256;
                uint8_t* st = sm + s * SC::STAGE;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    tma_load_2d(st + q * SK_BOXB, &tb, &full[s], k0 + 64 * q, nb * 64);
                    tma_load_2d(st + 4 * SK_BOXB + q * SC::BOXA, &ta, &full[s], k0 + 64 * q, 0);
                }
            }
        }
        return;
    }
    const int g = lane >> 2, i4 = lane & 3, mat = lane >> 3;
    float c[MT][8][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) c[mt][nt][0] = c[mt][nt][1] = c[mt][nt][2] = c[mt][nt][3] = 0.f;
    int cur_nb = -1;
    auto flush = [&](int nb) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int r0 = 16 * mt + g, r1 = r0 + 8;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const int col = nb * 64 + nt * 8 + 2 * i4;
                if (col < N) {
                    if (r0 < M)
                        atomicAdd(reinterpret_cast<float2*>(acc + int64_t(r0) * N + col),
                                  make_float2(c[mt][nt][0], c[mt][nt][1]));
                    if (r1 < M)
                        atomicAdd(reinterpret_cast<float2*>(acc + int64_t(r1) * N + col),
                                  make_float2(c[mt][nt][2], c[mt][nt][3]));
                }
                c[mt][nt][0] = c[mt][nt][1] = c[mt][nt][2] = c[mt][nt][3] = 0.f;
            }
        }
    };
    for (int64_t u = u0; u < u1; ++u) {
        const int j = int(u - u0), s = j % SK_ST;
        const int nb = int(u / ks_count);
        if (nb != cur_nb) {
            if (cur_nb >= 0) flush(cur_nb);
            cur_nb = nb;
        }
        mbar_wait(&full[s], uint32_t(j / SK_ST) & 1u);
        const uint32_t sb = smem_u32(sm + s * SC::STAGE);
        const uint32_t bb = sb + warp * SK_BOXB, ab = sb + 4 * SK_BOXB + warp * SC::BOXA;
#pragma unroll
        for (int kp = 0; kp < 2; ++kp) {  // two k-steps of 16 per pass
            uint32_t a0[MT][4], a1[MT][4];
            // A (m16 x k16) of m-tile mt: matrices (rows 0-7, k 0-7), (rows 8-15, k 0-7),
            // (rows 0-7, k 8-15), (rows 8-15, k 8-15); the 16 MT-row box keeps the swizzle row
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int ar = 16 * mt + ((mat & 1) << 3) + (lane & 7);
                ldsm_x4(ab + swz(ar, kp * 4 + (mat >> 1)), a0[mt][0], a0[mt][1], a0[mt][2], a0[mt][3]);
                ldsm_x4(ab + swz(ar, kp * 4 + 2 + (mat >> 1)), a1[mt][0], a1[mt][1], a1[mt][2], a1[mt][3]);
            }
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4(bb + swz(nt * 8 + (lane & 7), kp * 4 + mat), b0, b1, b2, b3);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    mma16816(c[mt][nt], a0[mt], b0, b1);
                    mma16816(c[mt][nt], a1[mt], b2, b3);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (cur_nb >= 0) flush(cur_nb);
}

float* splitk_workspace(int M, int N, cudaStream_t st) {
    // grow-only fp32 workspace per (device, stream): GEMMs in flight on
    // different streams (or contexts on different GPUs) never share one.
    // Zeroed once when it grows; every finalisation pass re-zeroes what it read.
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::unique_ptr<DevBuf>> pool;
    int dev = 0;
    KEEP_CUDA(cudaGetDevice(&dev));
    DevBuf* ws;
    {
        std::lock_guard<std::mutex> g(mu);
        auto& slot = pool[{dev, st}];
        if (!slot) slot.reset(new DevBuf());
        ws = slot.get();
    }
    const size_t need = sizeof(float) * size_t(M) * N;
    if (need > ws->bytes || !ws->p) {
        ws->ensure(need);
        KEEP_CUDA(cudaMemsetAsync(ws->p, 0, ws->bytes, st));
    }
    return ws->as<float>();
}

template <int MT>
void launch_skinny_mt(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bt, int64_t ldb, int M, int N, int K,
                      const EpiArgs& epi, cudaStream_t st, int max_ctas) {
    smem_attr(gemm_skinny_kernel<MT>, SkCfg<MT>::SMEM);
    const CUtensorMap ta = make_map_bf16(A, M, K, lda, 16 * MT);
    const CUtensorMap tb = make_map_bf16(Bt, N, K, ldb, 64);
    const int64_t units = ceil_div(N, 64) * ceil_div(K, 256);
    const int grid = int(std::min<int64_t>(units, std::max(1, std::min(max_ctas, kNumSMs))));
    float* acc = splitk_workspace(M, N, st);
    gemm_skinny_kernel<MT><<<grid, SK_THREADS, SkCfg<MT>::SMEM, st>>>(ta, tb, M, N, K, acc);
    KEEP_LAUNCH_CHECK();
    const int work = M * (N / 32);
    splitk_epilogue_kernel<<<unsigned(std::min<int64_t>(ceil_div(work, 128), kNumSMs * 4)), 128, 0, st>>>(acc, M, N, epi);
    KEEP_LAUNCH_CHECK();
}

void launch_skinny(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bt, int64_t ldb, int M, int N, int K,
                   const EpiArgs& epi, cudaStream_t st, int max_ctas) {
    if (M <= 16) launch_skinny_mt<1>(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas);
    else launch_skinny_mt<2>(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas);
}

template <int BN, int AR = BM>
void launch_bn(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bt, int64_t ldb, int M, int N, int K,
               const EpiArgs& epi, cudaStream_t st, int max_ctas = kNumSMs, int ksplit = 1) {
    using CF = Cfg<BN, AR>;
    static_assert(CF::SMEM <= 232448, "GEMM smem");
    smem_attr(gemm_tc_kernel<BN, AR>, int(CF::SMEM));
    const CUtensorMap ta = make_map_bf16(A, M, K, lda, AR);
    const CUtensorMap tb = make_map_bf16(Bt, N, K, ldb, BN);
    const int ntiles = int(ceil_div(M, BM) * ceil_div(N, BN)) * ksplit;
    const int grid = std::min(ntiles, std::max(1, std::min(max_ctas, kNumSMs)));
    float* acc = ksplit > 1 ? splitk_workspace(M, N, st) : nullptr;
    gemm_tc_kernel<BN, AR><<<grid, kThreads, CF::SMEM, st>>>(ta, tb, M, N, K, epi, ksplit, acc);
    KEEP_LAUNCH_CHECK();
    if (ksplit > 1) {
        const int work = M * (N / 32);
        splitk_epilogue_kernel<<<unsigned(std::min<int64_t>(ceil_div(work, 128), kNumSMs * 4)), 128, 0, st>>>(acc, M, N,
                                                                                                         epi);
        KEEP_LAUNCH_CHECK();
    }
}

}  // namespace

bool skinny_enabled() {  // KEEP_GEMM_SKINNY=0: the tcgen05 split-K path for M <= 16 too (A/B)
    static const bool on = [] {
        const char* e = std::getenv("KEEP_GEMM_SKINNY");
        return !(e && *e == '0');
    }();
    return on;
}

void launch_gemm_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bt, int64_t ldb, int M, int N, int K,
                      const EpiArgs& epi, cudaStream_t st, int max_ctas) {
    if (M == 0 || N == 0) return;
    if (K % BK != 0 || N % 32 != 0) raise(KEEP_ERR_CONFIG, "tcgen05 GEMM needs K % 64 == 0 and N % 32 == 0");
    // a few rows (deep layers: the query): 32-row A stages and split-K so that
    // ~4 waves of (tile, k-slice) units stream the weights through every SM
    if (M <= 32 && skinny_enabled()) {
        launch_skinny(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas);
        return;
    }
    if (M <= 32) {
        const int tiles = int(ceil_div(N, 64)), kb = K / BK;
        const int ksplit = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(4 * kNumSMs, tiles), kb / 8)));
        launch_bn<64, 32>(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas, ksplit);
        return;
    }
    // 128x256 tiles whenever they fill most of a wave: 64-wide tiles feed the
    // tensor core at well under half the rate (the A tile is re-staged per 64
    // columns).  Fewer tiles: split K across the idle SMs (fp32 reduction plus
    // the fused-epilogue pass), else fall back to narrow tiles.
    const int64_t t256 = ceil_div(M, BM) * ceil_div(N, 256);
    const int ctas = std::max(1, std::min(max_ctas, kNumSMs));
    if (t256 * 10 >= int64_t(ctas) * 7 || N % 256 != 0) {
        launch_bn<256>(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas);
        return;
    }
    const int ks = int(std::min<int64_t>(ctas / t256, (K / BK) / 8));
    if (ks >= 2)
        launch_bn<256>(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas, ks);
    else
        launch_bn<64>(A, lda, Bt, ldb, M, N, K, epi, st, max_ctas);
}

}  // namespace keep_b200

// Test hook: plain fp32-output GEMM on device pointers (C = A . Bt^T).
extern "C" int keep_debug_gemm_bf16(const void* A, const void* Bt, float* Cout,
                                                                           int M, int N, int K, int force_bn) {
    try {
        const bool sync = force_bn < 1000;  // force_bn + 1000: asynchronous (microbenchmarks)
        force_bn %= 1000;
        keep_b200::EpiArgs e{keep_b200::EPI_STORE, 0, Cout, N, nullptr, nullptr, nullptr, nullptr};
        auto a = static_cast<const __nv_bfloat16*>(A);
        auto b = static_cast<const __nv_bfloat16*>(Bt);
        if (force_bn == 256) keep_b200::launch_bn<256>(a, K, b, K, M, N, K, e, 0);
        else if (force_bn == 64) keep_b200::launch_bn<64>(a, K, b, K, M, N, K, e, 0);
        else if (force_bn == 32) keep_b200::launch_bn<32, 32>(a, K, b, K, M, N, K, e, 0);
        else if (force_bn == 16) keep_b200::launch_skinny(a, K, b, K, M, N, K, e, 0, keep_b200::kNumSMs);
        else keep_b200::launch_gemm_bf16(a, K, b, K, M, N, K, e, 0);
        if (!sync) return cudaGetLastError() == cudaSuccess ? 0 : KEEP_ERR_CUDA;
        return cudaDeviceSynchronize() == cudaSuccess ? 0 : KEEP_ERR_CUDA;
    } catch (const keep_b200::KeepError& e) {
        return e.code;
    }
}
