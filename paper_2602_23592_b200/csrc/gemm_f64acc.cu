// gemm_f64acc.cu -- PARITY projection GEMM: fp32 operands, fp64 accumulation.
//
// Every output element is accumulated by one thread over k in ascending order
// with DFMA.  The product of two fp32 values is exact in fp64, so
// fma(a, b, acc) == acc + a*b rounded once == the reference's
// `acc[j] += xi * wrow[j]` (tensor.hpp:36-39): the fp32 result is bit-exact
// with vec_mat for any tiling in M/N (no split-K, k never reordered).
// Fused epilogues: QKV split + scatter of K/V rows into the merged cache,
// fp32 residual add (prefill.hpp:289-291, 302-303), ReLU (299-300).
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>

#include "engine.hpp"

namespace keep_b200 {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, TR = 4, TC = 4;

__device__ __forceinline__ void epi_store1(const EpiArgs& epi, int m, int n, float v) {
    switch (epi.kind) {
        case EPI_QKV: {
            const int d = epi.d;
            if (n < d) {
                epi.out[int64_t(m) * epi.ldo + n] = v;
            } else if (n < 2 * d) {
                static_cast<float*>(epi.kdst)[int64_t(epi.rows[m]) * d + (n - d)] = v;
            } else {
                static_cast<float*>(epi.vdst)[int64_t(epi.rows[m]) * d + (n - 2 * d)] = v;
            }
            break;
        }
        case EPI_RESID: {
            float* o = epi.out + int64_t(m) * epi.ldo + n;
            const float x = *o + v;
            *o = x;
            if (epi.out_bf16) epi.out_bf16[int64_t(m) * epi.ldo + n] = __float2bfloat16_rn(x);
            break;
        }
        case EPI_RELU:
            epi.out[int64_t(m) * epi.ldo + n] = (v < 0.0f) ? 0.0f : v;
            break;
        default:
            epi.out[int64_t(m) * epi.ldo + n] = v;
    }
}
}  // namespace

__global__ void __launch_bounds__(256)
gemm_f64acc_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                   int M, int N, int K, EpiArgs epi) {
    __shared__ double As[BK][BM];
    __shared__ double Bs[BK][BN];
    const int t = threadIdx.x;
    const int ty = t / 16, tx = t % 16;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    double acc[TR][TC];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[r][c] = 0.0;

    const int la_row = t / 4, la_k = (t % 4) * 4;   // A: 64 rows x 16 k
    const int lb_k = t / 16, lb_n = (t % 16) * 4;   // B: 16 k x 64 cols
    for (int k0 = 0; k0 < K; k0 += BK) {
        {
            const int m = m0 + la_row;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int k = k0 + la_k + c;
                As[la_k + c][la_row] = (m < M && k < K) ? double(A[int64_t(m) * lda + k]) : 0.0;
            }
            const int k = k0 + lb_k;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int n = n0 + lb_n + c;
                Bs[lb_k][lb_n + c] = (k < K && n < N) ? double(B[int64_t(k) * ldb + n]) : 0.0;
            }
        }
        __syncthreads();
        const int kmax = min(BK, K - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            double a[TR], b[TC];
#pragma unroll
            for (int r = 0; r < TR; ++r) a[r] = As[kk][ty + 16 * r];
#pragma unroll
            for (int c = 0; c < TC; ++c) b[c] = Bs[kk][tx + 16 * c];
#pragma unroll
            for (int r = 0; r < TR; ++r)
#pragma unroll
                for (int c = 0; c < TC; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }

#pragma unroll
    for (int r = 0; r < TR; ++r) {
        const int m = m0 + ty + 16 * r;
        if (m >= M) continue;
#pragma unroll
        for (int c = 0; c < TC; ++c) {
            const int n = n0 + tx + 16 * c;
            if (n >= N) continue;
            epi_store1(epi, m, n, static_cast<float>(acc[r][c]));
        }
    }
}

namespace {
// ------------------------------------------------------------ skinny GEMM --
// M <= 32 rows (the layers after the walk recompute only the query): a
// weight stream, HBM-bound at 4 N K bytes.  CTA = 32 columns x every row x all
// of K; 256 threads = 8 row slots x 32 columns, RPT rows per thread.  B and A
// tiles (32 k x 32 columns, M x 32 k) arrive by cp.async in a 4-deep ring (several
// CTAs per SM keep ~64 KB of the stream in flight) and
// are widened to fp64 once per stage (not per use: the fp32 -> fp64 convert
// runs on the quarter-rate XU pipe).  Every output is still one thread's DFMA
// chain in ascending k: bit-exact with vec_mat, like the tiled kernel.
constexpr int SK_KB = 32, SK_ST = 4, SK_NC = 32;

__device__ __forceinline__ void cpa16(void* dst, const void* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

template <int RPT>
__global__ void __launch_bounds__(256) gemm_f64_skinny_kernel(const float* __restrict__ A, int64_t lda,
                                                              const float* __restrict__ B, int64_t ldb, int M, int N,
                                                              int K, int kchunk, double* __restrict__ part,
                                                              EpiArgs epi) {
    constexpr int MR = 8 * RPT;
    __shared__ __align__(16) float bst[SK_ST][SK_KB][SK_NC];
    __shared__ __align__(16) float ast[SK_ST][MR][SK_KB];
    __shared__ double bd[SK_KB][SK_NC];
    __shared__ double ad[MR][SK_KB];
    const int tid = threadIdx.x, col = tid & 31, rs = tid >> 5;
    const int n0 = blockIdx.x * SK_NC;
    // this CTA's k range [kbeg, kend) (split-K: blockIdx.y)
    const int kbeg = blockIdx.y * kchunk, kend = min(K, kbeg + kchunk);
    const int nkb = int(ceil_div(kend - kbeg, SK_KB));
    auto issue = [&](int kb) {
        if (kb < nkb) {
            const int s = kb % SK_ST, k0 = kbeg + kb * SK_KB;
            {  // B: 32 k-rows x 128 bytes
                const int r = tid >> 3, c = tid & 7;
                const bool ok = k0 + r < kend && n0 + 4 * c < N;
                cpa16(&bst[s][r][4 * c], B + (ok ? int64_t(k0 + r) * ldb + n0 + 4 * c : 0), ok);
            }
            for (int e = tid; e < M * 8; e += 256) {  // A: M rows x 128 bytes
                const int r = e >> 3, c = e & 7;
                const bool ok = k0 + 4 * c < kend;
                cpa16(&ast[s][r][4 * c], A + (ok ? int64_t(r) * lda + k0 + 4 * c : 0), ok);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int kb = 0; kb < SK_ST - 1; ++kb) issue(kb);
    double acc[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
    for (int kb = 0; kb < nkb; ++kb) {
        asm volatile("cp.async.wait_group %0;" ::"n"(SK_ST - 2) : "memory");
        __syncthreads();  // stage kb landed; the previous fp64 tile is consumed
        const int s = kb % SK_ST;
        for (int e = tid; e < SK_KB * SK_NC; e += 256) bd[e >> 5][e & 31] = double(bst[s][e >> 5][e & 31]);
        for (int e = tid; e < M * SK_KB; e += 256) ad[e >> 5][e & 31] = double(ast[s][e >> 5][e & 31]);
        __syncthreads();
        issue(kb + SK_ST - 1);
        const int kn = min(SK_KB, kend - kbeg - kb * SK_KB);
        for (int kk = 0; kk < kn; ++kk) {
            const double b = bd[kk][col];
#pragma unroll
            for (int r = 0; r < RPT; ++r) acc[r] = fma(ad[rs + 8 * r][kk], b, acc[r]);
        }
    }
    const int n = n0 + col;
    if (n >= N) return;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int m = rs + 8 * r;
        if (m >= M) continue;
        if (part) part[(int64_t(blockIdx.y) * M + m) * N + n] = acc[r];
        else if (epi.kind == EPI_F64) reinterpret_cast<double*>(epi.out)[int64_t(m) * epi.ldo + n] = acc[r];
        else epi_store1(epi, m, n, static_cast<float>(acc[r]));
    }
}

// ------------------------------------------------------------ weight stream --
// PARITY (split-K allowed) for M <= 32: a warp owns 32 CPL columns (CPL
// consecutive floats per lane: 128 CPL contiguous bytes per k-row) and streams
// its B strip through its own 3-stage cp.async ring in shared memory (8 k-rows
// per stage; each lane reads back only the bytes it copied, so no barrier);
// A's MR rows of the CTA's k-range are widened once into shared memory and read
// as broadcast k-pairs.  MR x CPL independent fp64 chains per lane in
// ascending k.  CTA = 8 warps; grid (column blocks, k splits, row groups).
constexpr int WS_UN = 8, WS_ST = 3, WS_KMAX = 512;

template <int CPL>
__device__ __forceinline__ void cpa_b(void* dst, const void* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    if constexpr (CPL == 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

size_t stream_smem(int MR, int CPL, int kchunk) {
    return sizeof(double) * size_t(MR) * kchunk + sizeof(float) * size_t(8) * WS_ST * WS_UN * 32 * CPL;
}

template <int MR, int CPL>
__global__ void __launch_bounds__(256, 2) gemm_f64_stream_kernel(const float* __restrict__ A, int64_t lda,
                                                              const float* __restrict__ B, int64_t ldb, int M, int N,
                                                              int K, int kchunk, double* __restrict__ part,
                                                              EpiArgs epi) {
    constexpr int WC = 32 * CPL;  // columns per warp
    extern __shared__ __align__(16) double as[];  // [MR][kchunk], then the warps' B rings
    const int kbeg = blockIdx.y * kchunk, kn = min(K, kbeg + kchunk) - kbeg;
    const int m0 = blockIdx.z * MR, mr = min(MR, M - m0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = (blockIdx.x * 8 + warp) * WC + CPL * lane;
    const bool nok = n < N;
    float* ring = reinterpret_cast<float*>(as + MR * kchunk) + warp * (WS_ST * WS_UN * WC) + CPL * lane;
    const float* bp = B + int64_t(kbeg) * ldb + (nok ? n : 0);
    const int nit = int(ceil_div(kn, WS_UN));
    auto issue = [&](int it) {  // k-rows 8 it .. 8 it + 7 into stage it % WS_ST
        if (it < nit) {
            float* dst = ring + (it % WS_ST) * (WS_UN * WC);
#pragma unroll
            for (int u = 0; u < WS_UN; ++u) {
                const int k = it * WS_UN + u;
                cpa_b<CPL>(dst + u * WC, bp + int64_t(k < kn ? k : 0) * ldb, nok && k < kn);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int it = 0; it < WS_ST - 1; ++it) issue(it);
    for (int e = threadIdx.x; e < MR * kchunk; e += 256) {
        const int r = e / kchunk, k = e - r * kchunk;
        as[e] = (r < mr && k < kn) ? double(A[int64_t(m0 + r) * lda + kbeg + k]) : 0.0;
    }
    __syncthreads();
    double acc[MR][CPL];
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[r][c] = 0.0;
    for (int it = 0; it < nit; ++it) {
        asm volatile("cp.async.wait_group %0;" ::"n"(WS_ST - 2) : "memory");
        const float* src = ring + (it % WS_ST) * (WS_UN * WC);
        issue(it + WS_ST - 1);  // into the stage read in the previous iteration
#pragma unroll
        for (int u = 0; u < WS_UN; u += 2) {  // rows past kn are zero-filled (0 * a adds nothing)
            const int k = it * WS_UN + u;
            double b0[CPL], b1[CPL];
            if constexpr (CPL == 4) {
                const float4 v0 = *reinterpret_cast<const float4*>(src + u * WC);
                const float4 v1 = *reinterpret_cast<const float4*>(src + (u + 1) * WC);
                b0[0] = v0.x, b0[1] = v0.y, b0[2] = v0.z, b0[3] = v0.w;
                b1[0] = v1.x, b1[1] = v1.y, b1[2] = v1.z, b1[3] = v1.w;
            } else {
                const float2 v0 = *reinterpret_cast<const float2*>(src + u * WC);
                const float2 v1 = *reinterpret_cast<const float2*>(src + (u + 1) * WC);
                b0[0] = v0.x, b0[1] = v0.y;
                b1[0] = v1.x, b1[1] = v1.y;
            }
#pragma unroll
            for (int r = 0; r < MR; ++r) {
                const double2 a = *reinterpret_cast<const double2*>(as + r * kchunk + k);
#pragma unroll
                for (int c = 0; c < CPL; ++c) acc[r][c] = fma(a.y, b1[c], fma(a.x, b0[c], acc[r][c]));
            }
        }
    }
    if (!nok) return;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
        if (r >= mr) break;
        const int m = m0 + r;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            if (part) part[(int64_t(blockIdx.y) * M + m) * N + n + c] = acc[r][c];
            else if (epi.kind == EPI_F64) reinterpret_cast<double*>(epi.out)[int64_t(m) * epi.ldo + n + c] = acc[r][c];
            else epi_store1(epi, m, n + c, static_cast<float>(acc[r][c]));
        }
    }
}

// split-K finish: the k-range partials summed in ascending split order
// (deterministic), one rounding to fp32, the fused epilogue
__global__ void f64_splitk_finish_kernel(const double* __restrict__ part, int ks, int M, int N, EpiArgs epi) {
    const int64_t MN = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < MN; e += int64_t(gridDim.x) * blockDim.x) {
        double acc = part[e];
        for (int s = 1; s < ks; ++s) acc += part[int64_t(s) * MN + e];
        if (epi.kind == EPI_F64) reinterpret_cast<double*>(epi.out)[(e / N) * epi.ldo + e % N] = acc;
        else epi_store1(epi, int(e / N), int(e % N), static_cast<float>(acc));
    }
}

// KEEP_PARITY_STREAM=0: the smem-staged skinny kernel for PARITY's few rows too (A/B)
bool stream_f64_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KEEP_PARITY_STREAM");
        return !(e && *e == '0');
    }();
    return on;
}

// KEEP_PARITY_SKINNY=0: the tiled kernel for few rows too (A/B)
bool skinny_f64_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KEEP_PARITY_SKINNY");
        return !(e && *e == '0');
    }();
    return on;
}
}  // namespace

double* f64_splitk_workspace(size_t bytes, cudaStream_t st) {
    // grow-only per (device, stream): GEMMs in flight on different streams (or
    // contexts on different GPUs) never share one
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
    ws->ensure(bytes);
    return ws->as<double>();
}

void launch_gemm_f64acc(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                        const EpiArgs& epi, cudaStream_t st, bool exact) {
    if (M == 0 || N == 0) return;
    // few rows: the weight stream (16-byte cp.async needs 16-byte aligned rows)
    if (!exact && M <= 32 && stream_f64_enabled() && N % 4 == 0 && ldb % 4 == 0 &&
        reinterpret_cast<uintptr_t>(B) % 16 == 0) {
        // PARITY: the weight stream, split K over ~2 resident CTAs per SM; 4 columns
        // per lane for up to 8 rows, 2 for up to 16 (register budget)
        const int MR = M <= 8 ? 8 : 16, CPL = MR == 8 ? 4 : 2;
        const int nct = int(ceil_div(N, 256 * CPL)), ng = int(ceil_div(M, MR));
        int ks = int(std::max<int64_t>(ceil_div(K, WS_KMAX), std::min<int64_t>(ceil_div(4 * kNumSMs, int64_t(nct) * ng),
                                                                                   std::max(1, K / 128))));
        const int kchunk = int(ceil_div(ceil_div(K, ks), WS_UN) * WS_UN);
        ks = int(ceil_div(K, kchunk));
        double* part = ks > 1 ? f64_splitk_workspace(sizeof(double) * size_t(ks) * M * N, st) : nullptr;
        const dim3 grid{unsigned(nct), unsigned(ks), unsigned(ng)};
        const size_t smem = stream_smem(MR, CPL, kchunk);
        if (MR == 8) {
            smem_attr(gemm_f64_stream_kernel<8, 4>, int(smem));
            gemm_f64_stream_kernel<8, 4><<<grid, 256, smem, st>>>(A, lda, B, ldb, M, N, K, kchunk, part, epi);
        } else {
            smem_attr(gemm_f64_stream_kernel<16, 2>, int(smem));
            gemm_f64_stream_kernel<16, 2><<<grid, 256, smem, st>>>(A, lda, B, ldb, M, N, K, kchunk, part, epi);
        }
        KEEP_LAUNCH_CHECK();
        if (ks > 1) {
            f64_splitk_finish_kernel<<<unsigned(std::min<int64_t>(ceil_div(int64_t(M) * N, 256), kNumSMs * 4)), 256, 0,
                                       st>>>(part, ks, M, N, epi);
            KEEP_LAUNCH_CHECK();
        }
        return;
    }
    if (M <= 32 && skinny_f64_enabled() && K % 4 == 0 && N % 4 == 0 && lda % 4 == 0 && ldb % 4 == 0) {
        const int nct = int(ceil_div(N, SK_NC));
        // split K over enough CTAs to keep ~4 per SM streaming (a lone 32-column
        // CTA per SM cannot keep the HBM busy); PARITY_EXACT keeps one k chain
        // per output (bit-exact with vec_mat)
        int ks = exact ? 1 : int(std::min<int64_t>(ceil_div(4 * kNumSMs, nct), std::max(1, K / 512)));
        const int kchunk = int(ceil_div(ceil_div(K, ks), SK_KB) * SK_KB);
        ks = int(ceil_div(K, kchunk));
        double* part = ks > 1 ? f64_splitk_workspace(sizeof(double) * size_t(ks) * M * N, st) : nullptr;
        const dim3 grid{unsigned(nct), unsigned(ks), 1u};
        if (M <= 8) gemm_f64_skinny_kernel<1><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, kchunk, part, epi);
        else if (M <= 16) gemm_f64_skinny_kernel<2><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, kchunk, part, epi);
        else gemm_f64_skinny_kernel<4><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, kchunk, part, epi);
        KEEP_LAUNCH_CHECK();
        if (ks > 1) {
            f64_splitk_finish_kernel<<<unsigned(std::min<int64_t>(ceil_div(int64_t(M) * N, 256), kNumSMs * 4)), 256, 0,
                                       st>>>(part, ks, M, N, epi);
            KEEP_LAUNCH_CHECK();
        }
        return;
    }
    if (epi.kind == EPI_F64) raise(KEEP_ERR_CONFIG, "fp64 output: the few-row DFMA path only");
    dim3 grid(static_cast<unsigned>(ceil_div(N, BN)), static_cast<unsigned>(ceil_div(M, BM)));
    gemm_f64acc_kernel<<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, epi);
    KEEP_LAUNCH_CHECK();
}

// x[m][n] += float(sum[m][n]) (the residual add of prefill.hpp:289-291 / 302-303
// on a cross-rank fp64 sum)
__global__ void f64_resid_kernel(const double* __restrict__ sum, float* __restrict__ x, int M, int N, int64_t ldx) {
    const int64_t MN = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < MN; e += int64_t(gridDim.x) * blockDim.x) {
        float* o = x + (e / N) * ldx + e % N;
        *o = *o + static_cast<float>(sum[e]);
    }
}

void launch_f64_resid(const double* sum, float* x, int M, int N, int64_t ldx, cudaStream_t st) {
    const int64_t MN = int64_t(M) * N;
    if (MN == 0) return;
    f64_resid_kernel<<<unsigned(std::min<int64_t>(ceil_div(MN, 256), kNumSMs * 4)), 256, 0, st>>>(sum, x, M, N, ldx);
    KEEP_LAUNCH_CHECK();
}

}  // namespace keep_b200
