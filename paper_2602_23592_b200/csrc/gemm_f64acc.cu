// gemm_f64acc.cu -- PARITY projection GEMM: fp32 operands, fp64 accumulation.
//
// Every output element is accumulated by one thread over k in ascending order
// with DFMA.  The product of two fp32 values is exact in fp64, so
// fma(a, b, acc) == acc + a*b rounded once == the reference's
// `acc[j] += xi * wrow[j]` (tensor.hpp:36-39): the fp32 result is bit-exact
// with vec_mat for any tiling in M/N (no split-K, k never reordered).
// Fused epilogues: QKV split + scatter of K/V rows into the merged cache,
// fp32 residual add (prefill.hpp:289-291, 302-303), ReLU (299-300).
#include "kernels.hpp"

namespace keep_b200 {

namespace {
constexpr int BM = 64, BN = 64, BK = 16, TR = 4, TC = 4;
}

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
            const float v = static_cast<float>(acc[r][c]);
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
    }
}

void launch_gemm_f64acc(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K,
                        const EpiArgs& epi, cudaStream_t st) {
    if (M == 0 || N == 0) return;
    dim3 grid(static_cast<unsigned>(ceil_div(N, BN)), static_cast<unsigned>(ceil_div(M, BM)));
    gemm_f64acc_kernel<<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, epi);
    KEEP_LAUNCH_CHECK();
}

}  // namespace keep_b200
