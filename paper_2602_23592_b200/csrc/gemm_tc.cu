// gemm_tc.cu -- FAST-mode projection GEMM (bf16 operands, fp32 accumulation).
// Interim SIMT implementation; replaced by the tcgen05/TMA kernel.
#include "engine.hpp"

namespace keep_b200 {

namespace {
constexpr int BM = 64, BN = 64, BK = 32;

__global__ void __launch_bounds__(256)
gemm_bf16_simt(const __nv_bfloat16* __restrict__ A, int64_t lda, const __nv_bfloat16* __restrict__ Bt,
               int64_t ldb, int M, int N, int K, EpiArgs epi) {
    __shared__ float As[BK][BM + 1];
    __shared__ float Bs[BK][BN + 1];
    const int t = threadIdx.x, ty = t / 16, tx = t % 16;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += BK) {
        for (int e = t; e < BM * BK; e += 256) {
            const int r = e / BK, k = e % BK;
            As[k][r] = (m0 + r < M && k0 + k < K) ? __bfloat162float(A[int64_t(m0 + r) * lda + k0 + k]) : 0.f;
            Bs[k][r] = (n0 + r < N && k0 + k < K) ? __bfloat162float(Bt[int64_t(n0 + r) * ldb + k0 + k]) : 0.f;
        }
        __syncthreads();
        for (int k = 0; k < BK; ++k) {
            float a[4], b[4];
            for (int r = 0; r < 4; ++r) a[r] = As[k][ty + 16 * r];
            for (int c = 0; c < 4; ++c) b[c] = Bs[k][tx + 16 * c];
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
    for (int r = 0; r < 4; ++r) {
        const int m = m0 + ty + 16 * r;
        if (m >= M) continue;
        for (int c = 0; c < 4; ++c) {
            const int n = n0 + tx + 16 * c;
            if (n >= N) continue;
            const float v = acc[r][c];
            const int d = epi.d;
            switch (epi.kind) {
                case EPI_QKV:
                    if (n < d) epi.out_bf16[int64_t(m) * d + n] = __float2bfloat16_rn(v);
                    else if (n < 2 * d)
                        static_cast<__nv_bfloat16*>(epi.kdst)[int64_t(epi.rows[m]) * d + n - d] = __float2bfloat16_rn(v);
                    else
                        static_cast<__nv_bfloat16*>(epi.vdst)[int64_t(epi.rows[m]) * d + n - 2 * d] = __float2bfloat16_rn(v);
                    break;
                case EPI_RESID: {
                    float* o = epi.out + int64_t(m) * epi.ldo + n;
                    const float x = *o + v;
                    *o = x;
                    epi.out_bf16[int64_t(m) * epi.ldo + n] = __float2bfloat16_rn(x);
                    break;
                }
                case EPI_RELU:
                    epi.out_bf16[int64_t(m) * epi.ldo + n] = __float2bfloat16_rn(v < 0.f ? 0.f : v);
                    break;
                default:
                    break;
            }
        }
    }
}
}  // namespace

void launch_gemm_bf16(const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bt, int64_t ldb, int M, int N,
                      int K, const EpiArgs& epi, cudaStream_t st) {
    if (M == 0 || N == 0) return;
    dim3 grid(static_cast<unsigned>(ceil_div(N, BN)), static_cast<unsigned>(ceil_div(M, BM)));
    gemm_bf16_simt<<<grid, 256, 0, st>>>(A, lda, Bt, ldb, M, N, K, epi);
    KEEP_LAUNCH_CHECK();
}

}  // namespace keep_b200
