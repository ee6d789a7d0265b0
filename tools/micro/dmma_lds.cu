// DMMA fed from shared memory (the attention kernels' pattern) vs from registers.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE>  // 0: B in registers; 1: B = LDS per DMMA (8 rows/warp); 2: one LDS feeds two m-tiles (16 rows/warp)
__global__ void k(double* out, int iters) {
    __shared__ double sm[32 * 132];
    for (int i = threadIdx.x; i < 32 * 132; i += blockDim.x) sm[i] = i * 1e-3;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    double a0 = lane * 1e-3, a1 = lane * 2e-3, breg = 1.0 + lane;
    double c[8][2] = {}, d[8][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                double b = MODE == 0 ? breg : sm[(8 * j + g) * 132 + 4 * i + t];
                dmma(c[j], a0, b);
                if (MODE == 2) dmma(d[j], a1, b);
            }
        }
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(double* out, int warps) {
    const int iters = 200;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE><<<148, warps * 32>>>(out, 2);
    cudaEventRecord(a);
    k<MODE><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fl = 512.0 * 32 * 4 * (MODE == 2 ? 2 : 1) * double(iters) * warps * 148;
    printf("mode %d warps %2d: %.1f TFLOP/s\n", MODE, warps, fl / ms / 1e9);
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    for (int w : {4, 8, 12, 16}) {
        run<0>(out, w);
        run<1>(out, w);
        run<2>(out, w);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
