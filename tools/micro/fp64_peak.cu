// fp64 throughput probe on this B200: DMMA (mma.sync m8n8k4 f64) vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[16];
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps : {4, 8, 16, 32}) {
        int iters = 20000;
        dmma_loop<<<148 * 2, warps * 32>>>(out, 10);
        cudaEventRecord(a);
        dmma_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double flops = 2.0 * 256 * 8 * double(iters) * warps * 148 * 2;
        printf("DMMA warps/CTA %d: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
        dfma_loop<<<148 * 2, warps * 32>>>(out, 10);
        cudaEventRecord(a);
        dfma_loop<<<148 * 2, warps * 32>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        flops = 2.0 * 16 * double(iters) * warps * 32 * 148 * 2;
        printf("DFMA warps/CTA %d: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
