// Sustained fp64 DMMA throughput on this B200: m8n8k4 with random operands
// that alternate every iteration (toggling inputs draw realistic power), run
// back to back for ~5 s -- the roofline peak for a DMMA kernel timed inside a
// long step (the burst loop in fp64_peak.cu keeps its operands constant).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters, unsigned seed) {
    unsigned x = seed ^ (blockIdx.x * 1024u + threadIdx.x) * 2654435761u;
    auto rnd = [&]() {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        return 1.0 + (x & 0xFFFFFF) * 0x1p-24;
    };
    const double a0 = rnd(), b0 = rnd(), a1 = -rnd(), b1 = rnd();
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b0));
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a1), "d"(b1));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 2 * 512 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int warps = 8, iters = 20000;
    dmma_loop<<<148 * 2, warps * 32>>>(out, 100, 1);
    double best = 0, last = 0;
    int n = 0;
    float total = 0;
    while (total < 5000.f) {
        cudaEventRecord(a);
        dmma_loop<<<148 * 2, warps * 32>>>(out, iters, 7 + n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        total += ms;
        last = 2.0 * 256 * 16 * double(iters) * warps * 148 * 2 / ms / 1e9;
        if (n == 0) best = last;
        ++n;
    }
    printf("{\"fp64_dmma_tflops_first\": %.2f, \"fp64_dmma_tflops_sustained\": %.2f, \"seconds\": %.1f, \"launches\": %d}\n",
           best, last, total / 1e3, n);
}
