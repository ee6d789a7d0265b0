// fp64 tensor-core shapes on this B200: m8n8k4 vs m16n8k{4,8,16} (sm_90+ PTX),
// and whether DFMA issued beside DMMA shares its pipe.
#include <cstdio>
#include <cuda_runtime.h>
template <int SHAPE, int NACC>
__global__ void loop(double* out, int iters, int dfma_per) {
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
    double c[NACC][4];
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    double f[8];
    for (int i = 0; i < 8; ++i) f[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) {
            if (SHAPE == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
            else if (SHAPE == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            else if (SHAPE == 2)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
        for (int k = 0; k < dfma_per; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = fma(a[i], b[i & 3], f[i]);
    }
    double s = 0;
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    for (int i = 0; i < 8; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int SHAPE, int NACC>
void run(const char* name, double* out, int warps, int dfma_per) {
    const int iters = 4000;
    const double fl[4] = {2.0 * 256, 2.0 * 512, 2.0 * 1024, 2.0 * 2048};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    loop<SHAPE, NACC><<<148, warps * 32>>>(out, 10, dfma_per);
    cudaEventRecord(a);
    loop<SHAPE, NACC><<<148, warps * 32>>>(out, iters, dfma_per);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double mma = fl[SHAPE] * NACC * double(iters) * warps * 148;
    const double fma_ = 2.0 * 8 * dfma_per * double(iters) * warps * 32 * 148;
    printf("%-10s warps %2d acc %d dfma/iter %2d: MMA %.1f TFLOP/s  DFMA %.1f TFLOP/s  (%.3f ms)\n", name, warps, NACC,
           dfma_per * 8, mma / ms / 1e9, fma_ / ms / 1e9, ms);
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    for (int w : {4, 8, 16}) {
        run<0, 8>("m8n8k4", out, w, 0);
        run<1, 8>("m16n8k4", out, w, 0);
        run<2, 8>("m16n8k8", out, w, 0);
        run<3, 8>("m16n8k16", out, w, 0);
    }
    for (int d : {1, 2, 4, 8}) {
        run<0, 8>("m8n8k4", out, 8, d);
        run<3, 8>("m16n8k16", out, 8, d);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
