// f64_exp.cuh -- fp64 exp for the PARITY attention softmax.
//
// On this B200 the fp64 CUDA-core instructions share the fp64 tensor pipe
// with DMMA: one DFMA warp instruction costs ~0.38 of an m8n8k4 DMMA's pipe
// time (tools/micro/fp64_shapes.cu: 8 DMMA + 8 DFMA per iteration run at
// 26.5 + 3.3 TFLOP/s against 36.5 for DMMA alone).  CUDA's exp() spends ~22
// fp64 instructions per call (an 11-term polynomial on |r| <= ln2 / 2 plus
// special cases), ~26% of the flash pass's DMMA time.  This one reduces to
// |r| <= ln2 / 128 with a 64-entry table of 2^(j/64) in shared memory:
//
//   x = (64 m + j) ln2/64 + r,  e^x = 2^m * 2^(j/64) * p(r),
//   p = 1 + r + r^2/2 + r^3/6 + r^4/24 + r^5/120   (truncation <= 3.5e-17)
//
// ~10 fp64 instructions; the result is within 2 ulp of the correctly rounded
// e^x (Cody-Waite reduction with a 36-bit ln2/64 head, table entries
// correctly rounded, Horner rounding) -- an fp64 rounding-level difference
// like the summation order; tests/test_gpu_exp.py
// measures it against the host libm.  Valid for x <= 709 (the softmax
// arguments are s - max <= 256); below -745.2 the result underflows to 0.
#pragma once

namespace keep_b200 {

__constant__ double kExp2Tab64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

// smem copy of the table (64 doubles), filled by the first 64 threads
__device__ __forceinline__ void exp_tab_load(double* tab) {
    if (threadIdx.x < 64) tab[threadIdx.x] = kExp2Tab64[threadIdx.x];
}

__device__ __forceinline__ double exp_f64(double x, const double* tab) {
    constexpr double kInvL = 0x1.71547652b82fep+6;   // 64 / ln 2
    constexpr double kLHi = 0x1.62e42fefa0000p-7;    // ln2/64, 36 significant bits: k * kLHi exact
    constexpr double kLLo = 0x1.cf79abc9e3b3ap-46;   // ln2/64 - kLHi
    constexpr double kShift = 0x1.8p52;              // round-to-integer magic
    if (x < -745.2) return 0.0;  // (also keeps kd in the magic range: deep layers see s - max ~ -1e18)
    const double kd = fma(x, kInvL, kShift);
    const int ki = __double2loint(kd);
    const double k = kd - kShift;
    double r = fma(k, -kLHi, x);
    r = fma(k, -kLLo, r);
    double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(r, p, 1.0 / 6.0);
    p = fma(r, p, 0.5);
    p = fma(r, p, 1.0);
    p = fma(r, p, 1.0);
    const double v = tab[ki & 63] * p;  // in [0.99, 2.01)
    const int e = ki >> 6;              // floor(k / 64)
    if (e >= -1021) return __hiloint2double(__double2hiint(v) + (e << 20), __double2loint(v));
    // subnormal result: one exact power-of-two scaling, then one rounding
    return (v * __hiloint2double((e + 600 + 1023) << 20, 0)) * 0x1p-600;
}

}  // namespace keep_b200
