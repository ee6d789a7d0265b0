// kernels_common.cu -- K0 init, K1 embed, row gathers, K4 merged-KV assembly,
// K6 summary reduce, K7 selector, K11 logits.  All HBM- or latency-bound
// integer/fp64 work: coalesced 16-byte accesses, grids sized in SM multiples.
#include <cstring>
#include <mutex>
#include <map>
#include <set>
#include <tuple>
#include "kernels.hpp"

#include <cfloat>

namespace keep_b200 {

void set_smem_attr(const void* fn, int bytes) {
    // the attribute only grows: a kernel launched with varying dynamic smem keeps
    // the largest opt-in it has seen on this device (lowering it after a larger
    // size was cached would fail the next larger launch)
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> seen;
    int dev = 0;
    KEEP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    int& cur = seen[{fn, dev}];
    if (bytes <= cur) return;
    KEEP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cur = bytes;
}

bool sync_debug() {
    static const bool on = [] {
        const char* e = std::getenv("KEEP_SYNC_DEBUG");
        return e && *e == '1';
    }();
    return on;
}

void trace_launch(const char* file, int line) {
    std::fprintf(stderr, "[keep] launch %s:%d ...", file, line);
    std::fflush(stderr);
    const cudaError_t e = cudaDeviceSynchronize();
    std::fprintf(stderr, " %s\n", cudaGetErrorString(e));
    std::fflush(stderr);
}

// ======================================================================= K0 ==
uint64_t fnv1a64_host(const char* s) {  // prng.hpp:23-30
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ULL;
    }
    return h;
}

__device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {  // prng.hpp:17-20
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Normal #e of the stream whose pre-warm-up state is s0: draws 12e..12e+11,
// draw n seeing state s0 + (n+3)*gamma (two warm-up draws, prng.hpp:34-38),
// summed in order in fp64 (Irwin-Hall, prng.hpp:57-61).
__device__ __forceinline__ float normal_at(uint64_t s0, uint64_t e, double std_) {
    const uint64_t g = 0x9e3779b97f4a7c15ULL;
    uint64_t st = s0 + (12ull * e + 3ull) * g;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        acc += static_cast<double>(sm64_mix(st) >> 11) * 0x1.0p-53;
        st += g;
    }
    return static_cast<float>((acc - 6.0) * std_);
}

// Output-order traversal so the (possibly transposed) stores coalesce; the
// counter-based stream lets every element be drawn independently.
__global__ void init_tensor_kernel(uint64_t s0, int64_t rows, int64_t cols, int64_t j0, int64_t jn, double std_,
                                   void* dst, int64_t ld, int64_t col_off, int transposed) {
    // columns [j0, j0 + jn) of the named [rows x cols] tensor (a head shard);
    // element (i, j) is normal #(i*cols + j) of the stream either way
    const int64_t n = rows * jn;
    for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < n;
         o += int64_t(gridDim.x) * blockDim.x) {
        if (!transposed) {
            const int64_t i = o / jn, jj = o % jn;
            static_cast<float*>(dst)[i * ld + col_off + jj] = normal_at(s0, uint64_t(i * cols + j0 + jj), std_);
        } else {
            const int64_t jj = o / rows, i = o % rows;  // dst row jj (output), col i (input)
            static_cast<__nv_bfloat16*>(dst)[(col_off + jj) * ld + i] =
                __float2bfloat16_rn(normal_at(s0, uint64_t(i * cols + j0 + jj), std_));
        }
    }
}

void launch_init_tensor(uint64_t seed, const char* name, int64_t rows, int64_t cols, double std_,
                        void* dst, int64_t ld, int64_t col_off, bool bf16_transposed,
                        cudaStream_t st, int64_t j0, int64_t jn) {
    const uint64_t s0 = seed ^ fnv1a64_host(name);
    if (jn < 0) jn = cols - j0;
    const int64_t n = rows * jn;
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), kNumSMs * 16));
    init_tensor_kernel<<<grid, 256, 0, st>>>(s0, rows, cols, j0, jn, std_, dst, ld, col_off,
                                             bf16_transposed ? 1 : 0);
    KEEP_LAUNCH_CHECK();
}

__global__ void pack_heads_kernel(const uint32_t* __restrict__ recv, int G, int cpr, int m, int wpr,
                                  uint32_t* __restrict__ rows) {
    // wpr = 32-bit words per (row, rank) slice
    const int64_t total = int64_t(m) * G * wpr;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int w = int(e % wpr);
        const int64_t rs = e / wpr;
        const int s = int(rs % G), i = int(rs / G);
        rows[e] = recv[(int64_t(s) * cpr + i) * wpr + w];
    }
}

void launch_pack_heads(const void* recv, int G, int cpr, int m, int dl, int es, void* rows, cudaStream_t st) {
    if (m <= 0) return;
    const int wpr = dl * es / 4;
    const int64_t total = int64_t(m) * G * wpr;
    pack_heads_kernel<<<unsigned(std::min<int64_t>(ceil_div(total, 256), kNumSMs * 8)), 256, 0, st>>>(
        static_cast<const uint32_t*>(recv), G, cpr, m, wpr, static_cast<uint32_t*>(rows));
    KEEP_LAUNCH_CHECK();
}

// Batched device copy: entry e moves bytes[e] (a multiple of 16) from src[e]
// to dst[e]; one CTA per entry, 16-byte vectors (in-place refresh scatter).
__global__ void batch_copy_kernel(const int4* const* __restrict__ src, int4* const* __restrict__ dst,
                                  const int64_t* __restrict__ bytes, int n) {
    for (int e = blockIdx.x; e < n; e += gridDim.x) {
        const int4* s = src[e];
        int4* d = dst[e];
        const int64_t nv = bytes[e] >> 4;
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) d[i] = s[i];
    }
}

void launch_batch_copy(const void* const* src, void* const* dst, const int64_t* bytes, int n, cudaStream_t st) {
    if (n <= 0) return;
    batch_copy_kernel<<<unsigned(std::min(n, kNumSMs * 16)), 256, 0, st>>>(
        reinterpret_cast<const int4* const*>(src), reinterpret_cast<int4* const*>(dst), bytes, n);
    KEEP_LAUNCH_CHECK();
}

// Host -> device upload through the kernel's parameter block (<= 31 KB per
// launch): the bytes travel with the launch, not through a copy engine, so a
// small upload never queues behind the layer loads streaming on the copy
// engines, and it never synchronises the host with the stream (pageable
// cudaMemcpyAsync does both).
template <int W>  // 32-bit words carried by one launch
struct ParamBlob {
    uint32_t w[W];
};
template <int W>
__global__ void param_copy_kernel(uint8_t* __restrict__ dst, const __grid_constant__ ParamBlob<W> blob, int n) {
    const int nw = n >> 2;
    if ((reinterpret_cast<uintptr_t>(dst) & 3) == 0) {
        uint32_t* d = reinterpret_cast<uint32_t*>(dst);
        for (int i = threadIdx.x; i < nw; i += blockDim.x) d[i] = blob.w[i];
        for (int i = (nw << 2) + threadIdx.x; i < n; i += blockDim.x)
            dst[i] = reinterpret_cast<const uint8_t*>(blob.w)[i];
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = reinterpret_cast<const uint8_t*>(blob.w)[i];
    }
}

template <int W>
void param_upload(uint8_t* dst, const uint8_t* src, int m, cudaStream_t st) {
    static thread_local ParamBlob<W> blob;
    std::memcpy(blob.w, src, size_t(m));
    param_copy_kernel<W><<<1, 256, 0, st>>>(dst, blob, m);
    KEEP_LAUNCH_CHECK();
}

void upload_bytes(void* dst, const void* src, size_t n, cudaStream_t st) {
    constexpr size_t kMax = 31 * 1024;  // the kernel parameter limit is 32,764 bytes
    for (size_t off = 0; off < n; off += kMax) {
        const int m = int(std::min(n - off, kMax));
        uint8_t* d = static_cast<uint8_t*>(dst) + off;
        const uint8_t* h = static_cast<const uint8_t*>(src) + off;
        // (the launch carries the whole parameter block: size it to the data)
        if (m <= 256) param_upload<64>(d, h, m, st);
        else if (m <= 4096) param_upload<1024>(d, h, m, st);
        else param_upload<int(kMax / 4)>(d, h, m, st);
    }
}

// Two contiguous device copies with the pointers passed by value (no upload,
// no copy engine: small copies issued while the copy engines stream a layer).
__global__ void copy2_kernel(int4* __restrict__ d0, const int4* __restrict__ s0, int4* __restrict__ d1,
                             const int4* __restrict__ s1, int64_t nv) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < 2 * nv; i += int64_t(gridDim.x) * blockDim.x) {
        if (i < nv) d0[i] = s0[i];
        else d1[i - nv] = s1[i - nv];
    }
}

void launch_copy2(void* d0, const void* s0, void* d1, const void* s1, int64_t bytes, cudaStream_t st) {
    if (bytes <= 0) return;
    if (bytes % 16) raise(KEEP_ERR_CONFIG, "copy2: size not a multiple of 16 bytes");
    const int64_t nv = bytes / 16;
    copy2_kernel<<<unsigned(std::min<int64_t>(ceil_div(2 * nv, 256), kNumSMs * 4)), 256, 0, st>>>(
        static_cast<int4*>(d0), static_cast<const int4*>(s0), static_cast<int4*>(d1), static_cast<const int4*>(s1), nv);
    KEEP_LAUNCH_CHECK();
}

// ======================================================================= K1 ==
__global__ void embed_kernel(const float* __restrict__ embed, const int32_t* __restrict__ tokens,
                             const int32_t* __restrict__ rows, int64_t n, int d,
                             float* __restrict__ x) {
    const int vec = d / 4;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        const float4* src = reinterpret_cast<const float4*>(embed + int64_t(tokens[rows[r]]) * d);
        float4* dst = reinterpret_cast<float4*>(x + r * d);
        for (int c = threadIdx.x; c < vec; c += blockDim.x) dst[c] = src[c];
    }
}

void launch_embed(const float* embed, const int32_t* tokens, const int32_t* rows, int64_t n, int d,
                  float* x, cudaStream_t st) {
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>(n, kNumSMs * 8));
    embed_kernel<<<grid, 256, 0, st>>>(embed, tokens, rows, n, d, x);
    KEEP_LAUNCH_CHECK();
}

__global__ void gather_rows_kernel(const float* __restrict__ src, const int32_t* __restrict__ idx,
                                   int64_t n, int d, float* __restrict__ dst,
                                   __nv_bfloat16* __restrict__ dstb) {
    const int vec = d / 4;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        const float4* s = reinterpret_cast<const float4*>(src + int64_t(idx[r]) * d);
        float4* o = reinterpret_cast<float4*>(dst + r * d);
        for (int c = threadIdx.x; c < vec; c += blockDim.x) {
            const float4 v = s[c];
            o[c] = v;
            if (dstb) {
                __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(dstb + r * d + 4 * c);
                ob[0] = __floats2bfloat162_rn(v.x, v.y);
                ob[1] = __floats2bfloat162_rn(v.z, v.w);
            }
        }
    }
}

void launch_gather_rows(const float* src, const int32_t* idx, int64_t n, int d, float* dst,
                        __nv_bfloat16* dst_bf16, cudaStream_t st) {
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>(n, kNumSMs * 8));
    gather_rows_kernel<<<grid, 256, 0, st>>>(src, idx, n, d, dst, dst_bf16);
    KEEP_LAUNCH_CHECK();
}

__global__ void to_bf16_kernel(const float* __restrict__ src, int64_t n4, __nv_bfloat16* __restrict__ dst) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(src)[i];
        __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(dst + 4 * i);
        o[0] = __floats2bfloat162_rn(v.x, v.y);
        o[1] = __floats2bfloat162_rn(v.z, v.w);
    }
}

void launch_to_bf16(const float* src, int64_t n, __nv_bfloat16* dst, cudaStream_t st) {
    if (n == 0) return;
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n / 4, 256), kNumSMs * 8));
    to_bf16_kernel<<<grid, 256, 0, st>>>(src, n / 4, dst);
    KEEP_LAUNCH_CHECK();
}

// ======================================================================= K4 ==
// One CTA per (entry, 16-row chunk); 16-byte vector copies of K and V rows.
__global__ void copy_cached_kernel(const void* const* __restrict__ ksrc,
                                   const void* const* __restrict__ vsrc,
                                   const int32_t* __restrict__ dst_row, const int32_t* __restrict__ nrows,
                                   int64_t row_bytes, uint8_t* __restrict__ kdst,
                                   uint8_t* __restrict__ vdst) {
    const int e = blockIdx.x;
    const int r0 = blockIdx.y * 16;
    const int nr = nrows[e];
    if (r0 >= nr) return;
    const int r1 = min(nr, r0 + 16);
    const int64_t vec = row_bytes / 16;
    const uint4* ks = static_cast<const uint4*>(ksrc[e]);
    const uint4* vs = static_cast<const uint4*>(vsrc[e]);
    uint4* kd = reinterpret_cast<uint4*>(kdst + int64_t(dst_row[e]) * row_bytes);
    uint4* vd = reinterpret_cast<uint4*>(vdst + int64_t(dst_row[e]) * row_bytes);
    const int64_t total = int64_t(r1 - r0) * vec, base = int64_t(r0) * vec;
    // four 16-byte loads of K and four of V in flight per thread before the
    // stores (the copy is latency-bound otherwise: ~10 rows per CTA)
    constexpr int U = 4;
    int64_t i = threadIdx.x;
    for (; i + (U - 1) * int64_t(blockDim.x) < total; i += U * int64_t(blockDim.x)) {
        uint4 k[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            k[u] = __ldg(ks + base + i + u * blockDim.x);
            v[u] = __ldg(vs + base + i + u * blockDim.x);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            kd[base + i + u * blockDim.x] = k[u];
            vd[base + i + u * blockDim.x] = v[u];
        }
    }
    for (; i < total; i += blockDim.x) {
        kd[base + i] = ks[base + i];
        vd[base + i] = vs[base + i];
    }
}

void launch_copy_cached(const void* const* ksrc, const void* const* vsrc, const int32_t* dst_row,
                        const int32_t* nrows, int n_entries, int64_t row_bytes, void* kdst,
                        void* vdst, int max_rows, cudaStream_t st) {
    if (n_entries == 0) return;
    dim3 grid(n_entries, static_cast<unsigned>(ceil_div(max_rows, 16)));
    copy_cached_kernel<<<grid, 256, 0, st>>>(ksrc, vsrc, dst_row, nrows, row_bytes,
                                             static_cast<uint8_t*>(kdst), static_cast<uint8_t*>(vdst));
    KEEP_LAUNCH_CHECK();
}

// ======================================================================= K6 ==
// sts[src][dst] = (sum over compact rows of src, in row order, of
// rowbin[row][dst]) / seg_len[src] for dst < src; qts[dst] likewise over the
// query rows / qlen (prefill.hpp:281-288, 306-315).  Inactive sources and the
// upper triangle are zero.
template <typename TB>
__global__ void summary_reduce_kernel(const TB* __restrict__ rowbin, int S,
                                      const int32_t* __restrict__ seg_cbeg,
                                      const int32_t* __restrict__ seg_cend,
                                      const int32_t* __restrict__ seg_len, int q_cbeg, int q_cend,
                                      int qlen, double* __restrict__ summ) {
    const int src = blockIdx.y - 1;  // -1 = the query row block
    double* out = src < 0 ? summ : summ + S + int64_t(src) * S;
    int cb, ce;
    double denom;
    if (src < 0) {
        cb = q_cbeg;
        ce = q_cend;
        denom = double(qlen);
    } else {
        cb = seg_cbeg[src];
        ce = seg_cend[src];
        denom = double(seg_len[src]);
    }
    for (int dst = blockIdx.x * blockDim.x + threadIdx.x; dst < S; dst += gridDim.x * blockDim.x) {
        double acc = 0.0;
        const bool live = (src < 0) ? (qlen > 0) : (dst < src);
        if (live)
            for (int r = cb; r < ce; ++r) acc += double(rowbin[int64_t(r) * S + dst]);
        out[dst] = live ? acc / denom : 0.0;
    }
}

template <typename TB>
void launch_summary_reduce(const TB* rowbin, int S, const int32_t* seg_cbeg, const int32_t* seg_cend,
                           const int32_t* seg_len, int q_cbeg, int q_cend, int qlen, double* summ,
                           cudaStream_t st) {
    dim3 grid(static_cast<unsigned>(ceil_div(S, 256)), S + 1);
    summary_reduce_kernel<TB><<<grid, 256, 0, st>>>(rowbin, S, seg_cbeg, seg_cend, seg_len, q_cbeg,
                                                    q_cend, qlen, summ);
    KEEP_LAUNCH_CHECK();
}
template void launch_summary_reduce<double>(const double*, int, const int32_t*, const int32_t*,
                                            const int32_t*, int, int, int, double*, cudaStream_t);
template void launch_summary_reduce<float>(const float*, int, const int32_t*, const int32_t*,
                                           const int32_t*, int, int, int, double*, cudaStream_t);

// ======================================================================= K7 ==
// converge (recompute.hpp:86-138) as one persistent CTA.  Column sums of the
// relevant set are kept incrementally (O(S) per hop instead of O(S*|R|));
// because the reference re-sums in ascending position, each hop arbitrates
// exactly: a forward error bound on the incremental sums yields the set of
// positions that could be the reference's pick, and when that set is not a
// single clear winner those positions are re-summed in the reference's order
// and compared with the reference's rule (strict >, lowest position, > 0).
constexpr int kSelThreads = 512;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelMaxS = 28 * kSelThreads;  // positions per thread <= 28 (bitmask)

// One hop's reduction in a single pass: the best lower bound (ties -> lower
// position) and the two largest upper bounds (with the position of the
// largest), so a unique winner is recognised without a second pass.
struct HopRed {
    double lo;  // best lower bound
    int i;      // its position (-1: none)
    double hi1; // largest upper bound
    int hi1_i;
    double hi2; // second largest upper bound
};

__device__ __forceinline__ HopRed hop_combine(HopRed a, HopRed b) {
    HopRed r;
    // best lower bound: larger wins, equal -> lower position
    if (b.i >= 0 && (a.i < 0 || b.lo > a.lo || (b.lo == a.lo && b.i < a.i))) {
        r.lo = b.lo;
        r.i = b.i;
    } else {
        r.lo = a.lo;
        r.i = a.i;
    }
    // top-2 upper bounds
    if (b.hi1 > a.hi1 || (b.hi1 == a.hi1 && b.hi1_i >= 0 && (a.hi1_i < 0 || b.hi1_i < a.hi1_i))) {
        r.hi1 = b.hi1;
        r.hi1_i = b.hi1_i;
        r.hi2 = fmax(a.hi1, b.hi2);
    } else {
        r.hi1 = a.hi1;
        r.hi1_i = a.hi1_i;
        r.hi2 = fmax(b.hi1, a.hi2);
    }
    return r;
}

__device__ __forceinline__ HopRed hop_shfl(HopRed x, int o) {
    HopRed y;
    y.lo = __shfl_xor_sync(0xffffffffu, x.lo, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    y.hi1 = __shfl_xor_sync(0xffffffffu, x.hi1, o);
    y.hi1_i = __shfl_xor_sync(0xffffffffu, x.hi1_i, o);
    y.hi2 = __shfl_xor_sync(0xffffffffu, x.hi2, o);
    return y;
}

__device__ HopRed block_hop_reduce(HopRed x, HopRed* scratch) {
    for (int o = 16; o > 0; o >>= 1) x = hop_combine(x, hop_shfl(x, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) scratch[w] = x;
    __syncthreads();
    if (w == 0) {
        x = l < kSelWarps ? scratch[l] : HopRed{0.0, -1, -INFINITY, -1, -INFINITY};
        for (int o = 16; o > 0; o >>= 1) x = hop_combine(x, hop_shfl(x, o));
        if (l == 0) scratch[kSelWarps] = x;
    }
    __syncthreads();
    return scratch[kSelWarps];
}

// State per position in shared memory: the incremental column sum over the
// relevant set (fp64), an fp32 upper bound of its absolute terms (the error
// radius of the sum), and a membership flag; the candidate mask of a thread's
// positions (tid + k * 512) is a register bitmask.
__device__ __forceinline__ void select_impl(int S, const double* __restrict__ qts, const double* __restrict__ sts,
                                            int64_t budget, const uint8_t* __restrict__ cand,
                                            int32_t* __restrict__ order, int32_t* n_out, int32_t* hops_out,
                                            int hop_cap) {
    extern __shared__ __align__(16) uint8_t sraw[];
    double* colsum = reinterpret_cast<double*>(sraw);               // [S]
    float* colabs = reinterpret_cast<float*>(colsum + S);           // [S]
    uint8_t* member = reinterpret_cast<uint8_t*>(colabs + S);       // [S] in the relevant set
    __shared__ HopRed red[kSelWarps + 1];

    const int items = int(ceil_div(S, kSelThreads));
    uint32_t allowed = 0;
    for (int k = 0; k < items; ++k) {
        const int i = threadIdx.x + k * kSelThreads;
        if (i < S && (cand == nullptr || cand[i] != 0)) allowed |= 1u << k;
        if (i < S) {
            colsum[i] = 0.0;
            colabs[i] = 0.f;
            member[i] = 0;
        }
    }
    __syncthreads();
    const double u = 0x1.0p-53;
    int n = 0, hop = 0;
    // score of position i and the radius within which the reference's
    // ascending re-sum can differ from the incremental one
    auto score_of = [&](int i, double& sc, double& err) {
        if (n == 0) {
            sc = qts[i];
            err = 0.0;
        } else {
            sc = colsum[i] / double(n);
            // colabs is rounded to fp32: inflate by 2^-20 to keep it an upper bound
            err = (2.0 * (n + 2)) * u * (double(colabs[i]) * (1.0 + 0x1.0p-20) / double(n)) + 4.0 * u * fabs(sc);
        }
    };
    // hop_cap = S: the reference's walk (recompute.hpp:133); smaller: the capped variant
    while (int64_t(n) < budget && hop < hop_cap) {
        HopRed x{0.0, -1, -INFINITY, -1, -INFINITY};
        for (int k = 0; k < items; ++k) {
            if (!(allowed >> k & 1u)) continue;
            const int i = threadIdx.x + k * kSelThreads;
            double sc, err;
            score_of(i, sc, err);
            const double up = sc + err;
            if (!(up > 0.0)) continue;  // can never be a strictly positive pick
            x = hop_combine(x, HopRed{sc - err, i, up, i, -INFINITY});
        }
        const HopRed r = block_hop_reduce(x, red);
        ++hop;
        if (r.i < 0) break;  // nothing can be strictly positive: stalled hop (recompute.hpp:124)
        // unique winner: its lower bound beats every other position's upper bound
        const double other_hi = r.hi1_i == r.i ? r.hi2 : r.hi1;
        int win;
        if (r.lo > 0.0 && r.lo > other_hi) {
            win = r.i;
        } else {
            // exact arbitration among the positions that could win: the
            // reference's ascending-position re-sum and its rule (strict >,
            // lowest position, > 0)
            HopRed ex{0.0, -1, -INFINITY, -1, -INFINITY};
            for (int k = 0; k < items; ++k) {
                if (!(allowed >> k & 1u)) continue;
                const int i = threadIdx.x + k * kSelThreads;
                double sc, err;
                score_of(i, sc, err);
                if (!(sc + err > 0.0 && sc + err >= r.lo)) continue;
                double v;
                if (n == 0) {
                    v = qts[i];
                } else {
                    double acc = 0.0;
                    for (int m = 0; m < S; ++m)
                        if (member[m]) acc += sts[int64_t(m) * S + i];
                    v = acc / double(n);
                }
                if (v > 0.0) ex = hop_combine(ex, HopRed{v, i, -INFINITY, -1, -INFINITY});
            }
            const HopRed w = block_hop_reduce(ex, red);
            win = w.i;
        }
        if (win < 0) break;  // the stalled hop still counts
        if (threadIdx.x == 0) {
            order[n] = win;
            member[win] = 1;
        }
        ++n;
        // fold the new member's row into the column sums (insertion order)
        const double* row = sts + int64_t(win) * S;
        for (int k = 0; k < items; ++k) {
            const int i = threadIdx.x + k * kSelThreads;
            if (i == win) allowed &= ~(1u << k);
            if (!(allowed >> k & 1u)) continue;
            const double t = row[i];
            colsum[i] += t;
            colabs[i] = __fadd_ru(colabs[i], __double2float_ru(fabs(t)));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_out = n;
        *hops_out = hop;
    }
}

__global__ void __launch_bounds__(kSelThreads, 1)
select_kernel(int S, const double* __restrict__ qts, const double* __restrict__ sts, int64_t budget,
              const uint8_t* __restrict__ cand, int32_t* __restrict__ order, int32_t* n_out,
              int32_t* hops_out, int hop_cap) {
    select_impl(S, qts, sts, budget, cand, order, n_out, hops_out, hop_cap);
}

// One walk per CTA (batched queries): CTA b reads summ[b] ([S] qts then
// [S x S] sts), candidates cand + b*S and writes out + b*(S+2) as
// {n, hops, order...}; CTAs with run[b] == 0 exit.
__global__ void __launch_bounds__(kSelThreads, 1)
select_batch_kernel(int S, const double* const* __restrict__ summ, int64_t budget, const uint8_t* __restrict__ cand,
                    const uint8_t* __restrict__ run, int32_t* __restrict__ out, int hop_cap) {
    const int b = blockIdx.x;
    if (!run[b]) return;
    const double* sm = summ[b];
    int32_t* o = out + int64_t(b) * (S + 2);
    select_impl(S, sm, sm + S, budget, cand + int64_t(b) * S, o + 2, o, o + 1, hop_cap);
}

static int hop_cap_of(int S, int max_hops) { return max_hops > 0 ? std::min(S, max_hops) : S; }

void launch_select_batch(int S, int B, const double* const* summ, int64_t budget, const uint8_t* cand,
                         const uint8_t* run, int32_t* out, cudaStream_t st, int max_hops) {
    if (S > kSelMaxS) raise(KEEP_ERR_CONFIG, "selector supports at most 14336 segments");
    const size_t smem = size_t(std::max(S, 1)) * (8 + 4 + 1) + 16;
    if (smem > 48 * 1024)
        KEEP_CUDA(cudaFuncSetAttribute(select_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    select_batch_kernel<<<B, kSelThreads, smem, st>>>(S, summ, budget, cand, run, out, hop_cap_of(S, max_hops));
    KEEP_LAUNCH_CHECK();
}

// single-hop ablation (recompute.hpp:166-176): the live segments stable-sorted
// by qts descending, the first `budget` kept -- as a rank per segment:
// rank(i) = #{live j : qts[j] > qts[i], or qts[j] == qts[i] and j < i}
__global__ void single_hop_kernel(const double* __restrict__ qts, const uint8_t* __restrict__ live, int S,
                                  int64_t budget, uint8_t* __restrict__ next) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
        if (!live[i]) {
            next[i] = 0;
            continue;
        }
        const double q = qts[i];
        int64_t rank = 0;
        for (int j = 0; j < S; ++j) rank += live[j] && (qts[j] > q || (qts[j] == q && j < i));
        next[i] = rank < budget ? 1 : 0;
    }
}

void launch_single_hop(const double* qts, const uint8_t* live, int S, int64_t budget, uint8_t* next,
                       cudaStream_t st) {
    single_hop_kernel<<<unsigned(std::max(1, std::min(int(ceil_div(S, 128)), kNumSMs * 4))), 128, 0, st>>>(
        qts, live, S, budget, next);
    KEEP_LAUNCH_CHECK();
}

void launch_select(int S, const double* qts, const double* sts, int64_t budget,
                   const uint8_t* candidates, int32_t* order, int32_t* n_out, int32_t* hops_out,
                   cudaStream_t st, int max_hops) {
    if (S > kSelMaxS) raise(KEEP_ERR_CONFIG, "selector supports at most 14336 segments");
    const size_t smem = size_t(std::max(S, 1)) * (8 + 4 + 1) + 16;
    if (smem > 48 * 1024)
        KEEP_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    select_kernel<<<1, kSelThreads, smem, st>>>(S, qts, sts, budget, candidates, order, n_out, hops_out,
                                                hop_cap_of(S, max_hops));
    KEEP_LAUNCH_CHECK();
}

// ====================================================================== K11 ==
__global__ void logits_kernel(const float* __restrict__ row, const float* __restrict__ unembed, int d,
                              int V, double* __restrict__ out) {
    extern __shared__ float srow[];
    for (int i = threadIdx.x; i < d; i += blockDim.x) srow[i] = row[i];
    __syncthreads();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc = fma(double(srow[i]), double(unembed[int64_t(i) * V + j]), acc);
    out[j] = acc;
}

// divergence (prefill.hpp:501-531): L2 of the row difference and the
// symmetric KL of softmax(logits_a) vs softmax(logits_b), fp64 throughout,
// the reference's formula per element (log of an underflowed p is -inf and
// propagates exactly as there).  One CTA; block reductions in fixed order.
__device__ double block_reduce_d(double v, double* sh, bool is_max) {
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, w) : v + w;
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < int(blockDim.x >> 5) ? sh[lane] : (is_max ? -INFINITY : 0.0);
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmax(v, w) : v + w;
        }
        if (lane == 0) sh[32] = v;
    }
    __syncthreads();
    return sh[32];
}

__global__ void __launch_bounds__(1024) divergence_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                          int d, const double* __restrict__ la,
                                                          const double* __restrict__ lb, int V, double* __restrict__ out) {
    __shared__ double sh[33];
    double acc = 0.0;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        const double delta = double(a[j]) - double(b[j]);
        acc += delta * delta;
    }
    const double l2 = sqrt(block_reduce_d(acc, sh, false));
    double ma = -INFINITY, mb = -INFINITY;
    for (int j = threadIdx.x; j < V; j += blockDim.x) {
        ma = fmax(ma, la[j]);
        mb = fmax(mb, lb[j]);
    }
    ma = block_reduce_d(ma, sh, true);
    mb = block_reduce_d(mb, sh, true);
    double sa = 0.0, sb = 0.0;
    for (int j = threadIdx.x; j < V; j += blockDim.x) {
        sa += exp(la[j] - ma);
        sb += exp(lb[j] - mb);
    }
    sa = block_reduce_d(sa, sh, false);
    sb = block_reduce_d(sb, sh, false);
    double kl = 0.0;
    for (int j = threadIdx.x; j < V; j += blockDim.x) {
        const double p = exp(la[j] - ma) / sa, q = exp(lb[j] - mb) / sb;
        kl += (p - q) * (log(p) - log(q));
    }
    kl = block_reduce_d(kl, sh, false);
    if (threadIdx.x == 0) {
        out[0] = l2;
        out[1] = kl;
    }
}

void launch_divergence(const float* a, const float* b, int d, const double* la, const double* lb, int V, double* out,
                       cudaStream_t st) {
    divergence_kernel<<<1, 1024, 0, st>>>(a, b, d, la, lb, V, out);
    KEEP_LAUNCH_CHECK();
}

// K11 for a batch of rows: the unembedding streams once for up to 16 rows;
// each logit is the same fp64 fma chain in ascending i as logits_kernel.
__global__ void logits_multi_kernel(const float* __restrict__ rows, int B, const float* __restrict__ unembed, int d,
                                    int V, double* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    double acc[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) acc[b] = 0.0;
    for (int i = 0; i < d; ++i) {
        const double u = double(unembed[int64_t(i) * V + j]);
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (b < B) acc[b] = fma(double(__ldg(rows + int64_t(b) * d + i)), u, acc[b]);
    }
#pragma unroll
    for (int b = 0; b < 16; ++b)
        if (b < B) out[int64_t(b) * V + j] = acc[b];
}

void launch_logits_multi(const float* rows, int B, const float* unembed, int d, int V, double* out, cudaStream_t st) {
    for (int b0 = 0; b0 < B; b0 += 16) {
        const int nb = std::min(16, B - b0);
        logits_multi_kernel<<<static_cast<unsigned>(ceil_div(V, 128)), 128, 0, st>>>(rows + int64_t(b0) * d, nb, unembed,
                                                                                     d, V, out + int64_t(b0) * V);
        KEEP_LAUNCH_CHECK();
    }
}

void launch_logits(const float* row, const float* unembed, int d, int V, double* out, cudaStream_t st) {
    logits_kernel<<<static_cast<unsigned>(ceil_div(V, 128)), 128, sizeof(float) * d, st>>>(row, unembed, d, V, out);
    KEEP_LAUNCH_CHECK();
}

// ================================================================ RoPE hook ==
// north_star subsystem (3): "the RoPE position re-shift of reused blocks".  The
// reference architecture is NoPE (model.hpp:3-8), so this is an
// opt-in hook (keep_set_rope), off -- the identity -- in every parity run.
// Rotary pairs are (2j, 2j + 1) inside each head, angle = pos * theta^(-2j/dh),
// computed in fp64.  Canonical KV is rotated at owner-local positions (a
// segment_prefill starts at 0); a reused block is re-shifted by its layout
// offset when it is copied into the merged KV.
namespace {
template <typename T> __device__ __forceinline__ float ldv(const T* p);
template <> __device__ __forceinline__ float ldv<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ldv<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void stv(float* p, double v) { *p = float(v); }
__device__ __forceinline__ void stv(__nv_bfloat16* p, double v) { *p = __float2bfloat16_rn(float(v)); }

template <typename T>
__device__ __forceinline__ void rotate_pair(T* x, int j, int dh, double pos, double theta) {
    const double ang = pos * pow(theta, -2.0 * j / dh);
    double sn, cs;
    sincos(ang, &sn, &cs);
    const double a = ldv(x), b = ldv(x + 1);
    stv(x, a * cs - b * sn);
    stv(x + 1, a * sn + b * cs);
}

// q[i] (compact) and k[rows[i]] (merged) at position rows[i] - key_lo[rows[i]]
template <typename T>
__global__ void rope_qk_kernel(T* q, T* k, int n, const int32_t* rows, const int32_t* key_lo, int dl, int dh,
                               double theta) {
    const int pairs = dl / 2;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(n) * pairs;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(e / pairs), pr = int(e % pairs);
        const int col = 2 * pr, j = (col % dh) / 2;
        const int r = rows[i];
        const double pos = double(r - (key_lo ? key_lo[r] : 0));
        rotate_pair(q + int64_t(i) * dl + col, j, dh, pos, theta);
        rotate_pair(k + int64_t(r) * dl + col, j, dh, pos, theta);
    }
}

// re-shift cached key rows: entry e = (first merged row, rows, delta)
template <typename T>
__global__ void rope_shift_kernel(T* k, const int32_t* tab, int n_entries, int dl, int dh, double theta) {
    const int e = blockIdx.y;
    if (e >= n_entries) return;
    const int r0 = tab[3 * e], nr = tab[3 * e + 1], delta = tab[3 * e + 2];
    const int pairs = dl / 2;
    for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < int64_t(nr) * pairs;
         x += int64_t(gridDim.x) * blockDim.x) {
        const int rr = int(x / pairs), col = 2 * int(x % pairs);
        rotate_pair(k + int64_t(r0 + rr) * dl + col, (col % dh) / 2, dh, double(delta), theta);
    }
}
}  // namespace

void launch_rope_qk(void* q, void* k, int n, const int32_t* rows, const int32_t* key_lo, int dl, int dh, double theta,
                    bool bf16, cudaStream_t st) {
    if (n == 0) return;
    const unsigned grid = unsigned(std::min<int64_t>(ceil_div(int64_t(n) * dl / 2, 256), kNumSMs * 8));
    if (bf16)
        rope_qk_kernel<<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(k), n, rows,
                                             key_lo, dl, dh, theta);
    else
        rope_qk_kernel<<<grid, 256, 0, st>>>(static_cast<float*>(q), static_cast<float*>(k), n, rows, key_lo, dl, dh,
                                             theta);
    KEEP_LAUNCH_CHECK();
}

void launch_rope_shift(void* k, const int32_t* tab, int n_entries, int max_rows, int dl, int dh, double theta,
                       bool bf16, cudaStream_t st) {
    if (n_entries == 0) return;
    const dim3 grid(unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(int64_t(max_rows) * dl / 2, 256), 64))),
                    unsigned(n_entries));
    if (bf16) rope_shift_kernel<<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(k), tab, n_entries, dl, dh, theta);
    else rope_shift_kernel<<<grid, 256, 0, st>>>(static_cast<float*>(k), tab, n_entries, dl, dh, theta);
    KEEP_LAUNCH_CHECK();
}

}  // namespace keep_b200
