// common.cuh -- shared definitions for the KEEP B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <stdexcept>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "keep_b200.h"

namespace keep_b200 {

// Error taxonomy of the reference (errors.hpp:8-26) plus device failures.
struct KeepError : std::runtime_error {
    int code;
    KeepError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline void raise(int code, const std::string& msg) { throw KeepError(code, msg); }

#define KEEP_CUDA(expr)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            ::keep_b200::raise(KEEP_ERR_CUDA, std::string(#expr) + ": " +               \
                                                  cudaGetErrorString(e_));               \
    } while (0)

// KEEP_SYNC_DEBUG=1: synchronise and trace after every launch (bring-up aid)
bool sync_debug();
void trace_launch(const char* file, int line);
#define KEEP_LAUNCH_CHECK()                                                \
    do {                                                                   \
        KEEP_CUDA(cudaGetLastError());                                     \
        if (::keep_b200::sync_debug()) ::keep_b200::trace_launch(__FILE__, __LINE__); \
    } while (0)

constexpr int kNumSMs = 148;

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current
// device only: set it once per (kernel, device), thread-safe.
void set_smem_attr(const void* fn, int bytes);
template <typename F>
inline void smem_attr(F* fn, int bytes) { set_smem_attr(reinterpret_cast<const void*>(fn), bytes); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- layouts --
// Device weight layouts (one context holds exactly one of them):
//  PARITY: fp32 row-major [K x N] exactly as the reference Mat (x . W),
//          with the three projections fused column-wise: wqkv [d x 3d].
//  FAST:   bf16 transposed [N x K] (K-major rows = the tcgen05 B operand),
//          wqkv_t [3d x d], wo_t [d x d], win_t [f x d], wout_t [d x f].
enum WeightSlot { W_QKV = 0, W_O = 1, W_IN = 2, W_OUT = 3 };

}  // namespace keep_b200
