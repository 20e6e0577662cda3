// spcv_internal.h — state and helpers shared by the C-ABI translation units
// (spcv_cu.cu: packing + entry points; launch_bh{1,2,4}.cu: kernel dispatch).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/spcv_cu.h"
#include "spmm_kernel.cuh"

struct spcv_cu_weights {
    int rows = 0, cols = 0, block_h = 1, brows = 0;
    int G = 1;           // block rows per warp group (32 / LPR)
    int LPR = 32;        // lanes per block row
    int NF = 4;          // float4 column quads per lane
    int T = 128;         // virtual columns per tile (LPR * NF * 4)
    int STEPS = 4;       // steps per chunk of the weight stream (2 or 4)
    int device = 0;
    size_t nblocks = 0;
    size_t nchunks = 0;
    // paper-format streams (north_star): counts, deltas, values
    uint32_t* d_nnz = nullptr;
    uint32_t* d_delta = nullptr;
    float* d_values = nullptr;
    // execution schedule
    uint4* d_stream = nullptr;
    uint32_t* d_bin_beg = nullptr;
};

namespace spcv_detail {

extern std::atomic<uint64_t> g_launches;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kTwoCtaSmem = 112 * 1024;

// Shared memory of one CTA of the tile kernel: [K+1][T] activation tile (row
// K = zeros for padded steps) + T int64 output column offsets + bias[M].
inline size_t smem_bytes(int K, int M, int T) {
    return static_cast<size_t>(K + 1) * T * 4 + static_cast<size_t>(T) * 8 +
           static_cast<size_t>(M) * 4;
}

// Kernel dispatch for one block height (launch_bh{1,2,4}.cu).
int launch_bh1(const spcvk::KernelArgs&, const spcv_cu_weights*, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t);
int launch_bh2(const spcvk::KernelArgs&, const spcv_cu_weights*, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t);
int launch_bh4(const spcvk::KernelArgs&, const spcv_cu_weights*, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t);

}  // namespace spcv_detail

#define SPCV_CUDA(call)                                                         \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess) return spcv_detail::cuda_fail(e_, #call);        \
    } while (0)
