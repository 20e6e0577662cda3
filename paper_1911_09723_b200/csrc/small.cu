// small.cu — SpMM for calls with few columns (batch 1, small planes).
//
// The tile kernel stages a [K][T] activation tile per CTA and runs a row-group
// stream per warp; with a few hundred columns (BASELINE configs[0] and the
// batch-1 MobileNet stack) there are fewer tiles than SMs and every CTA pays
// its staging / ring-fill / epilogue latency once for little work. Here one
// warp owns one block row x 32 virtual columns (lane = column): it reads the
// row's stored blocks once (coalesced, 32 at a time — the first 32 from a
// per-row head table, so they do not wait for row_ptr — then broadcast with
// shuffles) and gathers each block's activation straight from global memory
// (one coalesced 128 B row segment per block, L1/L2-resident at these sizes).
// There is no shared-memory staging and no CTA barrier, and the grid has
// (block rows) x (column groups) warps, enough to fill the GPU.
//
// Arithmetic per output is the reference strip kernels' (kernels.cpp:14-43,
// 101-130): acc = bias (or +0), then value * act for the stored blocks in
// ascending position, separately rounded in strict mode, then the ternary
// clamp (tensor.hpp:90-96) and the optional residual add (netdef.cpp:448-452).
#include <cuda_runtime.h>

#include "spcv_internal.h"

namespace spcvk {

struct SmallArgs {
    const float* act;         // [images][K_img][S]
    float* out;               // [images][M_out][S]
    const float* bias;        // [M] or nullptr
    const float* residual;    // [images][M_out][S] or nullptr
    const uint32_t* row_ptr;  // [brows + 1]
    const uint32_t* col_idx;  // [nblocks]
    const float* values;      // [nblocks][BH]
    const uint32_t* head_col; // [brows][32]: each block row's first 32 column indices (~0u past its end)
    const float* head_val;    // [brows][32][BH]: their values (0 past the end)
    long long N;              // images * S
    int S, K_img, M_out, brows;
    int act_kind;
    float lo, hi;
};

template <bool STRICT>
__device__ __forceinline__ float madd_s(float acc, float w, float x) {
    if constexpr (STRICT) {
        return __fadd_rn(acc, __fmul_rn(w, x));
    } else {
        return fmaf(w, x, acc);
    }
}

constexpr int kSmallWarps = 4;  // block rows per CTA (same column group)
#ifndef SPCV_SMALL_NG
#define SPCV_SMALL_NG 8
#endif
constexpr int kGathers = SPCV_SMALL_NG;  // activation gathers in flight per warp

template <int BH, bool STRICT, bool RES>
__global__ void __launch_bounds__(kSmallWarps * 32)
spmm_small_kernel(const SmallArgs a) {
    const int lane = threadIdx.x & 31;
    const int br = blockIdx.y * kSmallWarps + (threadIdx.x >> 5);
    if (br >= a.brows) return;
    const long long n = static_cast<long long>(blockIdx.x) * 32 + lane;
    const bool valid = n < a.N;
    long long abase = 0, obase = 0;
    if (valid) {
        const long long img = n / a.S;
        const long long s = n - img * a.S;
        abase = img * a.K_img * a.S + s;
        obase = img * a.M_out * a.S + s;
    }
    const float* act = a.act + abase;
    // The row's first 32 blocks come from the head table when the matrix has
    // one (no dependency on row_ptr, loaded in the same round trip), else from
    // col_idx / values at row_ptr[br]; later groups of 32 from there too.
    const uint32_t rb = __ldg(a.row_ptr + br), re = __ldg(a.row_ptr + br + 1);
    uint32_t kcol;
    float wv[BH];
    if (a.head_col != nullptr) {
        const size_t h = static_cast<size_t>(br) * 32 + lane;
        kcol = __ldg(a.head_col + h);
#pragma unroll
        for (int i = 0; i < BH; ++i) wv[i] = __ldg(a.head_val + h * BH + i);
    } else {
        const bool mine = rb + lane < re;
        kcol = mine ? __ldg(a.col_idx + rb + lane) : 0u;
#pragma unroll
        for (int i = 0; i < BH; ++i) wv[i] = mine ? __ldg(a.values + static_cast<size_t>(rb + lane) * BH + i) : 0.0f;
    }
    float acc[BH];
#pragma unroll
    for (int i = 0; i < BH; ++i) {
        const int r = br * BH + i;
        acc[i] = (a.bias != nullptr && r < a.M_out) ? __ldg(a.bias + r) : 0.0f;
    }
    for (uint32_t t0 = rb;;) {
        const uint32_t cnt = min(32u, re - t0);
        // kGathers gathers in flight, then their products, in stored order
        for (uint32_t t = 0; t < cnt; t += kGathers) {
            float x[kGathers];
#pragma unroll
            for (int q = 0; q < kGathers; ++q) {
                const int k = __shfl_sync(0xffffffffu, static_cast<int>(kcol), (t + q) & 31);
                x[q] = (valid && t + q < cnt) ? __ldg(act + static_cast<long long>(k) * a.S) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kGathers; ++q) {
#pragma unroll
                for (int i = 0; i < BH; ++i) {
                    const float w = __shfl_sync(0xffffffffu, wv[i], (t + q) & 31);
                    if (t + q < cnt) acc[i] = madd_s<STRICT>(acc[i], w, x[q]);
                }
            }
        }
        t0 += 32;
        if (t0 >= re) break;
        const bool mine = t0 + lane < re;
        kcol = mine ? __ldg(a.col_idx + t0 + lane) : 0u;
#pragma unroll
        for (int i = 0; i < BH; ++i) wv[i] = mine ? __ldg(a.values + static_cast<size_t>(t0 + lane) * BH + i) : 0.0f;
    }
    if (!valid) return;
#pragma unroll
    for (int i = 0; i < BH; ++i) {
        const int r = br * BH + i;
        if (r >= a.M_out) continue;  // padded row: computed, never stored
        float v = acc[i];
        if (a.act_kind == 1) v = v < a.lo ? a.lo : (v > a.hi ? a.hi : v);
        const long long o = obase + static_cast<long long>(r) * a.S;
        if constexpr (RES) v = __fadd_rn(v, __ldcs(a.residual + o));
        __stcs(a.out + o, v);
    }
}

}  // namespace spcvk

namespace spcv_detail {

template <int BH>
static int launch_small_bh(const spcvk::SmallArgs& a, bool strict, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((a.N + 31) / 32),
                    static_cast<unsigned>((a.brows + spcvk::kSmallWarps - 1) / spcvk::kSmallWarps));
    const dim3 threads(spcvk::kSmallWarps * 32);
    auto kern = strict ? (a.residual ? spcvk::spmm_small_kernel<BH, true, true> : spcvk::spmm_small_kernel<BH, true, false>)
                       : (a.residual ? spcvk::spmm_small_kernel<BH, false, true> : spcvk::spmm_small_kernel<BH, false, false>);
    SPCV_CUDA(launch_kernel(kern, grid, threads, 0, st, a));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

int launch_small(const spcv_cu_weights* w, const spcvk::KernelArgs& k, bool strict, cudaStream_t st) {
    if (!w->d_row_ptr || !w->d_col_idx) return SPCV_ERR_UNSUPPORTED;
    if ((k.N + 31) / 32 > 0x7FFFFFFFLL || w->brows > 65535 * spcvk::kSmallWarps) return SPCV_ERR_UNSUPPORTED;
    spcvk::SmallArgs a;
    a.act = k.act;
    a.out = k.out;
    a.bias = k.bias;
    a.residual = k.residual;
    a.row_ptr = w->d_row_ptr;
    a.col_idx = w->d_col_idx;
    a.values = w->d_values;
    a.head_col = w->d_head_col;
    a.head_val = w->d_head_val;
    a.N = k.N;
    a.S = k.S;
    a.K_img = k.K_img;
    a.M_out = k.M_out;
    a.brows = w->brows;
    a.act_kind = k.act_kind;
    a.lo = k.lo;
    a.hi = k.hi;
    switch (w->block_h) {
        case 1: return launch_small_bh<1>(a, strict, st);
        case 2: return launch_small_bh<2>(a, strict, st);
        default: return launch_small_bh<4>(a, strict, st);
    }
}

}  // namespace spcv_detail
