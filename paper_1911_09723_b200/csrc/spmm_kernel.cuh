// spmm_kernel.cuh — sm_100a SpMM kernel for sparse 1x1 convolutions.
//
// Replaces the reference strip microkernels spmm_strip_scalar / spmm_strip_vector
// (/root/reference/proj/src/kernels.cpp:14-43, 101-130) and their strip loop
// (kernels.cpp:324-333). Same per-element arithmetic:
//   acc = bias[r]  (or +0.0)                         kernels.cpp:21,110
//   for stored blocks of r's block row, ascending:   kernels.cpp:25,114
//       acc += value * act[col][s]                   kernels.cpp:30,120
//   out = clamp(acc) with the ternary compare        kernels.cpp:38, 93-99
//
// B200 mapping:
//  * The column dimension N = images x H*W ("virtual columns") is cut into
//    tiles of T = 4*32/G columns; one CTA owns one tile and stages the whole
//    [K][T] activation block into shared memory once (cp.async, 16 B vectors
//    when H*W % 4 == 0). Every output row of the tile is then produced from
//    shared memory, so each activation byte crosses HBM exactly once.
//  * A warp works on G block rows at a time (a "row group"); each block row
//    owns 32/G lanes, each lane owns 4 consecutive virtual columns (float4).
//    One activation LDS.128 per stored block feeds 4*block_h products.
//  * Weights arrive as a per-warp contiguous chunk stream built by the host
//    packer (row bucketing + LPT, see spcv_cu.cu). Every chunk is 4 steps of
//    (smem byte offset, block values) for each of the G rows, interleaved so a
//    warp-wide 16 B load is a single L1 wavefront; a register ring keeps
//    kRing chunks in flight to cover L2 latency.
//  * STRICT uses separately rounded multiply and add (__fmul_rn/__fadd_rn),
//    reproducing the reference bit-for-bit; !STRICT uses FFMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spcvk {

constexpr int kWarps = 16;              // warps per CTA
constexpr int kThreads = kWarps * 32;   // 512
constexpr int kBins = 128;              // schedule bins = kWarps x kMaxSplit
constexpr int kMaxSplit = kBins / kWarps;  // max CTAs sharing one column tile (8)

struct KernelArgs {
    const float* act;        // [images][K][S]
    float* out;              // [images][M][S]
    const float* bias;       // [M] or nullptr
    const uint4* stream;     // chunk stream, 16 B units
    const uint32_t* bin_beg; // kBins + 1 chunk offsets
    long long N;             // images * S
    int K, M, S;
    int act_kind;            // 0 none, 1 clamp
    float lo, hi;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

template <bool STRICT>
__device__ __forceinline__ float madd(float acc, float w, float a) {
    if constexpr (STRICT) {
        return __fadd_rn(acc, __fmul_rn(w, a));
    } else {
        return fmaf(w, a, acc);
    }
}

// Activation::apply (tensor.hpp:90-96): ternary compare, NaN and -0.0 pass.
__device__ __forceinline__ float clamp_ref(float v, int kind, float lo, float hi) {
    if (kind == 1) v = v < lo ? lo : (v > hi ? hi : v);
    return v;
}

constexpr uint32_t kHeader = 0xFFFFFFFFu;  // ix.w of a group header chunk
constexpr uint32_t kNoRow = 0xFFFFFFFFu;   // empty row slot

template <int BH>
struct Chunk {
    uint4 ix;       // 4 smem byte offsets (data) | {block_row, count, nchunks, kHeader} (header)
    uint4 v[BH];    // 4 steps x BH values, step-major
};

// Lane layout: LPR lanes per block row, G = 32/LPR rows per warp; each lane
// owns NF float4 column quads of its row (C = 4*NF columns), so a tile is
// T = LPR*C virtual columns. Within a quarter-warp the NF float4 loads of the
// G rows are swizzled ((j + gi) mod NF) so every 8-lane phase of an LDS.128
// touches 8 distinct bank quads (conflict-free for LPR >= 2 when NF % 4 == 0,
// for LPR >= 4 when NF == 2).
template <int BH, int LPR, int NF, bool STRICT, bool VEC>
__global__ void __launch_bounds__(kThreads, 1)
spmm_bcsr_kernel(const KernelArgs a) {
    constexpr int G = 32 / LPR;       // block rows per warp (row slots)
    constexpr int T = LPR * NF * 4;   // virtual columns per tile
    constexpr int CH = G * (1 + BH);  // chunk size in 16 B units
    constexpr int kRing = BH == 1 ? 3 : 2;  // weight-stream chunks in flight per warp

    extern __shared__ __align__(16) float smem[];
    float* s_act = smem;                                            // [K+1][T], row K = zeros
    long long* s_col = reinterpret_cast<long long*>(s_act + static_cast<size_t>(a.K + 1) * T);  // [T]
    float* s_bias = reinterpret_cast<float*>(s_col + T);            // [M]

    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    const long long n0 = static_cast<long long>(blockIdx.x) * T;
    const long long KS = static_cast<long long>(a.K) * a.S;
    const long long MS = static_cast<long long>(a.M) * a.S;

    // ---- stage bias, column bases and the [K][T] activation tile ----
    if (a.bias != nullptr)
        for (int i = tid; i < a.M; i += nthreads) cp_async4(s_bias + i, a.bias + i);
    for (int i = tid; i < T / 4; i += nthreads)  // zero row: target of padded steps
        reinterpret_cast<float4*>(s_act + static_cast<size_t>(a.K) * T)[i] =
            make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = tid; c < T; c += nthreads) {  // output offset of virtual column n0+c (-1: none)
        const long long n = n0 + c;
        long long v = -1;
        if (n < a.N) {
            const long long b = n / a.S;
            v = b * MS + (n - b * a.S);
        }
        s_col[c] = v;
    }
    if constexpr (VEC) {
        constexpr int Q = T / 4;              // float4 per tile row
        const long long n = n0 + 4 * (tid % Q);
        const bool valid = n < a.N;           // S % 4 == 0: a quad never straddles images
        long long src = 0;
        if (valid) {
            const long long b = n / a.S;
            src = b * KS + (n - b * a.S);
        }
        if (Q <= nthreads) {
            const int kstep = nthreads / Q;
            for (int k = tid / Q; k < a.K; k += kstep) {
                float* dst = s_act + static_cast<size_t>(k) * T + 4 * (tid % Q);
                if (valid)
                    cp_async16(dst, a.act + src + static_cast<long long>(k) * a.S);
                else
                    *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    } else {
        const int kstep = nthreads / T;       // T divides nthreads (T <= 128)
        const int c = tid % T;
        const long long n = n0 + c;
        const bool valid = n < a.N;
        long long src = 0;
        if (valid) {
            const long long b = n / a.S;
            src = b * KS + (n - b * a.S);
        }
        for (int k = tid / T; k < a.K; k += kstep) {
            float* dst = s_act + static_cast<size_t>(k) * T + c;
            if (valid)
                cp_async4(dst, a.act + src + static_cast<long long>(k) * a.S);
            else
                *dst = 0.f;
        }
    }

    // ---- per-lane geometry ----
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gi = lane / LPR;   // row slot within the group
    const int li = lane % LPR;
    uint32_t lane_off[NF];       // byte offset of this lane's j-th float4 within a tile row
#pragma unroll
    for (int j = 0; j < NF; ++j) lane_off[j] = 16u * (li + LPR * ((j + gi) % NF));

    // ---- this warp's contiguous slice of the weight stream ----
    // V = warps/CTA x CTAs sharing the tile virtual warps; each owns kBins/V
    // consecutive schedule bins (balanced by the packer's LPT at every split).
    const int nwarps = nthreads >> 5;
    const int per = kBins / (nwarps * gridDim.y);
    const int bin0 = (blockIdx.y * nwarps + warp) * per;
    uint32_t pos = __ldg(a.bin_beg + bin0);
    const uint32_t end = __ldg(a.bin_beg + bin0 + per);

    const uint4* stream = a.stream;
    auto load = [&](uint32_t c) {
        Chunk<BH> ch;
        if (c < end) {
            const uint4* p = stream + static_cast<size_t>(c) * CH;
            ch.ix = ldg_stream(p + gi);
#pragma unroll
            for (int j = 0; j < BH; ++j) ch.v[j] = ldg_stream(p + G + j * G + gi);
        } else {
            ch.ix = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int j = 0; j < BH; ++j) ch.v[j] = make_uint4(0, 0, 0, 0);
        }
        return ch;
    };
    Chunk<BH> ring[kRing];
#pragma unroll
    for (int d = 0; d < kRing; ++d) ring[d] = load(pos + d);

    cp_async_wait_all();
    __syncthreads();

    const char* s_bytes = reinterpret_cast<const char*>(s_act);
    const bool have_bias = a.bias != nullptr;

    float4 acc[BH][NF];
#pragma unroll
    for (int i = 0; i < BH; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t brow = kNoRow;

    auto finish = [&]() {
        if (brow == kNoRow) return;
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const int col = static_cast<int>(lane_off[j] >> 2);  // first column of the quad
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const long long roff = (static_cast<long long>(brow) * BH + i) * a.S;
                float4 v = acc[i][j];
                v.x = clamp_ref(v.x, a.act_kind, a.lo, a.hi);
                v.y = clamp_ref(v.y, a.act_kind, a.lo, a.hi);
                v.z = clamp_ref(v.z, a.act_kind, a.lo, a.hi);
                v.w = clamp_ref(v.w, a.act_kind, a.lo, a.hi);
                if constexpr (VEC) {
                    const long long o = s_col[col];
                    if (o >= 0) __stcs(reinterpret_cast<float4*>(a.out + o + roff), v);
                } else {
                    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const long long o = s_col[col + q];
                        if (o >= 0) __stcs(a.out + o + roff, e[q]);
                    }
                }
            }
        }
    };

    // One chunk: a group header (ix.w == kHeader) closes the previous group
    // and opens the next; a data chunk is 4 unconditional steps. Padding steps
    // point at the zero row with weight -0.0f: acc + (-0.0f * +0.0f) == acc
    // exactly for every acc (including -0.0), so no predication is needed.
    auto consume = [&](const Chunk<BH>& cur) {
        if (cur.ix.w == kHeader) {
            finish();
            brow = cur.ix.x;
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const float b = (brow != kNoRow && have_bias) ? s_bias[brow * BH + i] : 0.0f;
#pragma unroll
                for (int j = 0; j < NF; ++j) acc[i][j] = make_float4(b, b, b, b);
            }
            return;
        }
        const uint32_t off[4] = {cur.ix.x, cur.ix.y, cur.ix.z, cur.ix.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            float4 x[NF];
#pragma unroll
            for (int j = 0; j < NF; ++j)
                x[j] = *reinterpret_cast<const float4*>(s_bytes + (off[t] + lane_off[j]));
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const int f = t * BH + i;  // value index within the chunk (step-major)
                const uint4& vv = cur.v[f >> 2];
                const uint32_t wb = (f & 3) == 0 ? vv.x : (f & 3) == 1 ? vv.y : (f & 3) == 2 ? vv.z : vv.w;
                const float w = __uint_as_float(wb);
#pragma unroll
                for (int j = 0; j < NF; ++j) {
                    acc[i][j].x = madd<STRICT>(acc[i][j].x, w, x[j].x);
                    acc[i][j].y = madd<STRICT>(acc[i][j].y, w, x[j].y);
                    acc[i][j].z = madd<STRICT>(acc[i][j].z, w, x[j].z);
                    acc[i][j].w = madd<STRICT>(acc[i][j].w, w, x[j].w);
                }
            }
        }
    };

    // Ring rotation by static unrolling: slot d always holds chunk pos+d at
    // the top of a round, so no register moves are needed.
    while (pos + kRing <= end) {
#pragma unroll
        for (int d = 0; d < kRing; ++d) {
            const Chunk<BH> cur = ring[d];
            ring[d] = load(pos + kRing);
            ++pos;
            consume(cur);
        }
    }
#pragma unroll
    for (int d = 0; d < kRing; ++d)
        if (pos + d < end) consume(ring[d]);
    finish();
}

// Device decode of the paper-format streams (per-block-row nnz counts,
// per-block input-channel deltas, values) back into BCSR, for the bit-exact
// pack/unpack round trip. One thread per block row after a serial prefix over
// counts (block rows <= a few thousand).
__global__ void unpack_rowptr_kernel(const uint32_t* nnz, int brows, uint32_t* row_ptr) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint32_t acc = 0;
        row_ptr[0] = 0;
        for (int r = 0; r < brows; ++r) {
            acc += nnz[r];
            row_ptr[r + 1] = acc;
        }
    }
}

__global__ void unpack_cols_kernel(const uint32_t* row_ptr, const uint32_t* delta, int brows,
                                   uint32_t* col_idx) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= brows) return;
    uint32_t col = 0;
    for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
        col += delta[b];
        col_idx[b] = col;
    }
}

}  // namespace spcvk
