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
//    tiles of T columns; a CTA stages the whole [K][T] activation block of a
//    tile into shared memory once, so each activation byte crosses HBM once,
//    and every output row of the tile is produced from shared memory.
//  * A warp works on G block rows at a time (a "row group"); each block row
//    owns LPR = 32/G lanes and each lane owns NF float4 column quads. One
//    LDS.128 per stored block per quad feeds 4*block_h products.
//  * Weights arrive as a per-warp contiguous chunk stream built by the host
//    packer (row bucketing + LPT, see spcv_cu.cu). Every chunk is 4 steps of
//    (smem byte offset, block values) for each of the G rows; a register ring
//    keeps chunks in flight to cover L2 latency.
//  * spmm_bcsr_kernel: one tile per CTA, all warps stage it with cp.async
//    (any H*W, any alignment), then run the row-group executor (struct Exec).
//  * STRICT uses separately rounded multiply and add (__fmul_rn/__fadd_rn),
//    reproducing the reference bit-for-bit; !STRICT uses FFMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spcvk {

#ifndef SPCV_MAX_THREADS
#define SPCV_MAX_THREADS 512
#endif
#ifndef SPCV_MIN_BLOCKS
#define SPCV_MIN_BLOCKS 1
#endif
constexpr int kWarps = 16;                  // schedule granularity: warps of the widest CTA
constexpr int kThreads = SPCV_MAX_THREADS;  // launch bound (CTA sizes 128..kThreads)
constexpr int kMinBlocks = SPCV_MIN_BLOCKS;
constexpr int kBins = 128;              // schedule bins = kWarps x kMaxSplit
constexpr int kMaxSplit = kBins / kWarps;  // max CTAs sharing one column tile (8)

struct KernelArgs {
    const float* act;        // [images][K][S]
    float* out;              // [images][M][S]
    const float* bias;       // [M] or nullptr
    const uint4* stream;     // chunk stream (chunk_bytes_g<BH,STEPS>(G) bytes per chunk)
    const uint32_t* bin_beg; // kBins + 1 chunk offsets
    long long N;             // images * S
    int K, M, S;             // M: weight rows (block rows * block_h)
    int M_out;               // rows stored (<= M): the executor's padded-row truncation
    int K_img;               // channels between consecutive images of act (K, or more for a channel pass)
    const float* acc_in;     // nullptr: accumulators start at the bias; else at acc_in ([images][M_out][S],
                             // the previous channel pass's raw sums; may alias out)
    const float* residual;   // nullptr or [images][M_out][S], added after the activation
    int act_kind;            // 0 none, 1 clamp
    float lo, hi;
    // Tail splitting (kernel 1): CTAs blockIdx.x >= tail_start share their
    // tile with tail_split - 1 neighbours (each takes a slice of the rows), so
    // the last, partial wave of tiles still covers every SM.
    long long tail_start;
    int tail_split;
    int steps;               // steps per chunk of `stream` (host-side dispatch)
    int tail_pref;           // host-side: tail split chosen by the autotuner (-1: heuristic, 0: none)
    int split_pref;          // host-side: CTAs per tile chosen by the autotuner (0: heuristic)
    int coal;                // host-side: 1 = the coalesced epilogue build (unaligned layouts)
    // {1.0f, 1.0f} as f32x2, passed at run time so ptxas cannot fold the
    // strict pair mul.rn.f32x2 + fma.rn.f32x2(acc, one, p) into one FFMA2.
    unsigned long long one2;
#ifdef SPCV_TIMELINE
    // tools/timeline.py builds (make VARIANT=tl VFLAGS=-DSPCV_TIMELINE): per CTA
    // {SM id, entry, tile staged, first / last warp done, exit} in globaltimer ns
    unsigned long long* tl;
#endif
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

__device__ __forceinline__ uint2 ldg_stream2(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
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

// Two columns at once (f32x2: half the FP issue slots of scalar math).
// Strict: p = w*x rounded, then fma(acc, 1.0, p) = acc + p rounded once,
// identical to __fadd_rn(acc, __fmul_rn(w, x)) per column (acc*1 is exact).
// Fast: one fused FFMA2. Used where FP issue binds: block heights >= 2
// (each activation load feeds BH rows); for BH = 1 the kernel is bound by
// shared-memory wavefronts and the pairs only add register moves (measured).
template <bool STRICT>
__device__ __forceinline__ void madd2(float& ax, float& ay, float w, float xx, float xy,
                                      unsigned long long one2) {
    if constexpr (STRICT) {
        asm("{\n .reg .b64 a, x, p, w2;\n mov.b64 a, {%0, %1};\n mov.b64 x, {%3, %4};\n"
            " mov.b64 w2, {%2, %2};\n mul.rn.f32x2 p, w2, x;\n fma.rn.f32x2 a, a, %5, p;\n"
            " mov.b64 {%0, %1}, a;\n}"
            : "+f"(ax), "+f"(ay)
            : "f"(w), "f"(xx), "f"(xy), "l"(one2));
    } else {
        asm("{\n .reg .b64 a, x, w2;\n mov.b64 a, {%0, %1};\n mov.b64 x, {%3, %4};\n"
            " mov.b64 w2, {%2, %2};\n fma.rn.f32x2 a, w2, x, a;\n mov.b64 {%0, %1}, a;\n}"
            : "+f"(ax), "+f"(ay)
            : "f"(w), "f"(xx), "f"(xy));
    }
}

#ifndef SPCV_PAIRED_MIN_BH
#define SPCV_PAIRED_MIN_BH 2
#endif

// Activation::apply (tensor.hpp:90-96): ternary compare, NaN and -0.0 pass.
__device__ __forceinline__ float clamp_ref(float v, int kind, float lo, float hi) {
    if (kind == 1) v = v < lo ? lo : (v > hi ? hi : v);
    return v;
}
// Lower bound only: the same ternary when hi = +inf (v > +inf is false for
// every v, NaN included), i.e. ReLU — half the compare/select instructions.
__device__ __forceinline__ float clamp_lo(float v, float lo) { return v < lo ? lo : v; }

constexpr uint32_t kNoRow = 0xFFFFu;       // empty row slot (block rows < 65535)
constexpr uint32_t kHeaderHi = 0xFFFF0000u; // header word: kHeaderHi | block_row

// Chunk format, STEPS (2 or 4) steps per row slot:
//   index area: G slots x STEPS u16 activation-row indices (row K = the zero
//               row), padded to 16 B; a header's first word is
//               kHeaderHi | block_row (an index word's high half is <= K < 0xFFFF);
//   value area: G slots x STEPS*BH f32, step-major per slot; stored in 16 B
//               units [unit][slot] when STEPS*BH >= 4 (each warp-wide load is
//               contiguous), else 8 B per slot.
template <int BH, int STEPS>
struct Fmt {
    static constexpr int NI = STEPS / 2;      // 32-bit index words per slot
    static constexpr int NV = STEPS * BH;     // 32-bit value words per slot
    template <int G>
    __host__ __device__ static constexpr int idx_bytes() { return (G * NI * 4 + 15) / 16 * 16; }
    template <int G>
    __host__ __device__ static constexpr int bytes() { return idx_bytes<G>() + G * NV * 4; }
};

template <int BH, int STEPS>
__host__ __device__ constexpr int chunk_bytes_g(int G) {
    return (G * (STEPS / 2) * 4 + 15) / 16 * 16 + G * STEPS * BH * 4;
}

// A chunk as one lane sees it (its row slot).
template <int BH, int STEPS>
struct Chunk {
    uint32_t ix[STEPS / 2];
    uint32_t v[STEPS * BH];
};

// Lane layout: LPR lanes per block row, G = 32/LPR rows per warp; each lane
// owns NF float4 column quads of its row (C = 4*NF columns), so a tile is
// T = LPR*C virtual columns. Within a quarter-warp the NF float4 loads of the
// G rows are swizzled ((j + gi) mod NF) so every 8-lane phase of an LDS.128
// touches 8 distinct bank quads (conflict-free for LPR >= 2 when NF % 4 == 0,
// for LPR >= 4 when NF == 2).
// Image of virtual column n < N (a 32-bit divide when the column count allows:
// ~10x fewer instructions than the 64-bit one).
__device__ __forceinline__ long long image_of(long long n, const KernelArgs& a) {
    return a.N <= 0xFFFFFFFFLL ? static_cast<long long>(static_cast<uint32_t>(n) / static_cast<uint32_t>(a.S))
                               : n / a.S;
}
// Output offset of virtual column n (-1 when n >= N): image b, pixel s ->
// b*M*S + s; row r adds r*S.
__device__ __forceinline__ long long col_offset(long long n, const KernelArgs& a) {
    if (n >= a.N) return -1;
    const long long b = image_of(n, a);
    return b * static_cast<long long>(a.M_out) * a.S + (n - b * a.S);
}

#ifndef SPCV_HOIST
#define SPCV_HOIST 4
#endif
constexpr int kHoist = SPCV_HOIST;  // steps of activation loads issued ahead of their FMAs

// ACC: a channel pass — activations of K_img channels per image, and (after
// the first pass) accumulators starting at acc_in. A separate instantiation,
// so the single-pass kernels carry none of its code.
// COAL (unaligned layouts only, !VEC): the row group's outputs go through a
// per-warp shared-memory scratch and are stored row by row, lane = column
// (one or two contiguous segments per warp store instead of 32 scattered 4 B
// pieces over G rows: the scattered form costs as many L1 wavefronts as the
// whole gather once rows are short, e.g. H*W = 49 at >= 95 % sparsity).
template <int BH, int LPR, int NF, int STEPS, bool STRICT, bool VEC, bool RES = false, bool ACC = false,
          bool COAL = false>
struct Exec {
    static constexpr int G = 32 / LPR;
    static constexpr int T = LPR * NF * 4;
    static constexpr int RS = T + 4;           // scratch row stride (floats): rows 16 B-aligned, banks shifted
    static constexpr int CPL = (T + 31) / 32;  // columns per lane when lane = column

    float4 acc[BH][NF];
    uint32_t lane_off[NF];  // byte offset of this lane's j-th quad within a tile row
    long long ocol[VEC ? NF : (COAL ? CPL : 1)];  // VEC: output offset of each quad's first column;
                                                  // COAL: of columns lane, lane + 32, ...
    float* s_out;           // COAL: this warp's scratch [G][RS]
    int slot;               // this lane's row slot (lane / LPR)
    uint32_t brow;
    const char* s_bytes;    // current activation tile [K+1][T]
    const long long* s_col; // its output column offsets [T] (-1: past the end)
    const float* s_bias;
    bool have_bias;

    __device__ __forceinline__ void init(int gi, int li, const float* bias_smem, bool hb) {
#pragma unroll
        for (int j = 0; j < NF; ++j)  // LPR >= 8: a phase is one row, no swizzle needed
            lane_off[j] = 16u * (li + LPR * (LPR >= 8 ? j : (j + gi) % NF));
        slot = gi;
        brow = kNoRow;
        s_bias = bias_smem;
        have_bias = hb;
#pragma unroll
        for (int i = 0; i < BH; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) acc[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int i = 0; i < BH; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) acc[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    // VEC: per-lane output offsets of the tile starting at virtual column n0
    // (registers instead of s_col: avoids bank-conflicted 8 B shared loads).
    __device__ __forceinline__ void set_tile(long long n0, const KernelArgs& a) {
        if constexpr (VEC) {
#pragma unroll
            for (int j = 0; j < NF; ++j) ocol[j] = col_offset(n0 + (lane_off[j] >> 2), a);
        } else if constexpr (COAL) {
            const int lane = static_cast<int>(threadIdx.x) & 31;
#pragma unroll
            for (int c = 0; c < CPL; ++c) ocol[c] = lane + 32 * c < T ? s_col[lane + 32 * c] : -1;
        }
    }

    // COAL epilogue: every lane of the warp takes part (empty slots write nothing).
    __device__ __forceinline__ void finish_coalesced(const KernelArgs& a) {
        const bool relu = a.act_kind == 1 && a.hi == __int_as_float(0x7f800000);  // clamp(lo, +inf)
        const int lane = static_cast<int>(threadIdx.x) & 31;
#pragma unroll
        for (int i = 0; i < BH; ++i) {
#pragma unroll
            for (int j = 0; j < NF; ++j) {
                float4 v = acc[i][j];
                if (relu) {
                    v.x = clamp_lo(v.x, a.lo);
                    v.y = clamp_lo(v.y, a.lo);
                    v.z = clamp_lo(v.z, a.lo);
                    v.w = clamp_lo(v.w, a.lo);
                } else {
                    v.x = clamp_ref(v.x, a.act_kind, a.lo, a.hi);
                    v.y = clamp_ref(v.y, a.act_kind, a.lo, a.hi);
                    v.z = clamp_ref(v.z, a.act_kind, a.lo, a.hi);
                    v.w = clamp_ref(v.w, a.act_kind, a.lo, a.hi);
                }
                *reinterpret_cast<float4*>(s_out + slot * RS + (lane_off[j] >> 2)) = v;
            }
            __syncwarp();
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const uint32_t br = __shfl_sync(0xffffffffu, brow, g * LPR);  // slot g's block row
                const int r = static_cast<int>(br) * BH + i;
                if (br == kNoRow || r >= a.M_out) continue;  // empty slot / padded row (never stored)
                const long long roff = static_cast<long long>(r) * a.S;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const long long o = ocol[c];
                    if (o >= 0) {
                        float x = s_out[g * RS + lane + 32 * c];
                        if constexpr (RES) x = __fadd_rn(x, __ldcs(a.residual + o + roff));
                        __stcs(a.out + o + roff, x);
                    }
                }
            }
            __syncwarp();
        }
        brow = kNoRow;
    }

    __device__ __forceinline__ void finish(const KernelArgs& a) {
        if constexpr (!VEC && COAL) {
            finish_coalesced(a);
            return;
        }
        if (brow == kNoRow) return;
        const bool relu = a.act_kind == 1 && a.hi == __int_as_float(0x7f800000);  // clamp(lo, +inf)
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const int col = static_cast<int>(lane_off[j] >> 2);  // first column of the quad
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const int r = static_cast<int>(brow) * BH + i;
                if (r >= a.M_out) continue;  // padded row: computed, never stored (netdef.cpp:496-505)
                const long long roff = static_cast<long long>(r) * a.S;
                float4 v = acc[i][j];
                if (relu) {
                    v.x = clamp_lo(v.x, a.lo);
                    v.y = clamp_lo(v.y, a.lo);
                    v.z = clamp_lo(v.z, a.lo);
                    v.w = clamp_lo(v.w, a.lo);
                } else {
                    v.x = clamp_ref(v.x, a.act_kind, a.lo, a.hi);
                    v.y = clamp_ref(v.y, a.act_kind, a.lo, a.hi);
                    v.z = clamp_ref(v.z, a.act_kind, a.lo, a.hi);
                    v.w = clamp_ref(v.w, a.act_kind, a.lo, a.hi);
                }
                if constexpr (VEC) {
                    const long long o = ocol[j];
                    if (o >= 0) {
                        if constexpr (RES) {  // out = act(acc) + res (netdef.cpp:448-452,512)
                            const float4 rv = __ldcs(reinterpret_cast<const float4*>(a.residual + o + roff));
                            v.x = __fadd_rn(v.x, rv.x);
                            v.y = __fadd_rn(v.y, rv.y);
                            v.z = __fadd_rn(v.z, rv.z);
                            v.w = __fadd_rn(v.w, rv.w);
                        }
                        __stcs(reinterpret_cast<float4*>(a.out + o + roff), v);
                    }
                } else {
                    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const long long o = s_col[col + q];
                        if (o >= 0) {
                            float x = e[q];
                            if constexpr (RES) x = __fadd_rn(x, __ldcs(a.residual + o + roff));
                            __stcs(a.out + o + roff, x);
                        }
                    }
                }
            }
        }
        brow = kNoRow;
    }

    // Accumulators of the new group from acc_in (channel passes): the exact
    // fp32 running sums the previous pass stored (raw, before the clamp), so
    // the terms keep arriving in the reference order. Rows past M_out (never
    // stored) and columns past N start at 0.
    __device__ __forceinline__ void load_acc(const KernelArgs& a) {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const int col = static_cast<int>(lane_off[j] >> 2);
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const int r = static_cast<int>(brow) * BH + i;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (brow != kNoRow && r < a.M_out) {
                    const long long roff = static_cast<long long>(r) * a.S;
                    if constexpr (VEC) {
                        if (ocol[j] >= 0) v = *reinterpret_cast<const float4*>(a.acc_in + ocol[j] + roff);
                    } else {
                        float e[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const long long o = s_col[col + q];
                            e[q] = o >= 0 ? a.acc_in[o + roff] : 0.0f;
                        }
                        v = make_float4(e[0], e[1], e[2], e[3]);
                    }
                }
                acc[i][j] = v;
            }
        }
    }

    // One chunk: a group header closes the previous group and opens the next;
    // a data chunk is STEPS unconditional steps. Padding steps point at the
    // zero row with weight -0.0f: acc + (-0.0f * +0.0f) == acc exactly for
    // every acc (including -0.0), so no predication is needed.
    __device__ __forceinline__ void consume(const Chunk<BH, STEPS>& cur, const KernelArgs& a) {
        if ((cur.ix[0] & kHeaderHi) == kHeaderHi) {
            finish(a);
            brow = cur.ix[0] & 0xFFFFu;
            if constexpr (ACC) {  // channel pass: a later one continues the previous pass's sums
                if (a.acc_in) {
                    load_acc(a);
                    return;
                }
            }
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const float b = (brow != kNoRow && have_bias) ? s_bias[brow * BH + i] : 0.0f;
#pragma unroll
                for (int j = 0; j < NF; ++j) acc[i][j] = make_float4(b, b, b, b);
            }
            return;
        }
        constexpr int kShift = T == 32 ? 7 : (T == 64 ? 8 : (T == 128 ? 9 : 10));  // log2(T*4)
#pragma unroll
        for (int t = 0; t < STEPS; ++t) {
            if (kHoist < STEPS && t % kHoist == 0 && t > 0) __syncwarp();
            const uint32_t word = cur.ix[t >> 1];
            const uint32_t off = ((t & 1) ? (word >> 16) : (word & 0xFFFFu)) << kShift;
            float4 x[NF];
            if constexpr (LPR >= 8) {  // quads at fixed strides: one address, immediate offsets
                const char* row = s_bytes + (off + lane_off[0]);
#pragma unroll
                for (int j = 0; j < NF; ++j)
                    x[j] = *reinterpret_cast<const float4*>(row + 16 * LPR * j);
            } else {
#pragma unroll
                for (int j = 0; j < NF; ++j)
                    x[j] = *reinterpret_cast<const float4*>(s_bytes + (off + lane_off[j]));
            }
#pragma unroll
            for (int i = 0; i < BH; ++i) {
                const float w = __uint_as_float(cur.v[t * BH + i]);
#pragma unroll
                for (int j = 0; j < NF; ++j) {
                    if constexpr (BH >= SPCV_PAIRED_MIN_BH) {
                        madd2<STRICT>(acc[i][j].x, acc[i][j].y, w, x[j].x, x[j].y, a.one2);
                        madd2<STRICT>(acc[i][j].z, acc[i][j].w, w, x[j].z, x[j].w, a.one2);
                    } else {
                        acc[i][j].x = madd<STRICT>(acc[i][j].x, w, x[j].x);
                        acc[i][j].y = madd<STRICT>(acc[i][j].y, w, x[j].y);
                        acc[i][j].z = madd<STRICT>(acc[i][j].z, w, x[j].z);
                        acc[i][j].w = madd<STRICT>(acc[i][j].w, w, x[j].w);
                    }
                }
            }
        }
    }
};

template <int BH, int G, int STEPS>
__device__ __forceinline__ Chunk<BH, STEPS> load_chunk(const uint4* stream, uint32_t c, int gi) {
    using F = Fmt<BH, STEPS>;
    constexpr int CB = F::template bytes<G>();
    Chunk<BH, STEPS> ch;
    const char* p = reinterpret_cast<const char*>(stream) + static_cast<size_t>(c) * CB;
    if constexpr (F::NI == 1) {
        asm volatile("ld.global.nc.u32 %0, [%1];\n" : "=r"(ch.ix[0]) : "l"(p + gi * 4));
    } else {
        const uint2 v = ldg_stream2(p + gi * 8);
        ch.ix[0] = v.x;
        ch.ix[1] = v.y;
    }
    const char* pv = p + F::template idx_bytes<G>();
    if constexpr (F::NV == 2) {
        const uint2 v = ldg_stream2(pv + gi * 8);
        ch.v[0] = v.x;
        ch.v[1] = v.y;
    } else {
#pragma unroll
        for (int u = 0; u < F::NV / 4; ++u) {
            const uint4 v = ldg_stream(pv + (u * G + gi) * 16);
            ch.v[4 * u + 0] = v.x;
            ch.v[4 * u + 1] = v.y;
            ch.v[4 * u + 2] = v.z;
            ch.v[4 * u + 3] = v.w;
        }
    }
    return ch;
}

template <int BH, int STEPS>
__device__ __forceinline__ Chunk<BH, STEPS> zero_chunk() {
    Chunk<BH, STEPS> ch;
#pragma unroll
    for (int j = 0; j < STEPS / 2; ++j) ch.ix[j] = 0;
#pragma unroll
    for (int j = 0; j < STEPS * BH; ++j) ch.v[j] = 0;
    return ch;
}

// Chunk c of a warp's slice [.., end), or a zero chunk past its end (never consumed).
template <int BH, int G, int STEPS>
__device__ __forceinline__ Chunk<BH, STEPS> ring_chunk(const uint4* stream, uint32_t c, uint32_t end, int gi) {
    return c < end ? load_chunk<BH, G, STEPS>(stream, c, gi) : zero_chunk<BH, STEPS>();
}

// Issue the cp.async copies of tile [n0, n0+T) into s_act [K][T] (16 B when
// VEC, 4 B otherwise; zeros past column N) and write its column offsets.
// Completion: cp.async.wait_all by the issuing threads, then a CTA barrier.
template <int T, bool VEC, bool ACC = false>
__device__ __forceinline__ void stage_tile(float* s_act, long long* s_col, long long n0,
                                           const KernelArgs& a, int tid, int nthreads) {
    // image stride: K, or the whole matrix's K for a channel pass
    const long long KS = static_cast<long long>(ACC ? a.K_img : a.K) * a.S;
    for (int c = tid; c < T; c += nthreads) s_col[c] = col_offset(n0 + c, a);
    // (running pointers and the column test outside the loops: ~5 instructions
    // per copy instead of ~18, and the copies issue back to back)
    if constexpr (VEC) {
        constexpr int Q = T / 4;              // float4 per tile row (divides nthreads)
        const long long n = n0 + 4 * (tid % Q);
        const int k0 = tid / Q, kstep = nthreads / Q;
        float* dst = s_act + static_cast<size_t>(k0) * T + 4 * (tid % Q);
        const int dstep = kstep * T;
        if (n < a.N) {                        // S % 4 == 0: a quad never straddles images
            const long long b = image_of(n, a);
            const float* src = a.act + (b * KS + (n - b * a.S)) + static_cast<long long>(k0) * a.S;
            const long long sstep = static_cast<long long>(kstep) * a.S;
#pragma unroll 2
            for (int k = k0; k < a.K; k += kstep) {
                cp_async16(dst, src);
                dst += dstep;
                src += sstep;
            }
        } else {
            for (int k = k0; k < a.K; k += kstep) {
                *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
                dst += dstep;
            }
        }
    } else {
        const int c = tid % T;                // T divides nthreads (T <= 128)
        const long long n = n0 + c;
        const int k0 = tid / T, kstep = nthreads / T;
        float* dst = s_act + static_cast<size_t>(k0) * T + c;
        const int dstep = kstep * T;
        if (n < a.N) {
            const long long b = image_of(n, a);
            const float* src = a.act + (b * KS + (n - b * a.S)) + static_cast<long long>(k0) * a.S;
            const long long sstep = static_cast<long long>(kstep) * a.S;
#pragma unroll 2
            for (int k = k0; k < a.K; k += kstep) {
                cp_async4(dst, src);
                dst += dstep;
                src += sstep;
            }
        } else {
            for (int k = k0; k < a.K; k += kstep) {
                *dst = 0.f;
                dst += dstep;
            }
        }
    }
}

// Per-warp scratch of the COAL epilogue: [G][T + 4] floats.
__host__ __device__ constexpr int coal_scratch_floats(int G, int T) { return G * (T + 4); }

#ifdef SPCV_TIMELINE
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;\n" : "=r"(s));
    return s;
}
#endif

// ---------------------------------------------------------------- kernel 1
// One tile per CTA; all threads stage it with cp.async (16 B when VEC).
// CAP: compiled for three 8-warp CTAs per SM (at most 80 registers). ptxas
// otherwise settles on 83 for the unstructured 2-step kernels, which drops
// the K <= 512 layers to two CTAs per SM (measured: MBv1 pw5 237.6 vs 215.2 us,
// pw7 215.1 vs 206.8 us); the 16-warp launches of wide tiles use CAP = false.
constexpr int kCapThreads = 256, kCapBlocks = 3;
template <int BH, int LPR, int NF, int STEPS, bool STRICT, bool VEC, bool RES, bool ACC = false, bool CAP = false,
          bool COAL = false>
__global__ void __launch_bounds__(CAP ? kCapThreads : kThreads, CAP ? kCapBlocks : kMinBlocks)
spmm_bcsr_kernel(const KernelArgs a) {
    using E = Exec<BH, LPR, NF, STEPS, STRICT, VEC, RES, ACC, COAL>;
    constexpr int G = E::G;
    constexpr int T = E::T;
    constexpr int kRing = BH == 1 ? 3 : 2;  // weight-stream chunks in flight per warp

    extern __shared__ __align__(16) float smem[];
    float* s_act = smem;                                            // [K+1][T], row K = zeros
    long long* s_col = reinterpret_cast<long long*>(s_act + static_cast<size_t>(a.K + 1) * T);  // [T]
    float* s_bias = reinterpret_cast<float*>(s_col + T);            // [M]

    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
#ifdef SPCV_TIMELINE
    unsigned long long* tl = a.tl ? a.tl + 8ull * (blockIdx.x + static_cast<unsigned long long>(gridDim.x) * blockIdx.y) : nullptr;
    if (tl && tid == 0) {
        tl[0] = smid();
        tl[1] = gtime();
        tl[3] = ~0ull;
        tl[4] = 0;
    }
#endif
    // (tile, row part): full tiles first, then the tail tiles split tail_split ways
    long long tile = blockIdx.x;
    int part = blockIdx.y, nparts = gridDim.y;
    if (tile >= a.tail_start) {
        const long long k = tile - a.tail_start;
        tile = a.tail_start + k / a.tail_split;
        part = static_cast<int>(k % a.tail_split) * gridDim.y + blockIdx.y;
        nparts = a.tail_split * gridDim.y;
    }
    const long long n0 = tile * T;

    for (int i = tid; i < T / 4; i += nthreads)  // zero row: target of padded steps
        reinterpret_cast<float4*>(s_act + static_cast<size_t>(a.K) * T)[i] =
            make_float4(0.f, 0.f, 0.f, 0.f);

    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int gi = lane / LPR;

    // ---- this warp's contiguous slice of the weight stream ----
    // V = warps/CTA x CTAs sharing the tile virtual warps; each owns kBins/V
    // consecutive schedule bins (balanced by the packer at every split level).
    const int per = kBins / ((nthreads >> 5) * nparts);
    const int bin0 = (part * (nthreads >> 5) + warp) * per;
    uint32_t pos = __ldg(a.bin_beg + bin0);
    const uint32_t end = __ldg(a.bin_beg + bin0 + per);

    // ---- bias, column offsets and the [K][T] tile: issued while the slice bounds are in flight
    // (the ring's loads depend on them; the copies do not, and the volatile asms keep source order) ----
    if (a.bias != nullptr) {  // logical rows from bias; padded rows (never stored) get 0
        for (int i = tid; i < a.M_out; i += nthreads) cp_async4(s_bias + i, a.bias + i);
        for (int i = a.M_out + tid; i < a.M; i += nthreads) s_bias[i] = 0.0f;
    }
    stage_tile<T, VEC, ACC>(s_act, s_col, n0, a, tid, nthreads);

    Chunk<BH, STEPS> ring[kRing];
#pragma unroll
    for (int d = 0; d < kRing; ++d)
        ring[d] = ring_chunk<BH, G, STEPS>(a.stream, pos + d, end, gi);

    cp_async_wait_all();
    __syncthreads();
#ifdef SPCV_TIMELINE
    if (tl && tid == 0) tl[2] = gtime();
#endif

    E ex;
    ex.init(gi, lane % LPR, s_bias, a.bias != nullptr);
    ex.s_bytes = reinterpret_cast<const char*>(s_act);
    ex.s_col = s_col;
    if constexpr (COAL)  // per-warp output scratch after the bias (16 B-aligned)
        ex.s_out = s_bias + ((a.M + 3) & ~3) + warp * coal_scratch_floats(G, T);
    ex.set_tile(n0, a);

    // Ring rotation by static unrolling: slot d always holds chunk pos+d at
    // the top of a round, so no register moves are needed.
    while (pos + kRing <= end) {
#pragma unroll
        for (int d = 0; d < kRing; ++d) {
            const Chunk<BH, STEPS> cur = ring[d];
            ring[d] = ring_chunk<BH, G, STEPS>(a.stream, pos + kRing, end, gi);
            ++pos;
            ex.consume(cur, a);
        }
    }
#pragma unroll
    for (int d = 0; d < kRing; ++d)
        if (pos + d < end) ex.consume(ring[d], a);
    ex.finish(a);
#ifdef SPCV_TIMELINE
    if (tl) {
        if ((tid & 31) == 0) {
            const unsigned long long t = gtime();
            atomicMin(tl + 3, t);
            atomicMax(tl + 4, t);
        }
        __syncthreads();
        if (tid == 0) tl[5] = gtime();
    }
#endif
}

}  // namespace spcvk
