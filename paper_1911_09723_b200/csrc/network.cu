// network.cu — the executor (run_network, netdef.cpp:456-524) on the device.
//
// A loaded SPCV model (model.cu) runs a batch of HWC images end to end with
// every activation kept in HBM: the entry convolution, depthwise 3x3 layers,
// global average pooling, the sparse 1x1 / classifier layers through the SpMM
// path (spcv_cu_spmm_layer: padded rows truncated, residual fused into the
// epilogue) and dense ones through a strict fp32 GEMM (or cuBLAS in fast
// mode). Per-element arithmetic follows the reference kernels exactly, so in
// SPCV_MODE_STRICT the logits are bit-identical to run_network on the CPU:
//   entry conv   entry_conv_hwc_to_chw  kernels.cpp:424-474 (acc = bias; ky, kx, ci ascending)
//   depthwise    depthwise_conv_chw     kernels.cpp:385-422 (acc = bias; ky, kx ascending)
//   pooling      global_avg_pool_chw    kernels.cpp:476-487 (sequential sum, then / S)
//   dense 1x1    dense_gemm_into        kernels.cpp:345-373 (== matmul_reference, k ascending)
//   residual     add_residual           netdef.cpp:448-452 (after the activation)
// Out-of-range taps are skipped (SAME padding, tensor.cpp:7-16) — or, in the
// paired depthwise kernel, read as zeros where that provably changes no bit —
// and every multiply-add rounds the product and the sum separately.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "model_internal.h"

using namespace spcv_detail;
using namespace spcv_model;

namespace {

struct Pad {
    int out, before;
};
// same_pad (tensor.cpp:7-16)
Pad same_pad(int in, int kernel, int stride) {
    Pad p;
    p.out = (in + stride - 1) / stride;
    int total = (p.out - 1) * stride + kernel - in;
    if (total < 0) total = 0;
    p.before = total / 2;
    return p;
}

__device__ __forceinline__ float act_apply(float v, int kind, float lo, float hi) {
    return kind == 1 ? (v < lo ? lo : (v > hi ? hi : v)) : v;
}

// Division by a runtime constant for n < 2^31 (round-up multiplier, as in
// CUTLASS's FastDivmod): q = umulhi(n, m) >> (p - 32), p = 31 + ceil(log2 d).
struct FastDiv {
    uint32_t d = 1, m = 0, shift = 0;
    FastDiv() = default;
    explicit FastDiv(uint32_t div) : d(div) {
        if (d <= 1) return;
        uint32_t l = 0;
        while ((1ull << l) < d) ++l;
        const uint32_t p = 31 + l;
        m = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
        shift = p - 32;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return d == 1 ? n : (__umulhi(n, m) >> shift);
    }
};

struct ConvArgs {
    const float* in;
    const float* w;
    const float* bias;  // nullable
    float* out;
    long long total;    // images * C_out * OH * OW
    int H, W, C, CO, OH, OW, stride, pad_t, pad_l, act_kind;
    float lo, hi;
};

// Entry convolution: HWC image -> CHW, 3x3 taps, weights [co][ky][kx][ci].
// One thread per output pixel (image, oy, ox): its 9*C input taps are loaded
// once into registers (C <= kMaxEntryC), then every output channel is summed
// from them with the weights read from shared memory (warp-uniform, broadcast).
// Taps outside the image are skipped, as in the reference (not added as 0).
constexpr int kMaxEntryC = 4;
__global__ void entry_conv_kernel(const ConvArgs a) {
    extern __shared__ float wsm[];  // [CO][9*C] + bias[CO]
    const int taps = 9 * a.C;
    for (int i = threadIdx.x; i < a.CO * taps; i += blockDim.x) wsm[i] = a.w[i];
    float* bsm = wsm + a.CO * taps;
    for (int i = threadIdx.x; i < a.CO; i += blockDim.x) bsm[i] = a.bias ? a.bias[i] : 0.0f;
    __syncthreads();
    const long long pix = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long npix = a.total / a.CO;  // images * OH * OW
    if (pix >= npix) return;
    const int plane = a.OH * a.OW;
    const long long img = pix / plane;
    const int p = static_cast<int>(pix - img * plane);
    const int oy = p / a.OW, ox = p - oy * a.OW;
    const float* src = a.in + img * a.H * a.W * a.C;
    float x[9 * kMaxEntryC];
    bool ok[9];
    const int iy0 = oy * a.stride - a.pad_t, ix0 = ox * a.stride - a.pad_l;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int iy = iy0 + t / 3, ix = ix0 + t % 3;
        ok[t] = static_cast<unsigned>(iy) < static_cast<unsigned>(a.H) &&
                static_cast<unsigned>(ix) < static_cast<unsigned>(a.W);
        const float* px = src + (static_cast<long long>(ok[t] ? iy : 0) * a.W + (ok[t] ? ix : 0)) * a.C;
#pragma unroll
        for (int ci = 0; ci < kMaxEntryC; ++ci) x[t * kMaxEntryC + ci] = ci < a.C ? px[ci] : 0.0f;
    }
    float* dst = a.out + img * a.CO * plane + p;
    for (int co = 0; co < a.CO; ++co) {
        const float* k = wsm + co * taps;
        float acc = bsm[co];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            if (!ok[t]) continue;
#pragma unroll
            for (int ci = 0; ci < kMaxEntryC; ++ci)
                if (ci < a.C) acc = __fadd_rn(acc, __fmul_rn(k[t * a.C + ci], x[t * kMaxEntryC + ci]));
        }
        dst[static_cast<long long>(co) * plane] = act_apply(acc, a.act_kind, a.lo, a.hi);
    }
}

// Entry convolution with the weights in the kernel's parameter space (a
// __grid_constant__ struct, <= 32 KB): every FMUL takes its weight straight
// from the constant bank at a compile-time offset, no load instruction.
// Instantiated for C = 3 and the entry widths round_channels(32|16, width)
// produces (multiples of 8 up to 64).
template <int C, int CO>
struct EntryParams {
    float w[CO * 9 * C];  // [co][ky][kx][ci]
    float b[CO];
};

template <int C, int CO>
__global__ void __launch_bounds__(128) entry_conv_const(const ConvArgs a, const __grid_constant__ EntryParams<C, CO> prm) {
    const long long pix = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long npix = a.total / CO;
    if (pix >= npix) return;
    const int plane = a.OH * a.OW;
    const long long img = pix / plane;
    const int p = static_cast<int>(pix - img * plane);
    const int oy = p / a.OW, ox = p - oy * a.OW;
    const float* src = a.in + img * a.H * a.W * C;
    float x[9 * C];
    bool ok[9];
    const int iy0 = oy * a.stride - a.pad_t, ix0 = ox * a.stride - a.pad_l;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int iy = iy0 + t / 3, ix = ix0 + t % 3;
        ok[t] = static_cast<unsigned>(iy) < static_cast<unsigned>(a.H) &&
                static_cast<unsigned>(ix) < static_cast<unsigned>(a.W);
        const float* px = src + (static_cast<long long>(ok[t] ? iy : 0) * a.W + (ok[t] ? ix : 0)) * C;
#pragma unroll
        for (int ci = 0; ci < C; ++ci) x[t * C + ci] = __ldg(px + ci);
    }
    float* dst = a.out + img * CO * plane + p;
    bool interior = true;
#pragma unroll
    for (int t = 0; t < 9; ++t) interior = interior && ok[t];
    if (interior) {  // no tap skipped: straight-line code
#pragma unroll
        for (int co = 0; co < CO; ++co) {
            float acc = a.bias ? prm.b[co] : 0.0f;
#pragma unroll
            for (int t = 0; t < 9 * C; ++t) acc = __fadd_rn(acc, __fmul_rn(prm.w[co * 9 * C + t], x[t]));
            __stcs(dst + static_cast<long long>(co) * plane, act_apply(acc, a.act_kind, a.lo, a.hi));
        }
        return;
    }
#pragma unroll 1
    for (int co = 0; co < CO; ++co) {
        float acc = a.bias ? prm.b[co] : 0.0f;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            if (!ok[t]) continue;
#pragma unroll
            for (int ci = 0; ci < C; ++ci)
                acc = __fadd_rn(acc, __fmul_rn(prm.w[(co * 9 + t) * C + ci], x[t * C + ci]));
        }
        __stcs(dst + static_cast<long long>(co) * plane, act_apply(acc, a.act_kind, a.lo, a.hi));
    }
}

// f32 pair {a, b} as the .b64 operand of an f32x2 instruction
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a), "f"(b));
    return d;
}

// Entry convolution, two horizontally adjacent output pixels per thread in
// f32x2 registers: every weight (parameter space, a compile-time offset) is
// broadcast into both halves and multiplies the two pixels' taps at once.
// Out-of-image taps read 0 instead of being skipped, exact under the same
// conditions as depthwise_pair_kernel (finite weights, no -0.0 bias; checked
// per layer on the host). Strict: mul.rn.f32x2 + fma.rn.f32x2(acc, 1.0, p);
// per output the order stays bias, then (ky, kx, ci) ascending.
// Weights [co][tap] with the tap stride padded to a multiple of 4 floats, so
// the uniform-datapath loads of four consecutive taps are 16 B aligned.
template <int C, int CO>
struct EntryPairParams {
    static constexpr int kStride = (9 * C + 3) / 4 * 4;
    float w[CO * kStride];
    float b[CO];
};

template <int C, int CO, bool STRICT>
__global__ void __launch_bounds__(128) entry_conv_pair(const ConvArgs a, const __grid_constant__ EntryPairParams<C, CO> prm,
                                                       uint32_t pairs, FastDiv div_pw, FastDiv div_oh,
                                                       unsigned long long one) {
    const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= pairs) return;
    const int PW = (a.OW + 1) / 2;
    const uint32_t rowi = div_pw.div(it);             // img * OH + oy
    const int ox = 2 * static_cast<int>(it - rowi * PW);
    const uint32_t img = div_oh.div(rowi);
    const int oy = static_cast<int>(rowi - img * a.OH);
    const int plane = a.OH * a.OW;
    const float* src = a.in + static_cast<long long>(img) * a.H * a.W * C;
    const bool two = ox + 1 < a.OW;
    unsigned long long x[9 * C];
    const int iy0 = oy * a.stride - a.pad_t, ix0 = ox * a.stride - a.pad_l;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int iy = iy0 + t / 3, ixa = ix0 + t % 3, ixb = ixa + a.stride;
        const bool rok = static_cast<unsigned>(iy) < static_cast<unsigned>(a.H);
        const bool oka = rok && static_cast<unsigned>(ixa) < static_cast<unsigned>(a.W);
        const bool okb = two && rok && static_cast<unsigned>(ixb) < static_cast<unsigned>(a.W);
        const float* pa = src + (static_cast<long long>(iy) * a.W + ixa) * C;
        const float* pb = pa + a.stride * C;
#pragma unroll
        for (int ci = 0; ci < C; ++ci)
            x[t * C + ci] = pk2(oka ? __ldg(pa + ci) : 0.0f, okb ? __ldg(pb + ci) : 0.0f);
    }
    float* dst = a.out + static_cast<long long>(img) * CO * plane + oy * a.OW + ox;
    const bool vec = two && (a.OW % 2 == 0);  // float2 stores stay 8 B aligned
#pragma unroll
    for (int co = 0; co < CO; ++co) {
        const float b = a.bias ? prm.b[co] : 0.0f;
        unsigned long long acc = pk2(b, b);
#pragma unroll
        for (int t = 0; t < 9 * C; ++t) {
            const float wv = prm.w[co * EntryPairParams<C, CO>::kStride + t];
            const unsigned long long w = pk2(wv, wv);
            if constexpr (STRICT) {
                unsigned long long q;
                asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(q) : "l"(w), "l"(x[t]));
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc) : "l"(acc), "l"(one), "l"(q));
            } else {
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc) : "l"(w), "l"(x[t]), "l"(acc));
            }
        }
        float e0, e1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(e0), "=f"(e1) : "l"(acc));
        e0 = act_apply(e0, a.act_kind, a.lo, a.hi);
        e1 = act_apply(e1, a.act_kind, a.lo, a.hi);
        float* o = dst + static_cast<long long>(co) * plane;
        if (vec) {
            __stcs(reinterpret_cast<float2*>(o), make_float2(e0, e1));
        } else {
            __stcs(o, e0);
            if (two) __stcs(o + 1, e1);
        }
    }
}

template <int CO>
bool launch_entry_pair(const ConvArgs& a, const std::vector<float>& w_cikk, const std::vector<float>& bias,
                       int images, bool strict, cudaStream_t st) {
    using P = EntryPairParams<3, CO>;
    P prm{};
    for (int co = 0; co < CO; ++co)
        for (int t = 0; t < 9; ++t)
            for (int ci = 0; ci < 3; ++ci)  // [co][ci][ky][kx] -> [co][ky][kx][ci]
                prm.w[co * P::kStride + t * 3 + ci] = w_cikk[(static_cast<size_t>(co) * 3 + ci) * 9 + t];
    for (int co = 0; co < CO; ++co) prm.b[co] = bias.empty() ? 0.0f : bias[static_cast<size_t>(co)];
    const long long pairs = static_cast<long long>(images) * a.OH * ((a.OW + 1) / 2);
    if (pairs >= 0x7FFFFFFFLL) return false;
    const FastDiv dpw((a.OW + 1) / 2), doh(a.OH);
    const unsigned grid = static_cast<unsigned>((pairs + 127) / 128);
    const unsigned long long one = 0x3f8000003f800000ULL;
    if (strict)
        entry_conv_pair<3, CO, true><<<grid, 128, 0, st>>>(a, prm, static_cast<uint32_t>(pairs), dpw, doh, one);
    else
        entry_conv_pair<3, CO, false><<<grid, 128, 0, st>>>(a, prm, static_cast<uint32_t>(pairs), dpw, doh, one);
    return true;
}

template <int CO>
bool launch_entry_const(const ConvArgs& a, const std::vector<float>& w_cikk, const std::vector<float>& bias,
                        unsigned grid, cudaStream_t st) {
    EntryParams<3, CO> prm;
    for (int co = 0; co < CO; ++co)
        for (int t = 0; t < 9; ++t)
            for (int ci = 0; ci < 3; ++ci)  // [co][ci][ky][kx] -> [co][ky][kx][ci]
                prm.w[(co * 9 + t) * 3 + ci] = w_cikk[(static_cast<size_t>(co) * 3 + ci) * 9 + t];
    for (int co = 0; co < CO; ++co) prm.b[co] = bias.empty() ? 0.0f : bias[static_cast<size_t>(co)];
    entry_conv_const<3, CO><<<grid, 128, 0, st>>>(a, prm);
    return true;
}

bool launch_entry_fast(const ConvArgs& a, int C, int CO, const std::vector<float>& w,
                       const std::vector<float>& bias, unsigned grid, bool zero_pad, int images, bool strict,
                       cudaStream_t st) {
    if (C != 3) return false;
    if (zero_pad) {
        switch (CO) {
            case 8: return launch_entry_pair<8>(a, w, bias, images, strict, st);
            case 16: return launch_entry_pair<16>(a, w, bias, images, strict, st);
            case 24: return launch_entry_pair<24>(a, w, bias, images, strict, st);
            case 32: return launch_entry_pair<32>(a, w, bias, images, strict, st);
            case 40: return launch_entry_pair<40>(a, w, bias, images, strict, st);
            case 48: return launch_entry_pair<48>(a, w, bias, images, strict, st);
            case 56: return launch_entry_pair<56>(a, w, bias, images, strict, st);
            case 64: return launch_entry_pair<64>(a, w, bias, images, strict, st);
            default: break;
        }
    }
    switch (CO) {
        case 8: return launch_entry_const<8>(a, w, bias, grid, st);
        case 16: return launch_entry_const<16>(a, w, bias, grid, st);
        case 24: return launch_entry_const<24>(a, w, bias, grid, st);
        case 32: return launch_entry_const<32>(a, w, bias, grid, st);
        case 40: return launch_entry_const<40>(a, w, bias, grid, st);
        case 48: return launch_entry_const<48>(a, w, bias, grid, st);
        case 56: return launch_entry_const<56>(a, w, bias, grid, st);
        case 64: return launch_entry_const<64>(a, w, bias, grid, st);
        default: return false;
    }
}

// Depthwise 3x3, CHW in and out, weights [c][ky][kx]. A thread computes the
// outputs (oy .. oy+3, ox) of one column strip: it loads the 3 x (3*STRIDE+?)
// input window rows once into registers (consecutive lanes = consecutive ox:
// coalesced row loads), then sums each output's taps in the reference order.
template <int STRIDE>
__global__ void depthwise_kernel(const ConvArgs a, uint32_t items, int RB, FastDiv div_ow, FastDiv div_rb,
                                 FastDiv div_c) {
    constexpr int kRows = 4;                      // outputs per thread (vertical)
    constexpr int kIn = (kRows - 1) * STRIDE + 3;  // input rows in the window
    const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= items) return;
    const uint32_t strip = div_ow.div(it);        // plane * RB + rb
    const int ox = static_cast<int>(it - strip * a.OW);
    const uint32_t plane = div_rb.div(strip);
    const int oy0 = static_cast<int>(strip - plane * RB) * kRows;
    const int c = static_cast<int>(plane - div_c.div(plane) * a.CO);
    const float* src = a.in + static_cast<long long>(plane) * a.H * a.W;
    float k[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) k[t] = __ldg(a.w + c * 9 + t);
    const float b = a.bias ? __ldg(a.bias + c) : 0.0f;
    const int ix0 = ox * STRIDE - a.pad_l, iy0 = oy0 * STRIDE - a.pad_t;
    bool cok[3];
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) cok[kx] = static_cast<unsigned>(ix0 + kx) < static_cast<unsigned>(a.W);
    float v[kIn][3];
    bool rok[kIn];
#pragma unroll
    for (int r = 0; r < kIn; ++r) {
        const int iy = iy0 + r;
        rok[r] = static_cast<unsigned>(iy) < static_cast<unsigned>(a.H);
        const float* row = src + static_cast<long long>(rok[r] ? iy : 0) * a.W;
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) v[r][kx] = (rok[r] && cok[kx]) ? __ldg(row + ix0 + kx) : 0.0f;
    }
    float* dst = a.out + static_cast<long long>(plane) * a.OH * a.OW + ox;
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const int oy = oy0 + j;
        if (oy >= a.OH) break;
        float acc = b;
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
            const int r = j * STRIDE + ky;
            if (!rok[r]) continue;
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
                if (!cok[kx]) continue;  // tap outside the image: skipped (kernels.cpp:414-416)
                acc = __fadd_rn(acc, __fmul_rn(k[ky * 3 + kx], v[r][kx]));
            }
        }
        dst[static_cast<long long>(oy) * a.OW] = act_apply(acc, a.act_kind, a.lo, a.hi);
    }
}

// Depthwise 3x3, two horizontally adjacent outputs per thread in f32x2
// registers and a strip of DwRows<STRIDE> output rows, the input window held
// in registers (each input value loaded once per strip).
//
// Out-of-image taps read 0 instead of being skipped (kernels.cpp:410-416).
// That is exact under two conditions the host checks per layer: finite
// weights (w * 0 = +-0, never NaN) and no -0.0 bias. Then acc starts away
// from -0.0 and never reaches it (round-to-nearest: x + y = -0 only when both
// are -0), and acc + (+-0) == acc for every acc != -0.0, so the extra terms
// change no bit. Per output the order stays bias, then (ky, kx) ascending;
// strict multiplies and adds with separate roundings: mul.rn.f32x2, then
// fma.rn.f32x2(acc, 1.0, p) (acc * 1 is exact; `one` is a kernel argument so
// ptxas cannot fuse the pair). Fast mode uses one fma.rn.f32x2 per tap.
#ifndef SPCV_DW_R1
#define SPCV_DW_R1 7
#endif
template <int STRIDE>
struct DwRows {
    // output rows per thread: 7 divides every MobileNet plane height (112, 56,
    // 28, 14, 7), so no strip computes or loads rows past the plane
    static constexpr int R = STRIDE == 1 ? SPCV_DW_R1 : 4;
};

template <int STRIDE, bool STRICT>
__global__ void __launch_bounds__(256) depthwise_pair_kernel(const ConvArgs a, uint32_t items, int RB, int PW,
                                                             FastDiv div_pw, FastDiv div_rb, FastDiv div_c,
                                                             unsigned long long one) {
    constexpr int R = DwRows<STRIDE>::R;
    constexpr int NR = (R - 1) * STRIDE + 3;  // input rows of the strip
    constexpr int NC = STRIDE + 3;            // input columns of the output pair
    const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= items) return;
    const uint32_t strip = div_pw.div(it);   // plane * RB + rb
    const int xp = static_cast<int>(it - strip * PW);
    const uint32_t plane = div_rb.div(strip);
    const int rb = static_cast<int>(strip - plane * RB);
    const int c = static_cast<int>(plane - div_c.div(plane) * a.CO);
    const int ox0 = 2 * xp, oy0 = rb * R;
    const int ix0 = ox0 * STRIDE - a.pad_l, iy0 = oy0 * STRIDE - a.pad_t;
    const float* src = a.in + static_cast<long long>(plane) * a.H * a.W;
    float k[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) k[t] = __ldg(a.w + c * 9 + t);
    const float b = a.bias ? __ldg(a.bias + c) : 0.0f;
    bool cok[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) cok[q] = static_cast<unsigned>(ix0 + q) < static_cast<unsigned>(a.W);
    // window origin (may lie outside the plane: only valid taps dereference it)
    const float* p0 = src + static_cast<long long>(iy0) * a.W + ix0;
    float v[NR][NC];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const bool rok = static_cast<unsigned>(iy0 + r) < static_cast<unsigned>(a.H);
        const float* row = p0 + r * a.W;
#pragma unroll
        for (int q = 0; q < NC; ++q) v[r][q] = (rok && cok[q]) ? __ldg(row + q) : 0.0f;
    }
    float* dst = a.out + static_cast<long long>(plane) * a.OH * a.OW + ox0;
    const bool two = ox0 + 1 < a.OW;
    const bool vec = two && (a.OW % 2 == 0);  // float2 stores stay 8 B aligned
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int oy = oy0 + j;
        if (oy >= a.OH) break;
        unsigned long long acc = pk2(b, b);
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
            const int r = j * STRIDE + ky;
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
                const unsigned long long x = pk2(v[r][kx], v[r][kx + STRIDE]);
                const unsigned long long w = pk2(k[ky * 3 + kx], k[ky * 3 + kx]);
                if constexpr (STRICT) {
                    unsigned long long p;
                    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(w), "l"(x));
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc) : "l"(acc), "l"(one), "l"(p));
                } else {
                    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc) : "l"(w), "l"(x), "l"(acc));
                }
            }
        }
        float e0, e1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(e0), "=f"(e1) : "l"(acc));
        e0 = act_apply(e0, a.act_kind, a.lo, a.hi);
        e1 = act_apply(e1, a.act_kind, a.lo, a.hi);
        float* o = dst + static_cast<long long>(oy) * a.OW;
        if (vec) {
            *reinterpret_cast<float2*>(o) = make_float2(e0, e1);
        } else {
            o[0] = e0;
            if (two) o[1] = e1;
        }
    }
}

// Global average pool: one thread per (image, channel), sequential sum.
__global__ void global_pool_kernel(const float* in, float* out, long long planes, int S) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= planes) return;
    const float* src = in + p * S;
    float sum = 0.0f;
    for (int s = 0; s < S; ++s) sum = __fadd_rn(sum, src[s]);
    out[p] = __fdiv_rn(sum, static_cast<float>(S));
}

__global__ void residual_add_kernel(float* out, const float* res, long long n) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = __fadd_rn(out[i], res[i]);
}

// Strict dense 1x1: out[img][r][s] = act(bias[r] + sum_k w[r][k] * x[img][k][s]),
// k ascending, zero weights included (as dense_gemm_into / matmul_reference).
// 32x32 output tile per CTA (32 x 8 threads, 4 rows each), k staged by 32.
__global__ void dense_strict_kernel(const float* __restrict__ w, const float* __restrict__ act,
                                    const float* __restrict__ bias, float* __restrict__ out, int M,
                                    int K, long long N, int S, int act_kind, float lo, float hi) {
    __shared__ float ws[32][33];
    __shared__ float xs[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long n = blockIdx.x * 32LL + tx;
    const int r0 = blockIdx.y * 32;
    const long long img = n < N ? n / S : 0, s = n < N ? n - img * S : 0;
    const float* xcol = act + img * K * S + s;
    float acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int r = r0 + ty + 8 * q;
        acc[q] = (bias && r < M) ? bias[r] : 0.0f;
    }
    for (int k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int rr = ty + 8 * q;
            const int r = r0 + rr, k = k0 + tx;
            ws[rr][tx] = (r < M && k < K) ? w[static_cast<long long>(r) * K + k] : 0.0f;
            const int kk = k0 + rr;
            xs[rr][tx] = (n < N && kk < K) ? xcol[static_cast<long long>(kk) * S] : 0.0f;
        }
        __syncthreads();
        const int kn = min(32, K - k0);
        for (int kk = 0; kk < kn; ++kk) {
            const float x = xs[kk][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(ws[ty + 8 * q][kk], x));
        }
        __syncthreads();
    }
    if (n >= N) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int r = r0 + ty + 8 * q;
        if (r < M) out[(img * M + r) * S + s] = act_apply(acc[q], act_kind, lo, hi);
    }
}

// Strict dense 1x1, f32x2 version: a CTA computes 32 rows x 64 columns, a
// thread 4 rows x the column pair (n0 + tx, n0 + 32 + tx) as f32x2
// accumulators; per output the order is bias, then k ascending with every
// weight (zeros included), mul.rn then add.rn (fma.rn.f32x2(acc, 1.0, p)), as
// dense_gemm_into / matmul_reference. k is staged by 32 in shared memory.
__global__ void __launch_bounds__(256) dense_strict_pair_kernel(const float* __restrict__ w, const float* __restrict__ act,
                                                                const float* __restrict__ bias, float* __restrict__ out,
                                                                int M, int K, long long N, int S, int act_kind, float lo,
                                                                float hi, unsigned long long one) {
    __shared__ float ws[32][33];  // [row][k]
    __shared__ float xs[32][65];  // [k][column]
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long n0 = blockIdx.x * 64LL;
    const int r0 = blockIdx.y * 32;
    unsigned long long acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int r = r0 + 4 * ty + q;
        const float b = (bias && r < M) ? bias[r] : 0.0f;
        acc[q] = pk2(b, b);
    }
    const float* xcol[8];  // this thread's staging columns n0 + ty + 8q (null past N)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const long long n = n0 + ty + 8 * q;
        const long long img = n / S, s = n - img * S;
        xcol[q] = n < N ? act + img * K * S + s : nullptr;
    }
    for (int k0 = 0; k0 < K; k0 += 32) {
        const int k = k0 + tx;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int rr = ty + 8 * q, r = r0 + rr;
            ws[rr][tx] = (r < M && k < K) ? w[static_cast<long long>(r) * K + k] : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
            xs[tx][ty + 8 * q] = (xcol[q] && k < K) ? xcol[q][static_cast<long long>(k) * S] : 0.0f;
        __syncthreads();
        const int kn = min(32, K - k0);
        for (int kk = 0; kk < kn; ++kk) {
            const unsigned long long x = pk2(xs[kk][tx], xs[kk][32 + tx]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float wv = ws[4 * ty + q][kk];
                unsigned long long p;
                asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(pk2(wv, wv)), "l"(x));
                asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc[q]) : "l"(acc[q]), "l"(one), "l"(p));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const long long n = n0 + tx + 32 * h;
        if (n >= N) continue;
        const long long img = n / S, s = n - img * S;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = r0 + 4 * ty + q;
            if (r >= M) continue;
            float e0, e1;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(e0), "=f"(e1) : "l"(acc[q]));
            out[(img * M + r) * S + s] = act_apply(h ? e1 : e0, act_kind, lo, hi);
        }
    }
}

// SPCV_DW_PAIR=0: always the per-tap (skipping) entry / depthwise kernels and
// the scalar strict dense kernel.
bool pair_off() {
    static const bool off = [] {
        const char* e = std::getenv("SPCV_DW_PAIR");
        return e && std::atoi(e) == 0;
    }();
    return off;
}

unsigned blocks_for(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

namespace spcv_model {

// One entry-convolution, depthwise or global-pool layer of the executor on
// device tensors (in: the layer's input for `images` images, out: its output).
int run_spatial_layer(const spcv_cu_model* m, size_t i, const float* in, int images, float* out, int mode,
                      cudaStream_t st) {
    constexpr int kT = 256;
    const Layer& L = m->net.layers[i];
    const long long out_elems = static_cast<long long>(images) * L.cout * L.out_h * L.out_w;
    if (L.kind == kGlobalPool) {
        const long long planes = static_cast<long long>(images) * L.cin;
        global_pool_kernel<<<blocks_for(planes, kT), kT, 0, st>>>(in, out, planes, L.in_h * L.in_w);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return SPCV_OK;
    }
    if (L.kind != kEntryConv && L.kind != kDepthwise)
        return fail(SPCV_ERR_INVALID, "model: layer " + L.name + " is not a spatial layer");
    const Pad ph = same_pad(L.in_h, 3, L.stride), pw = same_pad(L.in_w, 3, L.stride);
    ConvArgs a{in, m->d_conv[i], m->d_bias[i], out, out_elems, L.in_h, L.in_w, L.cin, L.cout,
               ph.out, pw.out, L.stride, ph.before, pw.before, L.act_kind, L.lo, L.hi};
    const bool strict = mode == SPCV_MODE_STRICT;
    if (L.kind == kEntryConv) {
        if (L.cin > kMaxEntryC)
            return fail(SPCV_ERR_UNSUPPORTED, "model: entry convolution with more than 4 input channels");
        const long long npix = static_cast<long long>(images) * ph.out * pw.out;
        if (!launch_entry_fast(a, L.cin, L.cout, L.other, L.bias, blocks_for(npix, 128),
                               L.zero_pad_exact && !pair_off(), images, strict, st)) {
            const size_t smem = (static_cast<size_t>(L.cout) * 9 * L.cin + L.cout) * sizeof(float);
            entry_conv_kernel<<<blocks_for(npix, 128), 128, smem, st>>>(a);
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return SPCV_OK;
    }
    if (L.stride != 1 && L.stride != 2) return fail(SPCV_ERR_SHAPE, "depthwise_conv_chw: stride must be 1 or 2");
    if (L.zero_pad_exact && !pair_off()) {
        // output pairs x row strips per plane, in image chunks of < 2^31 threads
        const int R = L.stride == 1 ? DwRows<1>::R : DwRows<2>::R;
        const int RB = (ph.out + R - 1) / R, PW = (pw.out + 1) / 2;
        const long long per_img = static_cast<long long>(L.cout) * RB * PW;
        const int chunk = static_cast<int>(std::max<long long>(1, 0x7FFFFFFFLL / per_img));
        const FastDiv dpw(PW), drb(RB), dc(L.cout);
        const unsigned long long one = 0x3f8000003f800000ULL;  // {1.0f, 1.0f}
        for (int i0 = 0; i0 < images; i0 += chunk) {
            const int ni = std::min(chunk, images - i0);
            ConvArgs c = a;
            c.in = a.in + static_cast<long long>(i0) * L.cin * L.in_h * L.in_w;
            c.out = a.out + static_cast<long long>(i0) * L.cout * ph.out * pw.out;
            const uint32_t items = static_cast<uint32_t>(per_img * ni);
            const unsigned grid = blocks_for(items, kT);
            if (L.stride == 1)
                strict ? depthwise_pair_kernel<1, true><<<grid, kT, 0, st>>>(c, items, RB, PW, dpw, drb, dc, one)
                       : depthwise_pair_kernel<1, false><<<grid, kT, 0, st>>>(c, items, RB, PW, dpw, drb, dc, one);
            else
                strict ? depthwise_pair_kernel<2, true><<<grid, kT, 0, st>>>(c, items, RB, PW, dpw, drb, dc, one)
                       : depthwise_pair_kernel<2, false><<<grid, kT, 0, st>>>(c, items, RB, PW, dpw, drb, dc, one);
        }
    } else {
        // per-tap kernel (skips out-of-image taps): 4-row strips per plane,
        // launched in image chunks of < 2^31 threads
        const int RB = (ph.out + 3) / 4;
        const long long per_img = static_cast<long long>(L.cout) * RB * pw.out;
        const int chunk = static_cast<int>(std::max<long long>(1, 0x7FFFFFFFLL / per_img));
        const FastDiv dow(pw.out), drb(RB), dc(L.cout);
        for (int i0 = 0; i0 < images; i0 += chunk) {
            const int ni = std::min(chunk, images - i0);
            ConvArgs c = a;
            c.in = a.in + static_cast<long long>(i0) * L.cin * L.in_h * L.in_w;
            c.out = a.out + static_cast<long long>(i0) * L.cout * ph.out * pw.out;
            const uint32_t items = static_cast<uint32_t>(per_img * ni);
            if (L.stride == 1)
                depthwise_kernel<1><<<blocks_for(items, kT), kT, 0, st>>>(c, items, RB, dow, drb, dc);
            else
                depthwise_kernel<2><<<blocks_for(items, kT), kT, 0, st>>>(c, items, RB, dow, drb, dc);
        }
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

}  // namespace spcv_model

namespace {

// The forward pass on stream st. ws == nullptr: a stream-ordered workspace
// from the model's pool, freed at the end; else a persistent workspace
// (cudaMalloc'd on first use into *ws, reused after) — what a captured graph
// needs (no allocation inside the capture).
int forward_impl(const spcv_cu_model* m, const float* input, int images, float* logits, int mode,
                 cudaStream_t st, std::vector<float*>* ws) {
    const Net& net = m->net;
    const size_t n = net.layers.size();
    std::vector<char> save(n, 0);
    for (const Layer& L : net.layers)
        if (L.residual_src >= 0) save[static_cast<size_t>(L.residual_src)] = 1;
    size_t max_elems = 0;
    for (const Layer& L : net.layers)
        max_elems = std::max(max_elems, static_cast<size_t>(L.cout) * L.out_h * L.out_w);
    const size_t per_buf = max_elems * static_cast<size_t>(images) * sizeof(float);

    // Workspace: two ping-pong buffers + one per residual source.
    std::vector<float*> owned;
    size_t next = 0;  // persistent workspace: buffers in allocation order
    auto alloc = [&](size_t bytes, float** p) -> int {
        if (ws) {
            if (next == ws->size()) {  // from the model's pool, kept until the entry is evicted
                float* q = nullptr;
                SPCV_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&q), std::max<size_t>(bytes, 4),
                                                  m->pool, st));
                ws->push_back(q);
            }
            *p = (*ws)[next++];
            return SPCV_OK;
        }
        SPCV_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 4), m->pool, st));
        owned.push_back(*p);
        return SPCV_OK;
    };
    auto release = [&]() {
        for (float* p : owned) cudaFreeAsync(p, st);
    };
    float* ping[2] = {nullptr, nullptr};
    std::vector<float*> saved(n, nullptr);
    int rc = alloc(per_buf, &ping[0]);
    if (rc == SPCV_OK) rc = alloc(per_buf, &ping[1]);
    for (size_t i = 0; i < n && rc == SPCV_OK; ++i)
        if (save[i]) {
            const Layer& L = net.layers[i];
            rc = alloc(static_cast<size_t>(L.cout) * L.out_h * L.out_w * images * sizeof(float), &saved[i]);
        }
    if (rc != SPCV_OK) {
        release();
        return rc;
    }

    const float* cur = input;
    constexpr int kT = 256;
    for (size_t i = 0; i < n && rc == SPCV_OK; ++i) {
        const Layer& L = net.layers[i];
        // Depthwise -> sparse 1x1 pair (opt-in, SPCV_FUSE_DW=1): the 1x1 layer's
        // weight-specialised kernel computes the depthwise outputs it needs
        // itself (same arithmetic order), so the depthwise activation never goes
        // through HBM. Measured slower than two kernels on MBv1 (spcv_cu.cu).
        if (L.kind == kDepthwise && i + 1 < n && !save[i] && L.residual_src < 0 &&
            net.layers[i + 1].kind == kPointwise && m->w[i + 1] && (L.stride == 1 || L.stride == 2)) {
            const Layer& P = net.layers[i + 1];
            const Pad ph = same_pad(L.in_h, 3, L.stride), pw = same_pad(L.in_w, 3, L.stride);
            JitDwArgs dwa;
            dwa.in = cur;
            dwa.H = L.in_h;
            dwa.W = L.in_w;
            dwa.OW = pw.out;
            dwa.pad_t = ph.before;
            dwa.pad_l = pw.before;
            dwa.lo = L.lo;
            dwa.hi = L.hi;
            float* pdst = i + 2 == n ? logits : (save[i + 1] ? saved[i + 1] : (cur == ping[0] ? ping[1] : ping[0]));
            const float* pres = P.residual_src >= 0 ? saved[static_cast<size_t>(P.residual_src)] : nullptr;
            const int frc = spmm_dw_fused(m->w[i + 1], dwa, L.stride, L.other.data(),
                                          L.bias.empty() ? nullptr : L.bias.data(), L.act_kind == 1, images,
                                          ph.out, pw.out, m->d_bias[i + 1], P.act_kind, P.lo, P.hi, pres, pdst,
                                          P.cout, mode, st);
            if (frc == SPCV_OK) {
                cur = pdst;
                ++i;
                continue;
            }
            if (frc != SPCV_ERR_UNSUPPORTED) {
                rc = frc;
                break;
            }
        }
        float* dst = i + 1 == n ? logits : (save[i] ? saved[i] : (cur == ping[0] ? ping[1] : ping[0]));
        const long long out_elems = static_cast<long long>(images) * L.cout * L.out_h * L.out_w;
        const float* res = L.residual_src >= 0 ? saved[static_cast<size_t>(L.residual_src)] : nullptr;
        bool res_done = false;
        switch (L.kind) {
            case kEntryConv:
            case kDepthwise:
            case kGlobalPool:
                rc = spcv_model::run_spatial_layer(m, i, cur, images, dst, mode, st);
                break;
            case kPointwise:
            case kFullyConnected: {
                if (m->w[i]) {
                    rc = spcv_cu_spmm_layer(m->w[i], cur, images, L.cin, L.in_h, L.in_w, m->d_bias[i],
                                            L.bias.size(), L.act_kind, L.lo, L.hi, res, dst, L.cout, mode, st);
                    res_done = true;
                } else if (mode == SPCV_MODE_FAST) {
                    rc = spcv_cu_dense_gemm_into(m->d_dense[i], L.rows, L.cols, cur, SPCV_LAYOUT_CHW, images,
                                                 L.cin, L.in_h, L.in_w, m->d_bias[i], L.bias.size(), L.act_kind,
                                                 L.lo, L.hi, dst, SPCV_LAYOUT_CHW, L.cout, L.out_h, L.out_w, 0, st);
                } else {
                    const long long N = static_cast<long long>(images) * L.in_h * L.in_w;
                    dim3 grid(blocks_for(N, 32), static_cast<unsigned>((L.rows + 31) / 32));
                    if (pair_off()) {
                        dense_strict_kernel<<<grid, dim3(32, 8), 0, st>>>(m->d_dense[i], cur, m->d_bias[i], dst,
                                                                          L.rows, L.cols, N, L.in_h * L.in_w,
                                                                          L.act_kind, L.lo, L.hi);
                    } else {
                        const dim3 pgrid(blocks_for(N, 64), static_cast<unsigned>((L.rows + 31) / 32));
                        dense_strict_pair_kernel<<<pgrid, dim3(32, 8), 0, st>>>(
                            m->d_dense[i], cur, m->d_bias[i], dst, L.rows, L.cols, N, L.in_h * L.in_w, L.act_kind,
                            L.lo, L.hi, 0x3f8000003f800000ULL);
                    }
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                }
                break;
            }
            default:
                rc = fail(SPCV_ERR_MODEL_FORMAT, "model: unknown layer kind");
        }
        if (rc == SPCV_OK) {
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = cuda_fail(e, "model: layer launch");
        }
        if (rc == SPCV_OK && res && !res_done) {
            residual_add_kernel<<<blocks_for(out_elems, kT), kT, 0, st>>>(dst, res, out_elems);
            g_launches.fetch_add(1, std::memory_order_relaxed);
        }
        cur = dst;
    }
    release();
    return rc;
}

// Replays of a captured forward (serving): a forward issued a third time with
// the same (images, input, logits, mode, stream) replays a CUDA graph captured
// over a persistent workspace (one graph launch instead of ~30 kernel
// launches). The first sighting of a key only remembers it (plain launches,
// pool workspace); the second makes an entry and allocates its persistent
// workspace from the model's pool; the third captures. At most 4 entries are
// kept, least recently used evicted: its workspace returns to the pool
// stream-ordered behind its last replay (an event), with no device-wide sync.
// Only for batches up to SPCV_MODEL_GRAPH_MAX_IMAGES (default 16) on
// non-default streams; SPCV_MODEL_GRAPH=0 disables it. A failed capture
// falls back to plain launches for that key.
int graph_max_images() {
    static const int v = [] {
        const char* off = std::getenv("SPCV_MODEL_GRAPH");
        if (off && std::atoi(off) == 0) return 0;
        const char* e = std::getenv("SPCV_MODEL_GRAPH_MAX_IMAGES");
        return e ? std::atoi(e) : 16;
    }();
    return v;
}

}  // namespace

extern "C" int spcv_cu_model_forward(const spcv_cu_model* m, const float* input, int images,
                                     int in_h, int in_w, int in_c, float* logits, int mode,
                                     void* stream) {
    if (!m) return fail(SPCV_ERR_INVALID, "model: null model");
    if (mode != SPCV_MODE_STRICT && mode != SPCV_MODE_FAST)
        return fail(SPCV_ERR_INVALID, "model: unknown arithmetic mode");
    const Net& net = m->net;
    // check_run_inputs (netdef.cpp:433-441)
    if (images < 0 || in_c != net.input_c || in_h != net.input_h || in_w != net.input_w)
        return fail(SPCV_ERR_SHAPE, "run: input must be HWC " + std::to_string(net.input_h) + "x" +
                                        std::to_string(net.input_w) + "x" + std::to_string(net.input_c));
    if (images == 0) return SPCV_OK;
    if (!input || !logits) return fail(SPCV_ERR_INVALID, "model: null tensor pointer");
    int dev = 0;
    SPCV_CUDA(cudaGetDevice(&dev));
    if (dev != m->device) return fail(SPCV_ERR_INVALID, "model: loaded on another device");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread || images > graph_max_images())
        return forward_impl(m, input, images, logits, mode, st, nullptr);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    SPCV_CUDA(cudaStreamIsCapturing(st, &cap));
    if (cap != cudaStreamCaptureStatusNone)  // the caller is capturing: plain launches into its graph
        return forward_impl(m, input, images, logits, mode, st, nullptr);

    std::lock_guard<std::mutex> lk(m->graph_mu);
    using Entry = spcv_cu_model::GraphEntry;
    const spcv_cu_model::GraphKey key{images, mode, input, logits, st};
    auto& graphs = m->graphs;
    Entry* e = nullptr;
    for (size_t i = 0; i < graphs.size(); ++i)
        if (graphs[i].key == key) {  // hit: becomes the most recently used
            if (i + 1 != graphs.size()) {
                Entry moved = std::move(graphs[i]);
                graphs.erase(graphs.begin() + static_cast<long>(i));
                graphs.push_back(std::move(moved));
            }
            e = &graphs.back();
            break;
        }
    if (!e) {
        // First sighting of a key: plain launches from the pool, only remembered.
        // An entry (persistent workspace, later a graph) is made on the second.
        auto it = std::find(m->seen.begin(), m->seen.end(), key);
        if (it == m->seen.end()) {
            constexpr size_t kMaxSeen = 16;
            if (m->seen.size() == kMaxSeen) m->seen.pop_front();
            m->seen.push_back(key);
            return forward_impl(m, input, images, logits, mode, st, nullptr);
        }
        m->seen.erase(it);
        constexpr size_t kMaxGraphs = 4;  // least recently used evicted
        if (graphs.size() == kMaxGraphs) {
            Entry& old = graphs.front();
            // its workspace goes back to the pool once its last replay is done:
            // ordered on this stream behind that replay, no device-wide sync
            if (old.done) SPCV_CUDA(cudaStreamWaitEvent(st, old.done, 0));
            for (float* p : old.ws) cudaFreeAsync(p, st);
            if (old.exec) cudaGraphExecDestroy(old.exec);  // an in-flight replay finishes first
            if (old.done) cudaEventDestroy(old.done);
            graphs.pop_front();
        }
        graphs.emplace_back();
        e = &graphs.back();
        e->key = key;
        SPCV_CUDA(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming));
    }
    auto mark_done = [&](int rc) {
        if (rc == SPCV_OK && e->done) cudaEventRecord(e->done, st);
        return rc;
    };
    if (e->exec) {
        SPCV_CUDA(cudaGraphLaunch(e->exec, st));
        g_launches.fetch_add(e->launches, std::memory_order_relaxed);
        return mark_done(SPCV_OK);
    }
    if (e->failed || e->uses < 1) {
        // 2nd sighting: plain launches into the persistent workspace (kernels
        // compiled and configured, workspace allocated); from the 3rd on: the graph
        const int rc = forward_impl(m, input, images, logits, mode, st, e->failed ? nullptr : &e->ws);
        if (rc == SPCV_OK) ++e->uses;
        return mark_done(rc);
    }
    const uint64_t n0 = g_launches.load();
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    int rc = ce == cudaSuccess ? forward_impl(m, input, images, logits, mode, st, &e->ws) : SPCV_ERR_CUDA;
    if (ce == cudaSuccess) {
        const cudaError_t ee = cudaStreamEndCapture(st, &graph);
        if (ee != cudaSuccess) rc = SPCV_ERR_CUDA;
    }
    if (rc == SPCV_OK && graph && cudaGraphInstantiate(&e->exec, graph, 0) != cudaSuccess) {
        e->exec = nullptr;
        rc = SPCV_ERR_CUDA;
    }
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();  // a failed capture leaves a sticky-free error behind
    e->launches = g_launches.load() - n0;
    if (rc != SPCV_OK || !e->exec) {
        e->failed = true;
        return mark_done(forward_impl(m, input, images, logits, mode, st, nullptr));
    }
    g_launches.fetch_sub(e->launches, std::memory_order_relaxed);  // recorded, not launched
    SPCV_CUDA(cudaGraphLaunch(e->exec, st));
    g_launches.fetch_add(e->launches, std::memory_order_relaxed);
    return mark_done(SPCV_OK);
}
