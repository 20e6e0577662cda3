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
// Out-of-range taps are skipped (SAME padding, tensor.cpp:7-16), never added
// as zeros, and every multiply-add is __fmul_rn + __fadd_rn.
#include <algorithm>
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
__global__ void entry_conv_kernel(const ConvArgs a) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= a.total) return;
    const int ox = static_cast<int>(i % a.OW);
    const int oy = static_cast<int>((i / a.OW) % a.OH);
    const int co = static_cast<int>((i / (static_cast<long long>(a.OW) * a.OH)) % a.CO);
    const long long img = i / (static_cast<long long>(a.OW) * a.OH * a.CO);
    const float* src = a.in + img * a.H * a.W * a.C;
    const float* kb = a.w + static_cast<long long>(co) * 9 * a.C;
    float acc = a.bias ? a.bias[co] : 0.0f;
    const int iy0 = oy * a.stride - a.pad_t, ix0 = ox * a.stride - a.pad_l;
    for (int ky = 0; ky < 3; ++ky) {
        const int iy = iy0 + ky;
        if (static_cast<unsigned>(iy) >= static_cast<unsigned>(a.H)) continue;
        for (int kx = 0; kx < 3; ++kx) {
            const int ix = ix0 + kx;
            if (static_cast<unsigned>(ix) >= static_cast<unsigned>(a.W)) continue;
            const float* px = src + (static_cast<long long>(iy) * a.W + ix) * a.C;
            const float* kk = kb + (ky * 3 + kx) * a.C;
            for (int ci = 0; ci < a.C; ++ci) acc = __fadd_rn(acc, __fmul_rn(kk[ci], px[ci]));
        }
    }
    a.out[i] = act_apply(acc, a.act_kind, a.lo, a.hi);
}

// Depthwise 3x3, CHW in and out, weights [c][ky][kx].
__global__ void depthwise_kernel(const ConvArgs a) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= a.total) return;
    const int ox = static_cast<int>(i % a.OW);
    const int oy = static_cast<int>((i / a.OW) % a.OH);
    const long long plane = i / (static_cast<long long>(a.OW) * a.OH);  // img * C + c
    const int c = static_cast<int>(plane % a.CO);
    const float* src = a.in + plane * a.H * a.W;
    const float* k = a.w + c * 9;
    float acc = a.bias ? a.bias[c] : 0.0f;
    const int iy0 = oy * a.stride - a.pad_t, ix0 = ox * a.stride - a.pad_l;
    for (int ky = 0; ky < 3; ++ky) {
        const int iy = iy0 + ky;
        if (static_cast<unsigned>(iy) >= static_cast<unsigned>(a.H)) continue;
        const float* row = src + static_cast<long long>(iy) * a.W;
        for (int kx = 0; kx < 3; ++kx) {
            const int ix = ix0 + kx;
            if (static_cast<unsigned>(ix) >= static_cast<unsigned>(a.W)) continue;
            acc = __fadd_rn(acc, __fmul_rn(k[ky * 3 + kx], row[ix]));
        }
    }
    a.out[i] = act_apply(acc, a.act_kind, a.lo, a.hi);
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

unsigned blocks_for(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

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

    const size_t n = net.layers.size();
    std::vector<char> save(n, 0);
    for (const Layer& L : net.layers)
        if (L.residual_src >= 0) save[static_cast<size_t>(L.residual_src)] = 1;
    size_t max_elems = 0;
    for (const Layer& L : net.layers)
        max_elems = std::max(max_elems, static_cast<size_t>(L.cout) * L.out_h * L.out_w);
    const size_t per_buf = max_elems * static_cast<size_t>(images) * sizeof(float);

    // Stream-ordered workspace: two ping-pong buffers + one per residual source.
    std::vector<float*> owned;
    auto alloc = [&](size_t bytes, float** p) -> int {
        SPCV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 4), st));
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
        float* dst = i + 1 == n ? logits : (save[i] ? saved[i] : (cur == ping[0] ? ping[1] : ping[0]));
        const long long out_elems = static_cast<long long>(images) * L.cout * L.out_h * L.out_w;
        const float* res = L.residual_src >= 0 ? saved[static_cast<size_t>(L.residual_src)] : nullptr;
        bool res_done = false;
        switch (L.kind) {
            case kEntryConv:
            case kDepthwise: {
                const Pad ph = same_pad(L.in_h, 3, L.stride), pw = same_pad(L.in_w, 3, L.stride);
                ConvArgs a{cur, m->d_conv[i], m->d_bias[i], dst, out_elems, L.in_h, L.in_w, L.cin, L.cout,
                           ph.out, pw.out, L.stride, ph.before, pw.before, L.act_kind, L.lo, L.hi};
                if (L.kind == kEntryConv)
                    entry_conv_kernel<<<blocks_for(out_elems, kT), kT, 0, st>>>(a);
                else
                    depthwise_kernel<<<blocks_for(out_elems, kT), kT, 0, st>>>(a);
                g_launches.fetch_add(1, std::memory_order_relaxed);
                break;
            }
            case kGlobalPool: {
                const long long planes = static_cast<long long>(images) * L.cin;
                global_pool_kernel<<<blocks_for(planes, kT), kT, 0, st>>>(cur, dst, planes, L.in_h * L.in_w);
                g_launches.fetch_add(1, std::memory_order_relaxed);
                break;
            }
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
                    dense_strict_kernel<<<grid, dim3(32, 8), 0, st>>>(m->d_dense[i], cur, m->d_bias[i], dst,
                                                                      L.rows, L.cols, N, L.in_h * L.in_w,
                                                                      L.act_kind, L.lo, L.hi);
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
