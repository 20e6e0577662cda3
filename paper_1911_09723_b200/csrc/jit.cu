// jit.cu — weight-specialised SpMM kernels for small input-channel counts.
//
// For K <= 128 the whole activation column of an image fits in registers, so
// the sparse structure and the weights themselves can be compiled into the
// instruction stream (NVRTC at pack time): each thread loads its columns'
// K activations once (coalesced across the warp, straight from HBM), then
// every stored weight becomes one FMUL-with-immediate + FADD (strict) or one
// FFMA-with-immediate (fast). There is no shared-memory gather and no weight
// stream: the per-FMA cost is instruction issue, which for these layers is
// far below the HBM time, so the layer runs at the HBM roof.
//
// Arithmetic is the reference's per-element order exactly (bias first, blocks
// in ascending column, __fmul_rn then __fadd_rn, ternary clamp:
// kernels.cpp:14-43), so strict mode stays bit-exact.
#include <nvrtc.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "spcv_internal.h"

using namespace spcv_detail;

namespace {

std::string hexf(float v) {
    // exact C99 hex float literal (no decimal rounding)
    char buf[48];
    if (v == 0.0f) return std::signbit(v) ? "(-0.0f)" : "0.0f";
    std::snprintf(buf, sizeof buf, "%af", static_cast<double>(v));
    return std::string("(") + buf + ")";
}

// CUDA C for one matrix and one call shape (JitKey).
//
// One persistent CTA per SM of W warps (jit_geometry). Rounds: in each round
// warp w of CTA c owns the group of 32 virtual columns (image, pixel)
// g = round * gridDim.x * W + c * W + w, one column per lane. A group's K
// activation rows are copied global -> shared with cp.async into a per-warp
// [k][32] slot (16 B copies of 4 columns when key.vec), P rounds ahead, so
// HBM reads overlap the math of earlier rounds. A CTA barrier per round
// keeps the W warps in step: they execute the same straight-line code at the
// same time, which keeps the instruction-cache working set small.
//
// Math: each lane moves its column into registers (conflict-free LDS), then
// every stored weight is an immediate operand of FMUL+FADD (strict) or FFMA
// (fast); rows are emitted 4 at a time interleaved term by term (each row's
// own order unchanged: bias first, blocks ascending, kernels.cpp:14-43) to
// hide the add latency. Bias presence, activation kind, residual and the
// stored row count are compile-time; rows >= m_out (padding of a model layer,
// netdef.cpp:496-505) are not generated. Clamp is the ternary compare of
// Activation::apply (tensor.hpp:90-96).
std::string gen_source(int M, int K, int BH, const uint32_t* row_ptr, const uint32_t* col_idx,
                       size_t nblocks, const float* values, const JitKey& key) {
    const JitGeometry geo = jit_geometry(K);
    const int W = geo.warps, P = geo.stages;
    std::ostringstream o;
    o << "#define K " << K << "LL\n#define W " << W << "\n#define P " << P << "\n"
      << "__device__ __forceinline__ unsigned sa(const void* p) {"
         " return (unsigned)__cvta_generic_to_shared(p); }\n"
      << "__device__ __forceinline__ void cp16(float* d, const float* s) {"
         " asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\" :: \"r\"(sa(d)), \"l\"(s) : \"memory\"); }\n"
      << "__device__ __forceinline__ void cp4(float* d, const float* s) {"
         " asm volatile(\"cp.async.ca.shared.global [%0], [%1], 4;\" :: \"r\"(sa(d)), \"l\"(s) : \"memory\"); }\n"
      << "extern \"C\" __global__ void __launch_bounds__(W * 32, 1)"
         " spcv_jit(const float* __restrict__ act, float* __restrict__ out,"
         " const float* __restrict__ bias, long long N, long long S, float lo, float hi,"
         " const float* __restrict__ res) {\n"
      << "  extern __shared__ float4 smem4[];\n"
      << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
      << "  float* slot0 = reinterpret_cast<float*>(smem4) + warp * (K * 32);\n"
      << "  const long long G = (N + 31) >> 5, per_round = (long long)gridDim.x * W;\n"
      << "  const long long first = (long long)blockIdx.x * W + warp;\n"
      << "  const long long rounds = (G - (long long)blockIdx.x * W + per_round - 1) / per_round;\n"
      << "  auto issue = [&](long long r) {\n"
      << "    const long long gg = first + r * per_round;\n"
      << "    float* xs = slot0 + (r % P) * (W * K * 32);\n";
    if (key.vec)
        o << "    const long long nq = gg * 32 + 4 * (lane & 7);\n"
          << "    if (r < rounds && nq < N) {\n"
          << "      const long long b = nq / S, s = nq - b * S;\n"
          << "      const float* src = act + b * K * S + s;\n"
          << "      float* dst = xs + 4 * (lane & 7);\n"
          << "#pragma unroll 8\n"
          << "      for (int k = lane >> 3; k < K; k += 4) cp16(dst + k * 32, src + k * S);\n"
          << "    }\n";
    else
        o << "    const long long n = gg * 32 + lane;\n"
          << "    if (r < rounds && n < N) {\n"
          << "      const long long b = n / S, s = n - b * S;\n"
          << "      const float* src = act + b * K * S + s;\n"
          << "#pragma unroll 8\n"
          << "      for (int k = 0; k < K; ++k) cp4(xs + k * 32 + lane, src + k * S);\n"
          << "    }\n";
    o << "    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n"
      << "  };\n"
      << "#pragma unroll 1\n"
      << "  for (int r = 0; r < P; ++r) issue(r);\n"
      << "#pragma unroll 1\n"
      << "  for (long long r = 0; r < rounds; ++r) {\n"
      << "    asm volatile(\"cp.async.wait_group %0;\" :: \"n\"(P - 1) : \"memory\");\n"
      << "    __syncthreads();\n"
      << "    const float* xs = slot0 + (r % P) * (W * K * 32);\n";
    std::vector<char> used(static_cast<size_t>(K), 0);
    for (size_t b = 0; b < nblocks; ++b) used[col_idx[b]] = 1;
    for (int k = 0; k < K; ++k)
        if (used[k]) o << "    const float x" << k << " = xs[" << k * 32 << " + lane];\n";
    o << "    __syncwarp();\n"
      << "    issue(r + P);\n"
      << "    const long long n = (first + r * per_round) * 32 + lane;\n"
      << "    if (n >= N) continue;\n"
      << "    const long long b = n / S, s = n - b * S;\n"
      << "    float* o = out + b * " << key.m_out << "LL * S + s;\n";
    if (key.res) o << "    const float* rp = res + b * " << key.m_out << "LL * S + s;\n";
    // stored rows, emitted kIL at a time with their terms interleaved
    constexpr int kIL = 4;
    std::vector<int> rows;
    for (int r = 0; r < std::min(M, key.m_out); ++r) rows.push_back(r);
    for (size_t r0 = 0; r0 < rows.size(); r0 += kIL) {
        const size_t r1 = std::min(rows.size(), r0 + kIL);
        o << "    {\n";
        size_t longest = 0;
        for (size_t q = r0; q < r1; ++q) {
            const int row = rows[q], br = row / BH;
            longest = std::max<size_t>(longest, row_ptr[br + 1] - row_ptr[br]);
            o << "      float a" << q - r0 << " = "
              << (key.bias ? "__ldg(bias + " + std::to_string(row) + ")" : "0.0f") << ";\n";
        }
        for (size_t t = 0; t < longest; ++t) {
            for (size_t q = r0; q < r1; ++q) {
                const int row = rows[q], br = row / BH, i = row % BH;
                if (t >= row_ptr[br + 1] - row_ptr[br]) continue;
                const uint32_t blk = row_ptr[br] + static_cast<uint32_t>(t);
                const std::string A = "a" + std::to_string(q - r0);
                const std::string wv = hexf(values[static_cast<size_t>(blk) * BH + i]);
                const std::string x = "x" + std::to_string(col_idx[blk]);
                if (key.strict)
                    o << "      " << A << " = __fadd_rn(" << A << ", __fmul_rn(" << wv << ", " << x << "));\n";
                else
                    o << "      " << A << " = __fmaf_rn(" << wv << ", " << x << ", " << A << ");\n";
            }
        }
        for (size_t q = r0; q < r1; ++q) {
            const int row = rows[q];
            const std::string A = "a" + std::to_string(q - r0);
            if (key.clamp) o << "      " << A << " = " << A << " < lo ? lo : (" << A << " > hi ? hi : " << A << ");\n";
            if (key.res) o << "      " << A << " = __fadd_rn(" << A << ", __ldcs(rp + " << row << "LL * S));\n";
            o << "      __stcs(o + " << row << "LL * S, " << A << ");\n";
        }
        o << "    }\n";
    }
    o << "  }\n}\n";
    return o.str();
}

std::mutex g_jit_mu;

int jit_instr_budget() {
    static const int b = [] {
        const char* e = std::getenv("SPCV_JIT_MAX_INSTR");
        return e ? std::atoi(e) : kJitMaxInstr;
    }();
    return b;
}

// Straight-line instructions per group: 2 (strict) or 1 (fast) per stored
// weight of a stored row, one shared load per channel, ~6 per row (bias,
// clamp, address, store).
long long jit_instr_estimate(int M, int BH, const uint32_t* row_ptr, int K, const JitKey& key) {
    long long weights = 0;
    for (int r = 0; r < std::min(M, key.m_out); ++r)
        weights += row_ptr[r / BH + 1] - row_ptr[r / BH];
    return (key.strict ? 2 : 1) * weights + K + 6LL * std::min(M, key.m_out);
}

}  // namespace

// Compile (once per weights x mode) and cache in the weights object.
namespace spcv_detail {

// NVRTC: source -> sm_100a cubin. No device needed.
int jit_compile(const std::string& src, std::vector<char>& cubin) {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "spcv_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return fail(SPCV_ERR_UNSUPPORTED, "jit: nvrtcCreateProgram failed");
    // --fmad=false: strict kernels must keep FMUL and FADD separate (fast ones
    // use explicit __fmaf_rn, unaffected).
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false"};
    if (nvrtcCompileProgram(prog, 3, opts) != NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, log.data());
        nvrtcDestroyProgram(&prog);
        return fail(SPCV_ERR_UNSUPPORTED, "jit: compile failed: " + log.substr(0, 400));
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin.resize(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    return SPCV_OK;
}

const JitVariant* jit_prepare(spcv_cu_weights* w, const JitKey& key) {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    for (const JitVariant& v : w->jit)
        if (v.key == key) return v.fn ? &v : nullptr;
    w->jit.emplace_back();
    JitVariant& v = w->jit.back();
    v.key = key;
    if (jit_instr_estimate(w->rows, w->block_h, w->h_row_ptr.data(), w->cols, key) > jit_instr_budget())
        return nullptr;  // too much straight-line code: the tile kernel runs
    std::vector<char> cubin;
    const std::string src = gen_source(w->rows, w->cols, w->block_h, w->h_row_ptr.data(),
                                       w->h_col_idx.data(), w->h_col_idx.size(),
                                       w->h_values.data(), key);
    if (jit_compile(src, cubin) != SPCV_OK) return nullptr;
    cudaError_t e = cudaLibraryLoadData(&v.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
        cuda_fail(e, "jit: cudaLibraryLoadData");
        v.lib = nullptr;
        return nullptr;
    }
    e = cudaLibraryGetKernel(&v.fn, v.lib, "spcv_jit");
    if (e != cudaSuccess) {
        cuda_fail(e, "jit: cudaLibraryGetKernel");
        cudaLibraryUnload(v.lib);
        v.lib = nullptr;
        v.fn = nullptr;
        return nullptr;
    }
    const JitGeometry geo = jit_geometry(w->cols);
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(v.fn),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, geo.smem);
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v.blocks_per_sm,
                                                          reinterpret_cast<const void*>(v.fn),
                                                          geo.warps * 32, geo.smem);
    if (e != cudaSuccess || v.blocks_per_sm < 1) {
        cuda_fail(e, "jit: kernel attributes");
        cudaLibraryUnload(v.lib);
        v.lib = nullptr;
        v.fn = nullptr;
        return nullptr;
    }
    return &v;
}

void jit_release(spcv_cu_weights* w) {
    for (JitVariant& v : w->jit)
        if (v.lib) cudaLibraryUnload(v.lib);
    w->jit.clear();
}

int jit_launch(const JitVariant* v, int K, int sms, const spcvk::KernelArgs& a, cudaStream_t st) {
    // persistent: one wave of resident CTAs, rounds of W groups of 32 columns
    const JitGeometry geo = jit_geometry(K);
    const long long groups = (a.N + 31) / 32;
    const long long want = (groups + geo.warps - 1) / geo.warps;
    const long long blocks = std::min<long long>(want, static_cast<long long>(v->blocks_per_sm) * sms);
    long long N = a.N, S = a.S;
    float lo = a.lo, hi = a.hi;
    const float* act = a.act;
    float* out = a.out;
    const float* bias = a.bias;
    const float* res = a.residual;
    void* args[] = {&act, &out, &bias, &N, &S, &lo, &hi, &res};
    SPCV_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(v->fn), dim3(static_cast<unsigned>(blocks)),
                               dim3(geo.warps * 32), args, geo.smem, st));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

}  // namespace spcv_detail

// Test hook (not in the public header): generate and compile the specialised
// kernel for a host BCSR matrix without a device; reports the source and cubin
// sizes and, when src_out is non-null, copies up to src_cap bytes of source.
extern "C" int spcvx_jit_compile(int rows, int cols, int block_h, const uint32_t* row_ptr,
                                 const uint32_t* col_idx, size_t nblocks, const float* values,
                                 int mode, int act_kind, int has_bias, int has_res, int m_out,
                                 size_t* src_bytes, size_t* cubin_bytes, char* src_out,
                                 size_t src_cap) {
    JitKey key;
    key.strict = mode == SPCV_MODE_STRICT;
    key.clamp = act_kind == SPCV_ACT_CLAMP;
    key.bias = has_bias != 0;
    key.res = has_res != 0;
    key.m_out = m_out;
    key.vec = true;
    const std::string src = gen_source(rows, cols, block_h, row_ptr, col_idx, nblocks, values, key);
    if (src_bytes) *src_bytes = src.size();
    if (src_out && src_cap) {
        const size_t n = std::min(src_cap - 1, src.size());
        std::memcpy(src_out, src.data(), n);
        src_out[n] = '\0';
    }
    std::vector<char> cubin;
    const int rc = spcv_detail::jit_compile(src, cubin);
    if (cubin_bytes) *cubin_bytes = cubin.size();
    return rc;
}
