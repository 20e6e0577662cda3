// dense.cu — dense fp32 baseline: the reference's
// dense_gemm_into (kernels.cpp:345-373) on the B200 through cuBLAS SGEMM
// (pedantic fp32 math: no TF32) and a bias+clamp epilogue kernel. It exists to
// give the sparse kernel an honest same-hardware dense comparison, as the
// reference's bench does (bench.cpp:216-227).
#include <cublas_v2.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "spcv_internal.h"

using namespace spcv_detail;

namespace {

// out[b][r][s] = clamp(out[b][r][s] + bias[r]); float4 when S % 4 == 0.
__global__ void bias_clamp_kernel(float* out, const float* bias, long long total, int S, int M,
                                  int kind, float lo, float hi) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>((i / S) % M);
        float v = out[i];
        if (bias) v = v + bias[r];
        out[i] = spcvk::clamp_ref(v, kind, lo, hi);
    }
}

struct Handle {
    int device;
    cublasHandle_t h;
};

int get_handle(cublasHandle_t* out) {
    static std::mutex mu;
    static std::vector<Handle> handles;
    int dev = 0;
    SPCV_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (auto& h : handles)
        if (h.device == dev) {
            *out = h.h;
            return SPCV_OK;
        }
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS)
        return fail(SPCV_ERR_CUDA, "dense_gemm: cublasCreate failed");
    // fp32 without TF32: CUBLAS_DEFAULT_MATH never uses TF32 tensor cores for
    // SGEMM; SPCV_DENSE_MATH=pedantic additionally forbids reduced-precision
    // internals (slower).
    const char* m = std::getenv("SPCV_DENSE_MATH");
    cublasSetMathMode(h, (m && std::string(m) == "pedantic") ? CUBLAS_PEDANTIC_MATH : CUBLAS_DEFAULT_MATH);
    handles.push_back({dev, h});
    *out = h;
    return SPCV_OK;
}

}  // namespace

extern "C" int spcv_cu_dense_gemm_into(const float* w, int rows, int cols, const float* act,
                                       int act_layout, int images, int act_c, int act_h,
                                       int act_w, const float* bias, size_t bias_len,
                                       int act_kind, float lo, float hi, float* out,
                                       int out_layout, int out_c, int out_h, int out_w, int cfg_m,
                                       void* stream) {
    if (act_kind != SPCV_ACT_NONE && act_kind != SPCV_ACT_CLAMP)
        return fail(SPCV_ERR_INVALID, "dense_gemm: unknown activation kind");
    if (act_kind == SPCV_ACT_CLAMP && !(lo < hi)) return fail(SPCV_ERR_INVALID, "clamp requires lo < hi");
    if (act_layout != SPCV_LAYOUT_CHW) return fail(SPCV_ERR_LAYOUT, "dense_gemm: activation must be CHW");
    if (cols != act_c)
        return fail(SPCV_ERR_SHAPE, "dense_gemm: weight cols " + std::to_string(cols) +
                                        " != activation channels " + std::to_string(act_c));
    if (bias_len != 0 && bias_len != static_cast<size_t>(rows))
        return fail(SPCV_ERR_SHAPE, "dense_gemm: bias length != rows");
    if (out_layout != SPCV_LAYOUT_CHW || out_c != rows || out_h != act_h || out_w != act_w)
        return fail(SPCV_ERR_SHAPE, "dense_gemm: output tensor shape/layout mismatch");
    if (cfg_m != 0 && cfg_m != 4 && cfg_m != 8 && cfg_m != 16)
        return fail(SPCV_ERR_INVALID, "dense_gemm: strip width must be 4, 8 or 16");
    if (rows < 0 || cols < 1 || images < 0 || act_h < 1 || act_w < 1)
        return fail(SPCV_ERR_SHAPE, "dense_gemm: dims must be >= 1");
    const long long S = static_cast<long long>(act_h) * act_w;
    if (images == 0 || rows == 0) return SPCV_OK;
    if (!w || !act || !out) return fail(SPCV_ERR_INVALID, "dense_gemm: null pointer");
    cublasHandle_t h = nullptr;
    if (const int rc = get_handle(&h)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cublasSetStream(h, st);
    // Row-major out[b] (M x S) = W (M x K) * act[b] (K x S)  <=>  column-major
    // out[b]^T (S x M) = act[b]^T (S x K) * W^T (K x M).
    const float one = 1.0f, zero = 0.0f;
    // S == 1 (the classifier): the images are the GEMM's columns, one SGEMM
    // instead of `images` matrix-vector products: column-major out (M x B) =
    // W^T' (W row-major = K x M column-major, transposed) * act (K x B).
    const cublasStatus_t cs =
        S == 1 ? cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, rows, images, cols, &one, w, cols, act, cols,
                             &zero, out, rows)
               : cublasSgemmStridedBatched(
                     h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(S), rows, cols, &one, act,
                     static_cast<int>(S), static_cast<long long>(cols) * S, w, cols, 0, &zero, out,
                     static_cast<int>(S), static_cast<long long>(rows) * S, images);
    if (cs != CUBLAS_STATUS_SUCCESS) return fail(SPCV_ERR_CUDA, "dense_gemm: cuBLAS SGEMM failed");
    const long long total = static_cast<long long>(images) * rows * S;
    if (bias_len || act_kind != SPCV_ACT_NONE) {
        const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 32));
        bias_clamp_kernel<<<blocks, 256, 0, st>>>(out, bias_len ? bias : nullptr, total,
                                                  static_cast<int>(S), rows, act_kind, lo, hi);
        SPCV_CUDA(cudaGetLastError());
    }
    return SPCV_OK;
}
