// Microbenchmark: FP32 pipe throughput per SM on sm_100a for the instruction
// forms the SpMM kernels use: FFMA, FMUL, FADD (register operands), FMUL+FADD
// (strict scalar pair), FFMA2 / FMUL2 / FADD2 (f32x2), FMUL2 + FFMA2(acc, one, p)
// (the strict packed pair). 16 independent chains per thread, many warps per SM,
// so the result is the pipe's throughput, not latency. Prints products/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_rates fp_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;

__device__ __forceinline__ void ffma2(float& ax, float& ay, float wx, float wy, float xx, float xy) {
    asm volatile("{\n .reg .b64 a, x, w;\n mov.b64 a, {%0, %1};\n mov.b64 x, {%4, %5};\n mov.b64 w, {%2, %3};\n"
                 " fma.rn.f32x2 a, w, x, a;\n mov.b64 {%0, %1}, a;\n}"
                 : "+f"(ax), "+f"(ay) : "f"(wx), "f"(wy), "f"(xx), "f"(xy));
}
__device__ __forceinline__ void strict2(float& ax, float& ay, float w, float xx, float xy, unsigned long long one) {
    asm volatile("{\n .reg .b64 a, x, p, w2;\n mov.b64 a, {%0, %1};\n mov.b64 x, {%3, %4};\n"
                 " mov.b64 w2, {%2, %2};\n mul.rn.f32x2 p, w2, x;\n fma.rn.f32x2 a, a, %5, p;\n"
                 " mov.b64 {%0, %1}, a;\n}"
                 : "+f"(ax), "+f"(ay) : "f"(w), "f"(xx), "f"(xy), "l"(one));
}

template <int MODE>
__global__ void k(float* out, int iters, float w0, unsigned long long one) {
    float acc[CH], x[CH];
    for (int i = 0; i < CH; ++i) {
        acc[i] = threadIdx.x * 1e-3f + i;
        x[i] = 1.0f + i * 1e-4f;
    }
    float w = w0 + threadIdx.x * 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; i += 2) {
            if constexpr (MODE == 0) {  // FFMA
                acc[i] = fmaf(w, x[i], acc[i]);
                acc[i + 1] = fmaf(w, x[i + 1], acc[i + 1]);
            } else if constexpr (MODE == 1) {  // strict scalar FMUL + FADD
                acc[i] = __fadd_rn(acc[i], __fmul_rn(w, x[i]));
                acc[i + 1] = __fadd_rn(acc[i + 1], __fmul_rn(w, x[i + 1]));
            } else if constexpr (MODE == 2) {  // FFMA2
                ffma2(acc[i], acc[i + 1], w, w, x[i], x[i + 1]);
            } else if constexpr (MODE == 3) {  // strict packed pair
                strict2(acc[i], acc[i + 1], w, x[i], x[i + 1], one);
            } else if constexpr (MODE == 4) {  // FMUL only (x *= w)
                x[i] = __fmul_rn(x[i], w);
                x[i + 1] = __fmul_rn(x[i + 1], w);
            }
        }
        w = w * 0.999999f;
    }
    float s = 0;
    for (int i = 0; i < CH; ++i) s += acc[i] + x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int sms, float* d) {
    const int iters = 4096, threads = 512, blocks = sms * 2;
    k<MODE><<<blocks, threads>>>(d, 16, 1.0f, 0x3f8000003f800000ULL);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<blocks, threads>>>(d, iters, 1.0f, 0x3f8000003f800000ULL);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int khz;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double products = 1.0 * blocks * threads * iters * CH;
    const double clk = ms * 1e-3 * khz * 1e3;
    printf("%-28s %8.3f ms  %7.1f products/clk/SM (at %d MHz nominal)  %.1f Gproducts/s\n", name, ms,
           products / clk / sms, khz / 1000, products / (ms * 1e-3) / 1e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d;
    cudaMalloc(&d, sizeof(float) * sms * 2 * 512);
    run<0>("FFMA", sms, d);
    run<1>("FMUL+FADD (strict scalar)", sms, d);
    run<2>("FFMA2", sms, d);
    run<3>("FMUL2+FFMA2 (strict pair)", sms, d);
    run<4>("FMUL", sms, d);
    return 0;
}
