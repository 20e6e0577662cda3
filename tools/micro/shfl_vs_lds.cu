// Microbenchmark: does SHFL consume L1/LSU data-pipe bandwidth like LDS?
// Kernel A: LDS.128 stream only. Kernel B: same LDS stream + 2 SHFL per LDS.
// Compare time and l1tex__data_pipe_lsu_wavefronts under ncu.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHFL>
__global__ void k(float* out, int iters) {
    __shared__ float4 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    unsigned idx = threadIdx.x;
    float s = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float4 v = buf[(idx + u * 32) & 2047];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            if (SHFL) {
                s += __shfl_sync(0xffffffffu, v.x, (threadIdx.x + u) & 31);
                s += __shfl_sync(0xffffffffu, v.y, (threadIdx.x + u + 3) & 31);
            }
        }
        idx += 7;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w + s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 4 * 512 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        float ms0, ms1;
        cudaEventRecord(a);
        k<0><<<148 * 4, 512>>>(out, 4096);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms0, a, b);
        cudaEventRecord(a);
        k<1><<<148 * 4, 512>>>(out, 4096);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms1, a, b);
        const double lds_bytes = 148.0 * 4 * 512 * 4096 * 8 * 16;
        printf("LDS only: %.3f ms (%.1f B/clk/SM at 1.965GHz); LDS+2xSHFL: %.3f ms\n", ms0,
               lds_bytes / (ms0 * 1e-3) / 148 / 1.965e9, ms1);
    }
    return 0;
}
