// Microbenchmark: can tensor memory serve the SpMM activation gather, and does
// it add to the shared-memory gather? One CTA per SM owns 512 TMEM columns x
// 128 lanes (lane = output column, TMEM column = input channel); a warp reads
// its quadrant's 32 lanes at a data-dependent column (tcgen05.ld.32x32b.x1:
// one float per lane = the per-column gather), and/or LDS.128 from a shared
// tile like the tile kernel. Prints gathered bytes/clk/SM per mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_gather tmem_gather.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mode 0: all warps TMEM; 1: all warps LDS.128; 2: even warps TMEM, odd warps LDS
template <int NLD>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, int mode, unsigned long long* cyc,
                                            int lds_mult) {
    __shared__ uint32_t taddr_s;
    extern __shared__ float4 sm[];  // 64 KB tile: [128 rows][128 floats]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 512 * 8; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = taddr_s + ((static_cast<uint32_t>(warp & 3) * 32) << 16);
    // fill this warp's quadrant (warps 0-3 cover all 128 lanes)
    if (warp < 4) {
        for (int c = 0; c < 512; ++c) {
            const float v = lane * 1000.0f + c;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(tbase + c), "r"(__float_as_uint(v)));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");

    const bool use_tmem = mode == 0 || (mode == 2 && (warp & 1) == 0);
    float acc = 0.0f;
    uint32_t r = 12345u + warp * 7919u;
    const unsigned long long t0 = clock64();
    if (use_tmem) {
        for (int it = 0; it < iters; ++it) {
            uint32_t v[NLD];
#pragma unroll
            for (int j = 0; j < NLD; ++j) {
                const uint32_t col = (r >> (j * 3)) & 511u;  // data-dependent channel
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v[j]) : "r"(tbase + col));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int j = 0; j < NLD; ++j) acc += __uint_as_float(v[j]);
            r = r * 1664525u + 1013904223u;
        }
    } else {
        const char* base = reinterpret_cast<const char*>(sm);
        const int n = mode == 2 ? iters * lds_mult : iters;
        for (int it = 0; it < n; ++it) {
            // same floats gathered per warp-iteration as the TMEM path (NLD x 32)
#pragma unroll
            for (int j = 0; j < NLD / 4; ++j) {
                const uint32_t row = (r >> (j * 3)) & 127u;  // a warp reads 512 distinct B
                const float4 q = *reinterpret_cast<const float4*>(base + row * 512 + lane * 16);
                acc += q.x + q.y + q.z + q.w;
            }
            r = r * 1664525u + 1013904223u;
        }
    }
    const unsigned long long t1 = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr_s));
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NLD>
void run(const char* name, int mode, float* out, unsigned long long* cyc, int sms, int lds_mult = 1) {
    cudaFuncSetAttribute(k<NLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 32768 / NLD;
    k<NLD><<<sms, 512, 64 * 1024>>>(out, 4, mode, cyc, lds_mult);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<NLD><<<sms, 512, 64 * 1024>>>(out, iters, mode, cyc, lds_mult);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        std::printf("%s: %s\n", name, cudaGetErrorString(e));
        std::fflush(stdout);
        return;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per_warp = static_cast<double>(iters) * NLD * 32 * 4;
    const double bytes = (mode == 2 ? 8.0 * per_warp * (1 + lds_mult) : 16.0 * per_warp) * sms;
    std::printf("%-28s NLD=%2d lds_mult=%d %8.3f ms  %7.1f B/clk/SM at 1.965 GHz\n", name, NLD, lds_mult, ms,
                bytes / (ms * 1e-3) / 1.965e9 / sms);
    std::fflush(stdout);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, sms * 512 * sizeof(float));
    cudaMalloc(&cyc, sms * sizeof(unsigned long long));
    run<32>("TMEM only 16w", 0, out, cyc, sms);
    run<32>("LDS only 16w", 1, out, cyc, sms);
    run<32>("TMEM 8w + LDS 8w", 2, out, cyc, sms, 1);
    run<32>("TMEM 8w + LDS 8w", 2, out, cyc, sms, 2);
    run<32>("TMEM 8w + LDS 8w", 2, out, cyc, sms, 3);
    run<32>("TMEM 8w + LDS 8w", 2, out, cyc, sms, 4);
    return 0;
}
