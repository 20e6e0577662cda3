// Microbenchmark: staging a [K][T] fp32 tile (row pitch in global = S floats) into shared memory
// with cp.async 16 B (LDGSTS.128, what the tile kernel does) vs one cp.async.bulk per tile row
// (UBLKCP, T*4 bytes each, completing on an mbarrier). One CTA of 256 threads per SM, `iters`
// tiles each, every tile from a different place of a large buffer (HBM-resident).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_vs_ldgsts bulk_vs_ldgsts.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const float* src, long long tiles_total, int K, int T, int S, int iters,
                                            float* sink) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(s32(&bar)));
    __syncthreads();
    float acc = 0.f;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        const long long tile = (blockIdx.x + (long long)it * gridDim.x) % tiles_total;
        const float* base = src + tile * (long long)K * S;  // rows of S floats; the tile is the first T of each
        if (MODE == 0) {
            const int Q = T / 4;
            for (int i = tid; i < K * Q; i += 256) {
                const int kk = i / Q, q = i % Q;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s32(sm + kk * T + 4 * q)),
                             "l"(base + (long long)kk * S + 4 * q));
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
            __syncthreads();
        } else {
            if (tid == 0)
                asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(s32(&bar)),
                             "r"(K * T * 4)
                             : "memory");
            for (int kk = tid; kk < K; kk += 256)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                 s32(sm + kk * T)),
                             "l"(base + (long long)kk * S), "r"(T * 4), "r"(s32(&bar))
                             : "memory");
            uint32_t ok;
            do {
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(ok)
                             : "r"(s32(&bar)), "r"(phase)
                             : "memory");
            } while (!ok);
            phase ^= 1;
        }
        acc += sm[(tid * 33) % (K * T)];
        __syncthreads();
    }
    sink[blockIdx.x * 256 + tid] = acc;
}

template <int MODE>
void run(const char* name, const float* d, long long tiles_total, int K, int T, int S, float* sink, int sms) {
    const int iters = 64;
    const size_t smem = (size_t)K * T * 4;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<MODE><<<sms, 256, smem>>>(d, tiles_total, K, T, S, 2, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<sms, 256, smem>>>(d, tiles_total, K, T, S, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-10s K=%4d T=%3d: %7.2f us per tile per SM, %6.1f GB/s per SM, %6.2f TB/s chip  %s\n", name, K, T,
           ms * 1e3 / iters, smem / (ms * 1e-3 / iters) / 1e9, smem * (double)sms / (ms * 1e-3 / iters) / 1e12,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int S = 196;
    const long long tiles_total = 4096;  // x K x S x 4 B: 1.6 GB at K = 512
    float *d, *sink;
    cudaMalloc(&d, (size_t)tiles_total * 512 * S * 4);
    cudaMemset(d, 0, (size_t)tiles_total * 512 * S * 4);
    cudaMalloc(&sink, sizeof(float) * sms * 256);
    for (int T : {32, 64, 128}) {
        const int K = 512 * 32 / T;  // 64 KB tiles
        run<0>("ldgsts16", d, tiles_total, K, T, S, sink, sms);
        run<1>("bulk/row", d, tiles_total, K, T, S, sink, sms);
    }
    cudaDeviceSynchronize();
    return 0;
}
