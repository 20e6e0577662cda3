// Microbenchmark: shared-memory wavefronts per LDS.128 for the SpMM lane
// layouts (LPR lanes per row, NF quads per lane, rows at random offsets),
// versus a fully contiguous warp load. Prints achieved bytes/clk/SM; run
// under ncu for l1tex__data_pipe_lsu_wavefronts_mem_shared.
#include <cstdio>
#include <cuda_runtime.h>

// T floats per smem row; LPR lanes per row; NF quads per lane; swizzle as in spmm_kernel.cuh
template <int LPR, int NF, int T, bool SWZ>
__global__ void k(float* out, const unsigned* rows, int iters) {
    extern __shared__ float4 sm[];
    const int nrows = 40 * 1024 / (T * 4) ;  // ~40 KB of rows
    for (int i = threadIdx.x; i < nrows * T / 4; i += blockDim.x) sm[i] = make_float4(i, 1, 2, 3);
    __syncthreads();
    const int lane = threadIdx.x & 31, gi = lane / LPR, li = lane % LPR;
    unsigned lane_off[NF];
    for (int j = 0; j < NF; ++j) lane_off[j] = 16u * (li + LPR * (SWZ ? (j + gi) % NF : j));
    float4 acc = make_float4(0, 0, 0, 0);
    const char* base = reinterpret_cast<const char*>(sm);
    unsigned r = rows[(blockIdx.x * 131 + threadIdx.x / 32 * 7 + gi * 13) & 1023];
    for (int it = 0; it < iters; ++it) {
        const unsigned off = (r % nrows) * T * 4;
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(base + off + lane_off[j]);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        r = r * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int LPR, int NF, int T, bool SWZ>
void run(const char* name, float* out, const unsigned* rows) {
    cudaFuncSetAttribute(k<LPR, NF, T, SWZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2048;
    k<LPR, NF, T, SWZ><<<148 * 4, 512, 41 * 1024>>>(out, rows, 16);
    cudaEventRecord(a);
    k<LPR, NF, T, SWZ><<<148 * 4, 512, 41 * 1024>>>(out, rows, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 148.0 * 4 * 512 * iters * NF * 16;
    printf("%-28s %.3f ms  %.0f B/clk/SM (1.965 GHz)\n", name, ms, bytes / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    float* out;
    unsigned* rows;
    cudaMalloc(&out, 148 * 4 * 512 * 4);
    cudaMalloc(&rows, 1024 * 4);
    unsigned h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = i * 2654435761u;
    cudaMemcpy(rows, h, sizeof h, cudaMemcpyHostToDevice);
    run<32, 4, 512, false>("contig LPR32 NF4 T512", out, rows);
    run<8, 4, 128, false>("LPR8 NF4 T128", out, rows);
    run<4, 4, 64, true>("LPR4 NF4 T64 swz", out, rows);
    run<4, 4, 64, false>("LPR4 NF4 T64 noswz", out, rows);
    run<2, 4, 32, true>("LPR2 NF4 T32 swz", out, rows);
    run<2, 4, 32, false>("LPR2 NF4 T32 noswz", out, rows);
    run<16, 2, 128, false>("LPR16 NF2 T128", out, rows);
    run<8, 2, 64, false>("LPR8 NF2 T64", out, rows);
    run<4, 2, 32, true>("LPR4 NF2 T32 swz", out, rows);
    run<1, 8, 32, true>("LPR1 NF8 T32 swz", out, rows);
    return 0;
}
