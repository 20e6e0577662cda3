// spcv_internal.h — state and helpers shared by the C-ABI translation units
// (spcv_cu.cu: packing + entry points; launch_bh{1,2,4}.cu: kernel dispatch).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <deque>
#include <cstddef>
#include <mutex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/spcv_cu.h"
#include "spmm_kernel.cuh"

// Tuning knobs (SPCV_* environment variables), read once when a
// matrix is packed and kept in the weights object, so no launch reads the
// environment. 0 / -1 = not set (the library's own choice).
struct Knobs {
    int steps = 0;         // SPCV_STEPS: 2 or 4 steps per chunk
    int nf = 0;            // SPCV_NF: 2 or 4 float4 quads per lane
    int tile_t = 0;        // SPCV_TILE_T: 32 / 64 / 128 columns per tile
    int nwarps = 0;        // SPCV_NWARPS: 4 / 8 / 16 warps per CTA
    int split = 0;         // SPCV_SPLIT: CTAs per tile (power of two)
    int tail = -1;         // SPCV_TAIL: 0 = no tail split, n = n row slices
    bool autotune = true;  // SPCV_AUTOTUNE=0: tail split from the heuristic only
    bool jit = true;       // SPCV_JIT=0: the tile kernel everywhere
    bool fuse_dw = false;  // SPCV_FUSE_DW=1: depthwise fused into the next 1x1 (executor, opt-in)
    long long kmajor_min_cols = -1;  // SPCV_JIT_KMAJOR_MIN_COLS
    int jit_warps = 0, jit_stages = 0;                 // SPCV_JIT_WARPS / SPCV_JIT_STAGES
    int jit_seg_instr = 0, jit_max_segs = 0;           // SPCV_JIT_SEG_INSTR / SPCV_JIT_MAX_SEGS
    int jit_direct_maxk = 0, jit_interleave = 1;       // SPCV_JIT_DIRECT_MAXK / SPCV_JIT_INTERLEAVE
    int pass_k = 0;        // SPCV_PASS_K: run matrices wider than this as channel passes of this width
    int small = 1;         // SPCV_SMALL: 0 = never the few-column kernel, 2 = always (single pass)
    bool small_head = true;  // SPCV_SMALL_HEAD=0: no per-row head table for the few-column kernel
    int coal = 1;          // SPCV_COAL: coalesced epilogue for unaligned layouts 0 = never, 1 = where the first call measures it faster, 2 = always
    int regcap = 1;        // SPCV_REGCAP=0: never the 80-register build of the unstructured 2-step kernels
    static Knobs from_env();
    long long geometry_key() const {
        return (((static_cast<long long>(nwarps) * 64 + split) * 64 + tail + 1) * 2 + regcap) * 4 + coal;
    }
};

// A weight-specialised kernel compiled at run time (jit.cu), one per call
// shape: arithmetic mode, activation kind, bias/residual presence, stored
// rows, 16 B-vectorisable activations, SM count of the device.
struct JitKey {
    bool strict = true, clamp = false, bias = false, res = false;
    bool vec = false;  // S % 4 == 0 and 16 B aligned activations / 8 B aligned outputs
    int m_out = 0;
    int sms = 0;
    int warps = 8, stages = 3;  // CTA geometry (jit_geometry)
    int cpl = 2;                // k-major columns per lane (generator's choice; not part of the key)
    // Fused 3x3 depthwise producer (executor, network.cu): the direct variant
    // computes its input channels from the depthwise layer's input instead of
    // loading them; the depthwise weights/bias (host copies) become immediates.
    bool dw = false, dw_clamp = false;
    int dw_stride = 1;
    const float* dw_w = nullptr;  // [K][9] host
    const float* dw_b = nullptr;  // [K] host or null
    bool operator==(const JitKey& o) const {
        return strict == o.strict && clamp == o.clamp && bias == o.bias && res == o.res &&
               vec == o.vec && m_out == o.m_out && sms == o.sms && warps == o.warps &&
               stages == o.stages && dw == o.dw && dw_clamp == o.dw_clamp &&
               dw_stride == o.dw_stride && dw_w == o.dw_w && dw_b == o.dw_b;
    }
};
// Runtime arguments of a fused depthwise producer.
struct JitDwArgs {
    const float* in = nullptr;  // depthwise input [images][K][H][W]
    int H = 0, W = 0, OW = 1, pad_t = 0, pad_l = 0;
    float lo = 0.0f, hi = 0.0f;
};
struct JitVariant {
    JitKey key;
    bool eligible = false;      // the planner found a variant for (matrix, key)
    bool built = false;         // compile + load attempted (fn null: it failed)
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
    bool direct = false;        // one thread per column (small K) vs k-major segments
    int cpl = 2;                // k-major: columns per lane (2 = f32x2, 1 = scalar)
    int segments = 0;
};

struct spcv_cu_weights {
    int rows = 0, cols = 0, block_h = 1, brows = 0;
    int G = 1;           // block rows per warp group (32 / LPR)
    int LPR = 32;        // lanes per block row
    int NF = 4;          // float4 column quads per lane
    int T = 128;         // virtual columns per tile (LPR * NF * 4)
    int STEPS = 4;       // steps per chunk of the weight stream (2 or 4), strict mode
    int STEPS_fast = 4;  // fast mode (a second stream is packed when it differs)
    int device = 0;
    size_t nblocks = 0;
    size_t nchunks = 0;
    // paper-format streams (north_star): counts, deltas, values
    uint32_t* d_nnz = nullptr;
    uint32_t* d_delta = nullptr;
    float* d_values = nullptr;
    // execution schedule
    uint4* d_stream = nullptr;
    uint32_t* d_bin_beg = nullptr;
    uint4* d_stream_fast = nullptr;     // null: fast mode shares the strict stream
    uint32_t* d_bin_beg_fast = nullptr;
    // plain BCSR row_ptr / col_idx (d_values holds the blocks) for the few-column kernel (small.cu)
    uint32_t* d_row_ptr = nullptr;
    uint32_t* d_col_idx = nullptr;
    uint32_t* d_head_col = nullptr;  // [brows][32] first 32 column indices per block row (~0u past the end)
    float* d_head_val = nullptr;     // [brows][32][block_h]
    Knobs knobs;  // tuning knobs at pack time
    // small-K path (jit.cu): host copy of the matrix and the planned / compiled
    // variants (a cache inside a const weights object: mutable, guarded by jit.cu's mutex)
    bool jit_eligible = false;
    std::vector<uint32_t> h_row_ptr, h_col_idx;
    std::vector<float> h_values;
    mutable std::deque<JitVariant> jit;  // deque: variants never move (launching threads hold pointers)
    // Channel passes (K too wide for one shared-memory tile): the matrix split
    // by input-channel range, each part packed on its own; a call runs them in
    // channel order, each continuing the previous part's sums (spcv_cu.cu)
    std::vector<spcv_cu_weights*> parts;
    std::vector<int> part_k0;
    // autotuned launch geometry per call shape: coal * 4096 + split * 64 + tail + 1 (spcv_cu.cu: tuned_geometry)
    mutable std::mutex tune_mu;
    mutable std::vector<std::pair<long long, int>> tuned_tail;
};

namespace spcv_detail {

extern std::atomic<uint64_t> g_launches;
extern std::atomic<uint64_t> g_jit_compiles, g_jit_cache_hits;  // NVRTC compiles / on-disk cubin hits
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kTwoCtaSmem = 112 * 1024;

// Shared memory of one CTA of the tile kernel: [K+1][T] activation tile (row
// K = zeros for padded steps) + T int64 output column offsets + bias[M].
inline size_t smem_bytes(int K, int M, int T) {
    return static_cast<size_t>(K + 1) * T * 4 + static_cast<size_t>(T) * 8 +
           static_cast<size_t>(M) * 4;
}

// Kernel dispatch for one block height (launch_bh{1,2,4}.cu).
int launch_bh1(const spcvk::KernelArgs&, const spcv_cu_weights*, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t);
int launch_bh2(const spcvk::KernelArgs&, const spcv_cu_weights*, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t);
int launch_bh4(const spcvk::KernelArgs&, const spcv_cu_weights*, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t);
// Few-column kernel (small.cu): one warp per block row x 32 columns, gathers
// straight from global memory. SPCV_ERR_UNSUPPORTED when it cannot serve.
int launch_small(const spcv_cu_weights* w, const spcvk::KernelArgs& a, bool strict, cudaStream_t st);
constexpr double kSmallMaxProducts = 8.0e6;  // products (stored values x columns) per call

// Weight-specialised kernels (jit.cu): one persistent CTA of kJitWarps warps
// per SM, a kJitStages-deep ring of [32 channels][64 columns] fp32 per warp.
constexpr size_t kJitMaxWeights = size_t(1) << 21;  // host copy kept up to this many values
constexpr int kJitSegInstr = 5000;  // straight-line instructions per row segment (i-cache)
constexpr int kJitMaxSegs = 2;      // segments per matrix (more: i-cache misses, L2 re-reads)
constexpr int kJitDirectMaxK = 64;  // direct variant: activations of a column in registers
constexpr int kJitWarps = 8;
constexpr int kJitStages = 3;
inline int jit_smem_bytes(int warps, int stages, int cpl = 2) { return warps * stages * 32 * 32 * cpl * 4; }
void jit_geometry(JitKey& key, const Knobs& kn);  // warps/stages (knobs override)
// Plan (cheap: no compile) the variant serving (matrix, key); null when none does.
const JitVariant* jit_plan(const spcv_cu_weights* w, const JitKey& key);
// Compile + load a planned variant on first use (NVRTC, or the on-disk cubin
// cache); null when that fails (recorded, never retried).
const JitVariant* jit_build(const spcv_cu_weights* w, const JitVariant* v);
inline const JitVariant* jit_prepare(const spcv_cu_weights* w, const JitKey& key) {
    return jit_build(w, jit_plan(w, key));
}
int jit_launch(const JitVariant* v, const spcvk::KernelArgs& a, cudaStream_t st,
               const JitDwArgs* dw = nullptr);
// Depthwise 3x3 (host copies of its weights/bias) fused into the next sparse
// 1x1 layer through the direct JIT variant; SPCV_ERR_UNSUPPORTED when that
// variant does not serve the matrix (the caller then runs the two layers).
int spmm_dw_fused(const spcv_cu_weights* w, const JitDwArgs& dw, int dw_stride, const float* dw_w_host,
                  const float* dw_b_host, bool dw_clamp, int images, int out_h, int out_w,
                  const float* bias, int act_kind, float lo, float hi, const float* residual,
                  float* out, int out_c, int mode, cudaStream_t st);
void jit_release(spcv_cu_weights* w);

}  // namespace spcv_detail

// Launch `kern` on `st`. (Programmatic dependent launch was measured and
// removed: griddepcontrol in the kernels costs ~1 us per batch-1 launch even
// without the launch attribute, and with it the 32-image MBv1 step was 3.7 %
// slower — profiles/r2_notes.md, r2g.)
template <typename Kern, typename... Args>
cudaError_t launch_kernel(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

#define SPCV_CUDA(call)                                                         \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess) return spcv_detail::cuda_fail(e_, #call);        \
    } while (0)
