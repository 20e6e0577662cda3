// spcv_cu.cu — C-ABI shim (include/spcv_cu.h): weight packing, argument
// checks in the reference order, kernel selection and launch.
//
// Reference interface replaced: spcv::spmm_into (kernels.hpp:45-46,
// kernels.cpp:304-334) and the BcsrMatrix it consumes (sparse.hpp:65-79).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <queue>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/spcv_cu.h"
#include "spmm_kernel.cuh"

using spcvk::kBins;
using spcvk::kMaxSplit;
using spcvk::kWarps;

struct spcv_cu_weights {
    int rows = 0, cols = 0, block_h = 1, brows = 0;
    int G = 1;           // block rows per warp group (32 / LPR)
    int LPR = 32;        // lanes per block row
    int NF = 4;          // float4 column quads per lane
    int T = 128;         // virtual columns per tile (LPR * NF * 4)
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
};

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(SPCV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define SPCV_CUDA(call)                                  \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kTwoCtaSmem = 112 * 1024;

// Shared memory of one CTA: [K+1][T] activation tile (row K = zeros for
// padded steps) + T int64 output column offsets + bias[M].
size_t smem_bytes(int K, int M, int T) {
    return static_cast<size_t>(K + 1) * T * 4 + static_cast<size_t>(T) * 8 +
           static_cast<size_t>(M) * 4;
}

struct Layout {
    int LPR, NF, T;
};

// Tile layout for K input channels. Each lane owns NF float4 quads (16
// columns for block_h 1/2, 8 for block_h 4, bounded by accumulator
// registers); the widest tile T whose shared-memory footprint leaves room for
// two CTAs per SM wins, else the widest that fits one CTA.
// SPCV_TILE_T=32|64|128 overrides (tuning aid).
Layout choose_layout(int K, int M, int block_h) {
    const int NF = block_h == 4 ? 2 : 4;
    const int lprs_bh12[3] = {8, 4, 2};
    const int lprs_bh4[3] = {16, 8, 4};
    const int* lprs = block_h == 4 ? lprs_bh4 : lprs_bh12;
    if (const char* e = std::getenv("SPCV_TILE_T")) {
        const int want = std::atoi(e);
        for (int i = 0; i < 3; ++i)
            if (lprs[i] * NF * 4 == want && smem_bytes(K, M, want) <= kSmemLimit)
                return {lprs[i], NF, want};
    }
    for (size_t budget : {kTwoCtaSmem, kSmemLimit})
        for (int i = 0; i < 3; ++i) {
            const int T = lprs[i] * NF * 4;
            if (smem_bytes(K, M, T) <= budget) return {lprs[i], NF, T};
        }
    return {0, NF, 0};
}

int bitrev3(int i) { return ((i & 1) << 2) | (i & 2) | ((i & 4) >> 2); }

struct DevProps {
    int sms = 148;
};

DevProps props_for(int dev) {
    static std::mutex mu;
    static std::vector<std::pair<int, DevProps>> cache;
    std::lock_guard<std::mutex> lk(mu);
    for (auto& p : cache)
        if (p.first == dev) return p.second;
    DevProps d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cache.emplace_back(dev, d);
    return d;
}

template <typename T>
int upload(T** dst, const T* src, size_t n) {
    *dst = nullptr;
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    SPCV_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), bytes));
    if (n) SPCV_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
    return SPCV_OK;
}

void free_weights(spcv_cu_weights* w) {
    if (!w) return;
    cudaFree(w->d_nnz);
    cudaFree(w->d_delta);
    cudaFree(w->d_values);
    cudaFree(w->d_stream);
    cudaFree(w->d_bin_beg);
    delete w;
}

}  // namespace

// ------------------------------------------------------------------ packing

extern "C" int spcv_cu_pack(int rows, int cols, int block_h, const uint32_t* row_ptr,
                            size_t row_ptr_len, const uint32_t* col_idx, size_t nblocks,
                            const float* values, size_t nvalues, spcv_cu_weights** out) {
    g_last_error.clear();
    if (!out) return fail(SPCV_ERR_INVALID, "spcv_cu_pack: out is null");
    *out = nullptr;
    // BcsrMatrix::validate (sparse.cpp:16-51), same checks, same order.
    if (rows < 1 || cols < 1) return fail(SPCV_ERR_FORMAT, "bcsr: dims must be >= 1");
    if (block_h != 1 && block_h != 2 && block_h != 4)
        return fail(SPCV_ERR_FORMAT, "bcsr: block height must be 1, 2 or 4");
    if (rows % block_h != 0)
        return fail(SPCV_ERR_FORMAT, "bcsr: rows " + std::to_string(rows) +
                                         " not divisible by block height " +
                                         std::to_string(block_h));
    const int brows = rows / block_h;
    if (row_ptr_len != static_cast<size_t>(brows) + 1 || !row_ptr)
        return fail(SPCV_ERR_FORMAT, "bcsr: row_ptr length != block rows + 1");
    if (row_ptr[0] != 0) return fail(SPCV_ERR_FORMAT, "bcsr: row_ptr[0] != 0");
    for (int r = 0; r < brows; ++r)
        if (row_ptr[r] > row_ptr[r + 1])
            return fail(SPCV_ERR_FORMAT,
                        "bcsr: row_ptr not non-decreasing at block row " + std::to_string(r));
    if (row_ptr[brows] != nblocks)
        return fail(SPCV_ERR_FORMAT, "bcsr: row_ptr[-1] != block count");
    if (nvalues != nblocks * static_cast<size_t>(block_h))
        return fail(SPCV_ERR_FORMAT, "bcsr: values length != block count * block height");
    if (nblocks && (!col_idx || !values)) return fail(SPCV_ERR_FORMAT, "bcsr: null arrays");
    for (int r = 0; r < brows; ++r) {
        for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
            if (col_idx[b] >= static_cast<uint32_t>(cols))
                return fail(SPCV_ERR_FORMAT, "bcsr: column index " + std::to_string(col_idx[b]) +
                                                 " out of range in block row " + std::to_string(r));
            if (b > row_ptr[r] && col_idx[b] <= col_idx[b - 1])
                return fail(SPCV_ERR_FORMAT,
                            "bcsr: column indices not strictly increasing in block row " +
                                std::to_string(r));
        }
    }

    const Layout lay = choose_layout(cols, rows, block_h);
    if (lay.LPR == 0 || cols >= 0xFFFF)
        return fail(SPCV_ERR_UNSUPPORTED, "spcv_cu_pack: input channels " + std::to_string(cols) +
                                              " exceed the shared-memory tile limit");
    const int G = 32 / lay.LPR;
    const int T = lay.T;
    const int BH = block_h;

    // paper-format streams
    std::vector<uint32_t> nnz(brows), delta(nblocks);
    for (int r = 0; r < brows; ++r) {
        nnz[r] = row_ptr[r + 1] - row_ptr[r];
        uint32_t prev = 0;
        for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
            delta[b] = col_idx[b] - prev;
            prev = col_idx[b];
        }
    }

    // Row bucketing: sort block rows by nnz (descending), form groups of G
    // neighbours (similar lengths -> little predication), then LPT the groups
    // over kBins bins. Bin b = warp*kMaxSplit + i; ties go to the bin whose
    // (bit-reversed i, warp) is smallest so every split level stays balanced.
    std::vector<int> order(brows);
    for (int r = 0; r < brows; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return nnz[a] > nnz[b]; });
    const int ngroups = (brows + G - 1) / G;
    std::vector<int> gchunks(ngroups);
    for (int g = 0; g < ngroups; ++g) {
        uint32_t mx = 0;
        for (int s = 0; s < G; ++s) {
            const int k = g * G + s;
            if (k < brows) mx = std::max(mx, nnz[order[k]]);
        }
        gchunks[g] = static_cast<int>((mx + 3) / 4);
    }
    std::vector<std::vector<int>> bins(kBins);
    using Item = std::tuple<long long, int, int>;  // load, priority, bin
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    for (int b = 0; b < kBins; ++b) {
        const int warp = b / kMaxSplit, i = b % kMaxSplit;
        heap.emplace(0LL, bitrev3(i) * kWarps + warp, b);
    }
    std::vector<int> gorder(ngroups);
    for (int g = 0; g < ngroups; ++g) gorder[g] = g;
    std::stable_sort(gorder.begin(), gorder.end(),
                     [&](int a, int b) { return gchunks[a] > gchunks[b]; });
    for (int g : gorder) {
        auto [load, prio, b] = heap.top();
        heap.pop();
        bins[b].push_back(g);
        heap.emplace(load + gchunks[g] + 2, prio, b);  // +2: header + epilogue
    }

    // Chunk = G x 8 B (4 u16 activation-row indices per slot; row `cols` is the
    // zero row) + BH x G x 16 B values. Headers: {block_row | kNoRow, kHeader}.
    const size_t CB = static_cast<size_t>(G) * 8 + static_cast<size_t>(BH) * G * 16;
    size_t total = 0;
    for (int g = 0; g < ngroups; ++g) total += 1 + gchunks[g];
    std::vector<unsigned char> stream(total * CB + 16, 0);
    std::vector<uint32_t> bin_beg(kBins + 1);
    size_t cur = 0;
    auto put2 = [&](size_t chunk, int slot, uint32_t a, uint32_t b) {
        uint32_t* q = reinterpret_cast<uint32_t*>(stream.data() + chunk * CB + slot * 8);
        q[0] = a;
        q[1] = b;
    };
    for (int b = 0; b < kBins; ++b) {
        bin_beg[b] = static_cast<uint32_t>(cur);
        for (int g : bins[b]) {
            const int nch = gchunks[g];
            for (int s = 0; s < G; ++s) {
                const int k = g * G + s;
                put2(cur, s, k < brows ? static_cast<uint32_t>(order[k]) : spcvk::kNoRow,
                     spcvk::kHeader);
            }
            ++cur;
            for (int c = 0; c < nch; ++c, ++cur) {
                for (int s = 0; s < G; ++s) {
                    const int k = g * G + s;
                    // Padding steps read the zero row K with weight -0.0f, which
                    // leaves any accumulator bit-identical (see spmm_kernel.cuh).
                    uint32_t idx[4] = {static_cast<uint32_t>(cols), static_cast<uint32_t>(cols),
                                       static_cast<uint32_t>(cols), static_cast<uint32_t>(cols)};
                    float vals[16];
                    for (float& v : vals) v = -0.0f;
                    const int br = k < brows ? order[k] : -1;
                    for (int t = 0; t < 4 && br >= 0; ++t) {
                        const uint32_t e = static_cast<uint32_t>(4 * c + t);
                        if (e >= nnz[br]) continue;
                        const uint32_t blk = row_ptr[br] + e;
                        idx[t] = col_idx[blk];
                        for (int i = 0; i < BH; ++i)
                            vals[t * BH + i] = values[static_cast<size_t>(blk) * BH + i];
                    }
                    put2(cur, s, idx[0] | (idx[1] << 16), idx[2] | (idx[3] << 16));
                    for (int j = 0; j < BH; ++j)
                        std::memcpy(stream.data() + cur * CB + G * 8 + (j * G + s) * 16, vals + 4 * j, 16);
                }
            }
        }
    }
    bin_beg[kBins] = static_cast<uint32_t>(cur);
    if (cur > 0xFFFFFFF0ull) return fail(SPCV_ERR_UNSUPPORTED, "spcv_cu_pack: stream too large");

    auto* w = new (std::nothrow) spcv_cu_weights;
    if (!w) return fail(SPCV_ERR_CUDA, "spcv_cu_pack: out of host memory");
    w->rows = rows;
    w->cols = cols;
    w->block_h = block_h;
    w->brows = brows;
    w->G = G;
    w->LPR = lay.LPR;
    w->NF = lay.NF;
    w->T = T;
    w->nblocks = nblocks;
    w->nchunks = cur;
    cudaGetDevice(&w->device);
    int rc = SPCV_OK;
    if ((rc = upload(&w->d_nnz, nnz.data(), nnz.size())) ||
        (rc = upload(&w->d_delta, delta.data(), delta.size())) ||
        (rc = upload(&w->d_values, values, nvalues)) ||
        (rc = upload(&w->d_stream, reinterpret_cast<const uint4*>(stream.data()), stream.size() / 16)) ||
        (rc = upload(&w->d_bin_beg, bin_beg.data(), bin_beg.size()))) {
        free_weights(w);
        return rc;
    }
    *out = w;
    return SPCV_OK;
}

extern "C" int spcv_cu_unpack(const spcv_cu_weights* w, uint32_t* row_ptr, uint32_t* col_idx,
                              float* values) {
    g_last_error.clear();
    if (!w || !row_ptr || (w->nblocks && (!col_idx || !values)))
        return fail(SPCV_ERR_INVALID, "spcv_cu_unpack: null argument");
    int prev = 0;
    cudaGetDevice(&prev);
    SPCV_CUDA(cudaSetDevice(w->device));
    uint32_t *d_rp = nullptr, *d_ci = nullptr;
    int rc = SPCV_OK;
    cudaError_t e = cudaMalloc(&d_rp, sizeof(uint32_t) * (w->brows + 1));
    if (e == cudaSuccess) e = cudaMalloc(&d_ci, sizeof(uint32_t) * std::max<size_t>(w->nblocks, 1));
    if (e == cudaSuccess) {
        spcvk::unpack_rowptr_kernel<<<1, 1>>>(w->d_nnz, w->brows, d_rp);
        spcvk::unpack_cols_kernel<<<(w->brows + 127) / 128, 128>>>(d_rp, w->d_delta, w->brows, d_ci);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpy(row_ptr, d_rp, sizeof(uint32_t) * (w->brows + 1), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && w->nblocks)
        e = cudaMemcpy(col_idx, d_ci, sizeof(uint32_t) * w->nblocks, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && w->nblocks)
        e = cudaMemcpy(values, w->d_values, sizeof(float) * w->nblocks * w->block_h,
                       cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "spcv_cu_unpack");
    cudaFree(d_rp);
    cudaFree(d_ci);
    cudaSetDevice(prev);
    return rc;
}

extern "C" int spcv_cu_weights_info(const spcv_cu_weights* w, int* rows, int* cols, int* block_h,
                                    size_t* nblocks, int* row_slots, int* device) {
    if (!w) return fail(SPCV_ERR_INVALID, "spcv_cu_weights_info: null weights");
    if (rows) *rows = w->rows;
    if (cols) *cols = w->cols;
    if (block_h) *block_h = w->block_h;
    if (nblocks) *nblocks = w->nblocks;
    if (row_slots) *row_slots = w->G;
    if (device) *device = w->device;
    return SPCV_OK;
}

extern "C" void spcv_cu_free(spcv_cu_weights* w) { free_weights(w); }

// ------------------------------------------------------------------- launch

namespace {

struct Geometry {
    long long ntiles;      // column tiles
    int split;             // CTAs sharing every tile (grid.y)
    int nwarps;            // warps per CTA
    size_t smem;           // dynamic shared memory per CTA
    long long tail_start;  // first tile of the split tail (== ntiles: none)
    int tail_split;        // CTAs per tail tile (grid.x counts them)
    long long grid_x;
};

template <typename Kern>
Geometry geometry(Kern kern, const spcv_cu_weights* w, long long ntiles, int sms);

template <int BH, int LPR, int NF, bool STRICT, bool VEC>
int launch_one(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
               cudaStream_t st) {
    auto kern = spcvk::spmm_bcsr_kernel<BH, LPR, NF, STRICT, VEC>;
    // cudaFuncSetAttribute is per device; remember which devices are done.
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load() & bit)) {
        SPCV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kSmemLimit)));
        configured.fetch_or(bit);
    }
    // Geometry depends only on (kernel, weights, tile count): cache the last one.
    static thread_local long long key[5] = {-1, -1, -1, -1, -1};
    static thread_local Geometry g;
    const long long k[5] = {ntiles, dev, w->cols, w->rows, w->T};
    if (!std::equal(k, k + 5, key)) {
        g = geometry(kern, w, ntiles, sms);
        std::copy(k, k + 5, key);
    }
    dim3 grid(static_cast<unsigned>(g.grid_x), static_cast<unsigned>(g.split));
    spcvk::KernelArgs at = a;
    at.tail_start = g.tail_start;
    at.tail_split = g.tail_split;
    kern<<<grid, g.nwarps * 32, g.smem, st>>>(at);
    SPCV_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

// Shared memory of the pipelined kernel with `ns` stages.
size_t pipe_smem_bytes(int K, int M, int T, int ns) {
    const size_t stage = static_cast<size_t>(K + 1) * T * 4 + static_cast<size_t>(T) * 8;
    return 2 * spcvk::kPipeMaxStages * 8 + ((static_cast<size_t>(M) * 4 + 127) & ~size_t{127}) +
           stage * ns;
}

// Stages of the pipelined kernel that fit (0 when fewer than two do).
int pipe_stages(const spcv_cu_weights* w) {
    for (int ns = spcvk::kPipeMaxStages; ns >= 2; --ns)
        if (pipe_smem_bytes(w->cols, w->rows, w->T, ns) <= kSmemLimit) return ns;
    return 0;
}

template <int BH, int LPR, int NF, bool STRICT>
int launch_pipe(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                int ns, cudaStream_t st) {
    auto kern = spcvk::spmm_bcsr_pipelined<BH, LPR, NF, STRICT>;
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load() & bit)) {
        SPCV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kSmemLimit)));
        configured.fetch_or(bit);
    }
    const size_t smem = pipe_smem_bytes(w->cols, w->rows, w->T, ns);
    const long long grid_x = std::min<long long>(ntiles, sms);
    dim3 grid(static_cast<unsigned>(grid_x), 1u);
    kern<<<grid, spcvk::kPipeThreads, smem, st>>>(a, ns, ntiles);
    SPCV_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

template <int BH, int LPR, int NF>
int launch_g(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long nt, int sms,
             bool strict, bool vec, cudaStream_t st) {
    // Pipelined persistent kernel when the tile ring fits >= 2 stages and there
    // are enough tiles to keep every SM streaming; else one tile per CTA.
    const int ns = vec ? pipe_stages(w) : 0;
    const char* env = std::getenv("SPCV_PIPELINE");
    // Opt-in for now: with 8 consumer warps it trails the tile kernel (profiles/).
    const bool pipe = ns >= 2 && env && std::atoi(env) != 0 && nt >= 1;
    if (pipe)
        return strict ? launch_pipe<BH, LPR, NF, true>(a, w, nt, sms, ns, st)
                      : launch_pipe<BH, LPR, NF, false>(a, w, nt, sms, ns, st);
    if (strict)
        return vec ? launch_one<BH, LPR, NF, true, true>(a, w, nt, sms, st)
                   : launch_one<BH, LPR, NF, true, false>(a, w, nt, sms, st);
    return vec ? launch_one<BH, LPR, NF, false, true>(a, w, nt, sms, st)
               : launch_one<BH, LPR, NF, false, false>(a, w, nt, sms, st);
}

template <int BH>
int launch_bh(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long nt, int sms,
              bool strict, bool vec, cudaStream_t st) {
    if constexpr (BH == 4) {
        switch (w->LPR) {
            case 16: return launch_g<BH, 16, 2>(a, w, nt, sms, strict, vec, st);
            case 8: return launch_g<BH, 8, 2>(a, w, nt, sms, strict, vec, st);
            default: return launch_g<BH, 4, 2>(a, w, nt, sms, strict, vec, st);
        }
    } else {
        switch (w->LPR) {
            case 8: return launch_g<BH, 8, 4>(a, w, nt, sms, strict, vec, st);
            case 4: return launch_g<BH, 4, 4>(a, w, nt, sms, strict, vec, st);
            default: return launch_g<BH, 2, 4>(a, w, nt, sms, strict, vec, st);
        }
    }
}

// Warps per CTA and CTAs per tile. Among 4/8/16 warps per CTA, take the
// one with the most resident warps per SM (occupancy API: shared memory and
// the kernel's real register count), preferring more, smaller CTAs on ties:
// each CTA stages its own tile, so more CTAs keep more bytes in flight. Then
// split tiles across CTAs (row split) until the grid covers the GPU.
template <typename Kern>
Geometry geometry(Kern kern, const spcv_cu_weights* w, long long ntiles, int sms) {
    Geometry g;
    g.ntiles = ntiles;
    g.smem = smem_bytes(w->cols, w->rows, w->T);
    int best = 0, per_sm = 1;
    g.nwarps = 16;
    const char* env_nw = std::getenv("SPCV_NWARPS");
    for (int nw : {4, 8, 16}) {
        if (nw * 32 > spcvk::kThreads) continue;
        if (env_nw && std::atoi(env_nw) != nw) continue;
        int ctas = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, kern, nw * 32, g.smem) != cudaSuccess)
            ctas = 0;
        if (ctas * nw > best) {
            best = ctas * nw;
            per_sm = ctas;
            g.nwarps = nw;
        }
    }
    g.split = 1;
    while (g.nwarps * g.split * 2 <= kBins && ntiles * g.split < static_cast<long long>(sms) * per_sm)
        g.split *= 2;
    if (const char* e = std::getenv("SPCV_SPLIT")) {
        const int want = std::atoi(e);
        if (want >= 1 && g.nwarps * want <= kBins && (want & (want - 1)) == 0) g.split = want;
    }
    // Tail splitting: if the last wave of CTAs is partial, split its tiles
    // across more CTAs (row slices) so it covers the SMs.
    g.tail_start = ntiles;
    g.tail_split = 1;
    const long long resident = static_cast<long long>(sms) * per_sm;
    const long long total = ntiles * g.split;
    const long long full_rounds = total / resident;
    const long long left = total - full_rounds * resident;  // CTAs in the partial round
    const char* env_tail = std::getenv("SPCV_TAIL");
    if (full_rounds >= 1 && left > 0 && !(env_tail && std::atoi(env_tail) == 0)) {
        int ts = 1;
        while (ts < 8 && g.nwarps * g.split * ts * 2 <= kBins && left * ts * 4 < resident * 3) ts *= 2;
        if (ts > 1) {
            g.tail_split = ts;
            g.tail_start = ntiles - left / g.split;
        }
    }
    g.grid_x = g.tail_start + (ntiles - g.tail_start) * g.tail_split;
    return g;
}

// Argument checks in the order of spmm_into (kernels.cpp:306-322).
int check_args(const spcv_cu_weights* w, int act_layout, int images, int act_c, int act_h,
               int act_w, size_t bias_len, int act_kind, float lo, float hi, int out_layout,
               int out_c, int out_h, int out_w, int cfg_m, int cfg_n, int mode) {
    if (!w) return fail(SPCV_ERR_INVALID, "spmm: null weights");
    if (act_kind != SPCV_ACT_NONE && act_kind != SPCV_ACT_CLAMP)
        return fail(SPCV_ERR_INVALID, "spmm: unknown activation kind");
    if (act_kind == SPCV_ACT_CLAMP && !(lo < hi))
        return fail(SPCV_ERR_INVALID, "clamp requires lo < hi");
    if (mode != SPCV_MODE_STRICT && mode != SPCV_MODE_FAST)
        return fail(SPCV_ERR_INVALID, "spmm: unknown arithmetic mode");
    if (act_layout != SPCV_LAYOUT_CHW) return fail(SPCV_ERR_LAYOUT, "spmm: activation must be CHW");
    if (w->cols != act_c)
        return fail(SPCV_ERR_SHAPE, "spmm: weight cols " + std::to_string(w->cols) +
                                        " != activation channels " + std::to_string(act_c));
    if (cfg_n != w->block_h)
        return fail(SPCV_ERR_FORMAT, "spmm: cfg out_block " + std::to_string(cfg_n) +
                                         " != matrix block height " + std::to_string(w->block_h));
    if (bias_len != 0 && bias_len != static_cast<size_t>(w->rows))
        return fail(SPCV_ERR_SHAPE, "spmm: bias length != rows");
    if (out_layout != SPCV_LAYOUT_CHW || out_c != w->rows || out_h != act_h || out_w != act_w)
        return fail(SPCV_ERR_SHAPE, "spmm: output tensor shape/layout mismatch");
    if (cfg_m != 0 && cfg_m != 4 && cfg_m != 8 && cfg_m != 16)
        return fail(SPCV_ERR_INVALID, "spmm: strip width must be 4, 8 or 16");
    if (images < 0 || act_h < 1 || act_w < 1)
        return fail(SPCV_ERR_SHAPE, "spmm: tensor dims must be >= 1");
    return SPCV_OK;
}

int launch(const spcv_cu_weights* w, const float* act, int images, int act_h, int act_w,
           const float* bias, int act_kind, float lo, float hi, float* out, int mode,
           cudaStream_t st) {
    const long long S = static_cast<long long>(act_h) * act_w;
    const long long N = S * images;
    if (N == 0) return SPCV_OK;
    if (S > 0x7FFFFFFFLL) return fail(SPCV_ERR_UNSUPPORTED, "spmm: spatial extent too large");
    if (!act || !out) return fail(SPCV_ERR_INVALID, "spmm: null tensor pointer");
    int dev = 0;
    SPCV_CUDA(cudaGetDevice(&dev));
    if (dev != w->device)
        return fail(SPCV_ERR_INVALID, "spmm: weights were packed on device " +
                                          std::to_string(w->device) + ", current device is " +
                                          std::to_string(dev));
    spcvk::KernelArgs a;
    a.act = act;
    a.out = out;
    a.bias = bias;
    a.stream = w->d_stream;
    a.bin_beg = w->d_bin_beg;
    a.N = N;
    a.K = w->cols;
    a.M = w->rows;
    a.S = static_cast<int>(S);
    a.act_kind = act_kind;
    a.lo = lo;
    a.hi = hi;
    a.tail_start = 0x7FFFFFFFFFFFFFFFLL;
    a.tail_split = 1;
    const long long ntiles = (N + w->T - 1) / w->T;
    if (ntiles > 0x7FFFFFFFLL) return fail(SPCV_ERR_UNSUPPORTED, "spmm: too many column tiles");
    const int sms = props_for(dev).sms;
    const bool vec = (S % 4 == 0) && (reinterpret_cast<uintptr_t>(act) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    const bool strict = mode == SPCV_MODE_STRICT;
    switch (w->block_h) {
        case 1: return launch_bh<1>(a, w, ntiles, sms, strict, vec, st);
        case 2: return launch_bh<2>(a, w, ntiles, sms, strict, vec, st);
        default: return launch_bh<4>(a, w, ntiles, sms, strict, vec, st);
    }
}

// Per-thread device scratch and streams of the host-tensor entry point:
// copies in (h2d), kernels (k) and copies out (d2h) run on three streams so
// that chunk c+1 uploads while chunk c computes and chunk c-1 downloads.
struct HostScratch {
    int device = -1;
    cudaStream_t h2d = nullptr, k = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_done;
    float* buf = nullptr;
    size_t cap = 0;  // floats
    void release() {
        if (buf) cudaFree(buf);
        for (cudaStream_t* s : {&h2d, &k, &d2h})
            if (*s) cudaStreamDestroy(*s), *s = nullptr;
        for (auto& e : ev_in) cudaEventDestroy(e);
        for (auto& e : ev_done) cudaEventDestroy(e);
        ev_in.clear();
        ev_done.clear();
        buf = nullptr;
        cap = 0;
    }
    ~HostScratch() { release(); }
};
thread_local HostScratch g_scratch;

constexpr size_t kHostChunkBytes = 48u << 20;  // activations + outputs per pipelined chunk

}  // namespace

extern "C" int spcv_cu_spmm_into(const spcv_cu_weights* w, const float* act, int act_layout,
                                 int images, int act_c, int act_h, int act_w, const float* bias,
                                 size_t bias_len, int act_kind, float lo, float hi, float* out,
                                 int out_layout, int out_c, int out_h, int out_w, int cfg_m,
                                 int cfg_n, int mode, void* stream) {
    g_last_error.clear();
    const int rc = check_args(w, act_layout, images, act_c, act_h, act_w, bias_len, act_kind, lo,
                              hi, out_layout, out_c, out_h, out_w, cfg_m, cfg_n, mode);
    if (rc) return rc;
    return launch(w, act, images, act_h, act_w, bias_len ? bias : nullptr, act_kind, lo, hi, out,
                  mode, static_cast<cudaStream_t>(stream));
}

extern "C" int spcv_cu_spmm_into_host(const spcv_cu_weights* w, const float* act, int act_layout,
                                      int images, int act_c, int act_h, int act_w,
                                      const float* bias, size_t bias_len, int act_kind, float lo,
                                      float hi, float* out, int out_layout, int out_c, int out_h,
                                      int out_w, int cfg_m, int cfg_n, int mode) {
    g_last_error.clear();
    int rc = check_args(w, act_layout, images, act_c, act_h, act_w, bias_len, act_kind, lo, hi,
                        out_layout, out_c, out_h, out_w, cfg_m, cfg_n, mode);
    if (rc) return rc;
    const size_t S = static_cast<size_t>(act_h) * act_w;
    const size_t n_in = S * act_c * images, n_out = S * out_c * images;
    const size_t n_bias = bias_len ? bias_len : 0;
    if (n_in + n_out == 0) return SPCV_OK;
    int prev = 0;
    SPCV_CUDA(cudaGetDevice(&prev));
    SPCV_CUDA(cudaSetDevice(w->device));
    HostScratch& hs = g_scratch;
    if (hs.device != w->device) {
        hs.release();
        hs.device = w->device;
        for (cudaStream_t* st : {&hs.h2d, &hs.k, &hs.d2h})
            SPCV_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    }
    // 16 B-aligned sub-buffers: act | out | bias
    auto up4 = [](size_t n) { return (n + 3) & ~static_cast<size_t>(3); };
    const size_t need = up4(n_in) + up4(n_out) + up4(n_bias);
    if (need > hs.cap) {
        if (hs.buf) cudaFree(hs.buf);
        hs.buf = nullptr;
        hs.cap = 0;
        SPCV_CUDA(cudaMalloc(&hs.buf, need * sizeof(float)));
        hs.cap = need;
    }
    float* d_act = hs.buf;
    float* d_out = d_act + up4(n_in);
    float* d_bias = n_bias ? d_out + up4(n_out) : nullptr;

    // Image chunks of ~kHostChunkBytes; each chunk: H2D -> kernel -> D2H.
    const size_t per_image = S * (static_cast<size_t>(act_c) + out_c) * sizeof(float);
    const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(images, kHostChunkBytes / std::max<size_t>(per_image, 1))));
    const int nchunks = images > 0 ? (images + chunk - 1) / chunk : 0;
    while (static_cast<int>(hs.ev_in.size()) < nchunks) {
        cudaEvent_t a = nullptr, b = nullptr;
        SPCV_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        SPCV_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        hs.ev_in.push_back(a);
        hs.ev_done.push_back(b);
    }
    const size_t in_img = S * act_c, out_img = S * out_c;
    if (n_bias)
        SPCV_CUDA(cudaMemcpyAsync(d_bias, bias, n_bias * sizeof(float), cudaMemcpyHostToDevice, hs.h2d));
    for (int c = 0; c < nchunks; ++c) {
        const int i0 = c * chunk, ni = std::min(chunk, images - i0);
        SPCV_CUDA(cudaMemcpyAsync(d_act + i0 * in_img, act + i0 * in_img, ni * in_img * sizeof(float),
                                  cudaMemcpyHostToDevice, hs.h2d));
        SPCV_CUDA(cudaEventRecord(hs.ev_in[c], hs.h2d));
        SPCV_CUDA(cudaStreamWaitEvent(hs.k, hs.ev_in[c], 0));
        rc = launch(w, d_act + i0 * in_img, ni, act_h, act_w, d_bias, act_kind, lo, hi,
                    d_out + i0 * out_img, mode, hs.k);
        if (rc) {
            cudaStreamSynchronize(hs.h2d);
            cudaStreamSynchronize(hs.k);
            cudaSetDevice(prev);
            return rc;
        }
        SPCV_CUDA(cudaEventRecord(hs.ev_done[c], hs.k));
        SPCV_CUDA(cudaStreamWaitEvent(hs.d2h, hs.ev_done[c], 0));
        SPCV_CUDA(cudaMemcpyAsync(out + i0 * out_img, d_out + i0 * out_img, ni * out_img * sizeof(float),
                                  cudaMemcpyDeviceToHost, hs.d2h));
    }
    SPCV_CUDA(cudaStreamSynchronize(hs.d2h));
    SPCV_CUDA(cudaStreamSynchronize(hs.k));
    cudaSetDevice(prev);
    return SPCV_OK;
}

extern "C" uint64_t spcv_cu_launch_count(void) { return g_launches.load(); }

extern "C" const char* spcv_cu_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* spcv_cu_version(void) {
    return "spcv_cu 0.1 sm_100a (strict+fast, block_h 1/2/4, row slots 1/2/4)";
}
