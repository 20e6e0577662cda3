// spcv_cu.cu — C-ABI shim (include/spcv_cu.h): weight packing, argument
// checks in the reference order, kernel selection and launch.
//
// Reference interface replaced: spcv::spmm_into (kernels.hpp:45-46,
// kernels.cpp:304-334) and the BcsrMatrix it consumes (sparse.hpp:65-79).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <list>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "spcv_internal.h"

using spcvk::kBins;
using spcvk::kMaxSplit;
using spcvk::kWarps;

namespace spcv_detail {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(SPCV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace spcv_detail

using namespace spcv_detail;

Knobs Knobs::from_env() {
    auto get = [](const char* name, long long dflt) -> long long {
        const char* e = std::getenv(name);
        return e ? std::atoll(e) : dflt;
    };
    Knobs k;
    k.steps = static_cast<int>(get("SPCV_STEPS", 0));
    k.nf = static_cast<int>(get("SPCV_NF", 0));
    k.tile_t = static_cast<int>(get("SPCV_TILE_T", 0));
    k.nwarps = static_cast<int>(get("SPCV_NWARPS", 0)) & 31;
    k.split = static_cast<int>(get("SPCV_SPLIT", 0)) & 31;
    k.tail = static_cast<int>(std::min<long long>(get("SPCV_TAIL", -1), 31));
    k.autotune = get("SPCV_AUTOTUNE", 1) != 0;
    k.jit = get("SPCV_JIT", 1) != 0;
    k.fuse_dw = get("SPCV_FUSE_DW", 0) != 0;
    k.kmajor_min_cols = get("SPCV_JIT_KMAJOR_MIN_COLS", -1);
    k.jit_warps = static_cast<int>(get("SPCV_JIT_WARPS", 0));
    k.jit_stages = static_cast<int>(get("SPCV_JIT_STAGES", 0));
    k.jit_seg_instr = static_cast<int>(get("SPCV_JIT_SEG_INSTR", 0));
    k.jit_max_segs = static_cast<int>(get("SPCV_JIT_MAX_SEGS", 0));
    k.jit_direct_maxk = static_cast<int>(get("SPCV_JIT_DIRECT_MAXK", 0));
    k.jit_interleave = static_cast<int>(get("SPCV_JIT_INTERLEAVE", 1));
    k.pass_k = static_cast<int>(get("SPCV_PASS_K", 0));
    k.small = static_cast<int>(get("SPCV_SMALL", 1));
    k.regcap = get("SPCV_REGCAP", 1) != 0;
    k.coal = static_cast<int>(get("SPCV_COAL", 1)) & 3;
    k.small_head = get("SPCV_SMALL_HEAD", 1) != 0;
    return k;
}

namespace spcvk {

// Device decode of the paper-format streams (per-block-row nnz counts,
// per-block input-channel deltas, values) back into BCSR, for the bit-exact
// pack/unpack round trip. One thread per block row after a serial prefix over
// counts (block rows <= a few thousand).
__global__ void unpack_rowptr_kernel(const uint32_t* nnz, int brows, uint32_t* row_ptr) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint32_t acc = 0;
        row_ptr[0] = 0;
        for (int r = 0; r < brows; ++r) {
            acc += nnz[r];
            row_ptr[r + 1] = acc;
        }
    }
}

__global__ void unpack_cols_kernel(const uint32_t* row_ptr, const uint32_t* delta, int brows,
                                   uint32_t* col_idx) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= brows) return;
    uint32_t col = 0;
    for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
        col += delta[b];
        col_idx[b] = col;
    }
}

}  // namespace spcvk

namespace {

struct Layout {
    int LPR, NF, T;
};

// Tile layout for K input channels. Each lane owns NF float4 quads: 8
// columns (NF=2) for block_h 4 and for layers with few output rows (M <= 96:
// little work per staged tile, so more resident warps/CTAs matter more),
// 16 columns (NF=4) otherwise (halves the weight-stream share of the pipe) (halves the weight-stream share of
// the shared-memory pipe). The widest tile T whose shared-memory footprint
// leaves room for two CTAs per SM wins, else the widest that fits one CTA.
// SPCV_NF=2|4 and SPCV_TILE_T=32|64|128 override (tuning aids).
Layout choose_layout(int K, int M, int block_h, const Knobs& kn) {
    int NF = (block_h == 4 || M <= 96) ? 2 : 4;
    if (block_h != 4 && (kn.nf == 2 || kn.nf == 4)) NF = kn.nf;  // tuning aid
    const int lprs_nf4[3] = {8, 4, 2};
    const int lprs_nf2[3] = {16, 8, 4};
    const int* lprs = NF == 2 ? lprs_nf2 : lprs_nf4;
    if (kn.tile_t) {
        const int want = kn.tile_t;
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
    cudaFree(w->d_stream_fast);
    cudaFree(w->d_bin_beg_fast);
    cudaFree(w->d_row_ptr);
    cudaFree(w->d_col_idx);
    cudaFree(w->d_head_col);
    cudaFree(w->d_head_val);
    for (spcv_cu_weights* p : w->parts) free_weights(p);
    jit_release(w);
    delete w;
}

}  // namespace

// ------------------------------------------------------------------ packing

namespace {

// Input channels per pass when K is too wide for one [K][T] tile.
constexpr int kPassChannels = 1024;

int pack_impl(int rows, int cols, int block_h, const uint32_t* row_ptr, size_t row_ptr_len,
              const uint32_t* col_idx, size_t nblocks, const float* values, size_t nvalues,
              spcv_cu_weights** out, bool pass_part);

// A matrix too wide for one shared-memory tile: packed as parts over channel
// ranges [k0, k0 + kPassChannels), column indices rebased, every block row
// present in every part (empty where it has no block in the range). The
// paper-format streams of the whole matrix are kept for spcv_cu_unpack.
int pack_passes(int rows, int cols, int block_h, const uint32_t* row_ptr, const uint32_t* col_idx, size_t nblocks,
                const float* values, spcv_cu_weights** out, int pass_channels) {
    const int brows = rows / block_h;
    auto* w = new (std::nothrow) spcv_cu_weights;
    if (!w) return fail(SPCV_ERR_CUDA, "spcv_cu_pack: out of host memory");
    w->rows = rows;
    w->cols = cols;
    w->block_h = block_h;
    w->brows = brows;
    w->nblocks = nblocks;
    w->knobs = Knobs::from_env();
    cudaGetDevice(&w->device);
    int rc = SPCV_OK;
    for (int k0 = 0; k0 < cols && rc == SPCV_OK; k0 += pass_channels) {
        const uint32_t k1 = static_cast<uint32_t>(std::min(cols, k0 + pass_channels));
        std::vector<uint32_t> rp(static_cast<size_t>(brows) + 1, 0), ci;
        std::vector<float> va;
        for (int r = 0; r < brows; ++r) {
            for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b)
                if (col_idx[b] >= static_cast<uint32_t>(k0) && col_idx[b] < k1) {
                    ci.push_back(col_idx[b] - static_cast<uint32_t>(k0));
                    for (int i = 0; i < block_h; ++i) va.push_back(values[static_cast<size_t>(b) * block_h + i]);
                }
            rp[r + 1] = static_cast<uint32_t>(ci.size());
        }
        spcv_cu_weights* part = nullptr;
        rc = pack_impl(rows, static_cast<int>(k1) - k0, block_h, rp.data(), rp.size(), ci.data(), ci.size(),
                       va.data(), va.size(), &part, true);
        if (rc == SPCV_OK) {
            part->jit_eligible = false;  // passes run the tile kernel (it continues sums)
            w->parts.push_back(part);
            w->part_k0.push_back(k0);
        }
    }
    if (rc == SPCV_OK) {
        w->G = w->parts[0]->G;
        w->LPR = w->parts[0]->LPR;
        w->NF = w->parts[0]->NF;
        w->T = w->parts[0]->T;
        std::vector<uint32_t> nnz(brows), delta(nblocks);
        for (int r = 0; r < brows; ++r) {
            nnz[r] = row_ptr[r + 1] - row_ptr[r];
            uint32_t prev = 0;
            for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
                delta[b] = col_idx[b] - prev;
                prev = col_idx[b];
            }
        }
        if ((rc = upload(&w->d_nnz, nnz.data(), nnz.size())) == SPCV_OK &&
            (rc = upload(&w->d_delta, delta.data(), delta.size())) == SPCV_OK)
            rc = upload(&w->d_values, values, nblocks * static_cast<size_t>(block_h));
    }
    if (rc != SPCV_OK) {
        free_weights(w);
        return rc;
    }
    *out = w;
    return SPCV_OK;
}

}  // namespace

extern "C" int spcv_cu_pack(int rows, int cols, int block_h, const uint32_t* row_ptr,
                            size_t row_ptr_len, const uint32_t* col_idx, size_t nblocks,
                            const float* values, size_t nvalues, spcv_cu_weights** out) {
    return pack_impl(rows, cols, block_h, row_ptr, row_ptr_len, col_idx, nblocks, values, nvalues, out, false);
}

namespace {

int pack_impl(int rows, int cols, int block_h, const uint32_t* row_ptr, size_t row_ptr_len,
              const uint32_t* col_idx, size_t nblocks, const float* values, size_t nvalues,
              spcv_cu_weights** out, bool pass_part) {
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

    // channel-pass parts: the one layout launch.cuh instantiates for them
    const Knobs kn = Knobs::from_env();
    const Layout lay = pass_part ? (block_h == 4 ? Layout{4, 2, 32} : Layout{2, 4, 32})
                                 : choose_layout(cols, rows, block_h, kn);
    if (lay.LPR == 0 || cols >= 0xFFFF)
        return pack_passes(rows, cols, block_h, row_ptr, col_idx, nblocks, values, out, kPassChannels);
    if (!pass_part && kn.pass_k > 0 && cols > kn.pass_k)  // tuning aid: narrower passes
        return pack_passes(rows, cols, block_h, row_ptr, col_idx, nblocks, values, out, kn.pass_k);
    const int G = 32 / lay.LPR;
    const int T = lay.T;
    const int BH = block_h;
    if (brows >= static_cast<int>(spcvk::kNoRow))
        return fail(SPCV_ERR_UNSUPPORTED, "spcv_cu_pack: too many block rows");
    // Steps per chunk: rows are padded to a multiple of STEPS (zero row,
    // weight -0.0f) and the max over a row group, so short rows (mean < 16
    // blocks) use 2-step chunks. Measured per layer (profiles/r1_notes.md):
    // in strict mode unstructured square/expanding matrices up to 512 rows
    // also run faster with 2 (MBv1 512x512: 218 -> 207 us) while projections
    // (rows < cols), 1024-row matrices and block heights 2/4 keep 4; in fast
    // mode 4 wins for all but short rows (FFMA leaves more issue slots for
    // the index work). When the two modes differ both streams are packed.
    // SPCV_STEPS=2|4 overrides both.
    const bool short_rows = nblocks < static_cast<size_t>(16) * brows;
    const bool small_square = block_h == 1 && rows <= 512 && rows >= cols;
    int steps_strict = (short_rows || small_square) ? 2 : 4;
    int steps_fast = short_rows ? 2 : 4;
    if (kn.steps == 2 || kn.steps == 4) steps_strict = steps_fast = kn.steps;
    if (pass_part) steps_strict = steps_fast = 4;

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
    // neighbours (similar lengths -> little predication), then balance the
    // groups over kBins bins at every power-of-two level (see build below).
    std::vector<int> order(brows);
    for (int r = 0; r < brows; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return nnz[a] > nnz[b]; });
    const int ngroups = (brows + G - 1) / G;

    // One execution stream for STEPS steps per chunk.
    struct Built {
        std::vector<unsigned char> stream;
        std::vector<uint32_t> bin_beg;
        size_t nchunks = 0;
    };
    auto build = [&](int STEPS, Built& out) {
        const int group_overhead = STEPS == 2 ? 3 : 2;  // a header + epilogue pass costs about this many chunks
        std::vector<int> gchunks(ngroups);
        for (int g = 0; g < ngroups; ++g) {
            uint32_t mx = 0;
            for (int s = 0; s < G; ++s) {
                const int k = g * G + s;
                if (k < brows) mx = std::max(mx, nnz[order[k]]);
            }
            gchunks[g] = static_cast<int>((mx + STEPS - 1) / STEPS);
        }
        // Longest group first, each one walked down the binary tree over the
        // kBins bins into the lighter half at every level: any aligned range
        // of kBins / V bins is the work of one of V virtual warps (warps per
        // CTA x CTAs sharing a tile), so every V the launcher may pick gets
        // balanced loads. (A flat LPT over the bins balances nothing while
        // there are fewer groups than bins: the longest group of every round
        // of 16 landed on warp 0 — measured on the per-CTA timeline, the
        // slowest warp finished 9-33 % after the first: pw13 +4.0 of 46 us,
        // c5 @90 % +23 of 71 us.)
        std::vector<std::vector<int>> bins(kBins);
        std::vector<long long> load(2 * kBins, 0);  // heap-ordered tree: node 1 = all bins, leaves kBins..2*kBins-1
        std::vector<int> gorder(ngroups);
        for (int g = 0; g < ngroups; ++g) gorder[g] = g;
        std::stable_sort(gorder.begin(), gorder.end(),
                         [&](int a, int b) { return gchunks[a] > gchunks[b]; });
        for (int g : gorder) {
            const long long cost = gchunks[g] + group_overhead;  // header + epilogue, in chunks
            int node = 1;
            while (node < kBins) {
                load[node] += cost;
                node = 2 * node + (load[2 * node] <= load[2 * node + 1] ? 0 : 1);
            }
            load[node] += cost;
            bins[node - kBins].push_back(g);
        }

        // Chunk (spmm_kernel.cuh, Fmt): index area G x STEPS u16 (padded to 16 B),
        // value area G x STEPS*BH f32 in 16 B units [unit][slot] (8 B per slot
        // when STEPS*BH == 2). Headers: first index word kHeaderHi | block_row.
        const int NI = STEPS / 2, NV = STEPS * BH;
        const size_t IB = (static_cast<size_t>(G) * NI * 4 + 15) / 16 * 16;
        const size_t CB = IB + static_cast<size_t>(G) * NV * 4;
        size_t total = 0;
        for (int g = 0; g < ngroups; ++g) total += 1 + gchunks[g];
        std::vector<unsigned char>& stream = out.stream;
        stream.assign((total + 1) * CB, 0);  // + one padding chunk (ring stand-in past the end)
        out.bin_beg.assign(kBins + 1, 0);
        size_t cur = 0;
        auto idx_word = [&](size_t chunk, int slot, int wi) -> uint32_t* {
            return reinterpret_cast<uint32_t*>(stream.data() + chunk * CB + (slot * NI + wi) * 4);
        };
        auto val_word = [&](size_t chunk, int slot, int f) -> float* {
            unsigned char* base = stream.data() + chunk * CB + IB;
            if (NV == 2) return reinterpret_cast<float*>(base + slot * 8 + f * 4);
            return reinterpret_cast<float*>(base + ((f / 4) * G + slot) * 16 + (f % 4) * 4);
        };
        for (int b = 0; b < kBins; ++b) {
            out.bin_beg[b] = static_cast<uint32_t>(cur);
            for (int g : bins[b]) {
                const int nch = gchunks[g];
                for (int s = 0; s < G; ++s) {
                    const int k = g * G + s;
                    *idx_word(cur, s, 0) =
                        spcvk::kHeaderHi | (k < brows ? static_cast<uint32_t>(order[k]) : spcvk::kNoRow);
                }
                ++cur;
                for (int c = 0; c < nch; ++c, ++cur) {
                    for (int s = 0; s < G; ++s) {
                        const int k = g * G + s;
                        const int br = k < brows ? order[k] : -1;
                        for (int t = 0; t < STEPS; ++t) {
                            // Padding steps read the zero row K with weight -0.0f, which
                            // leaves any accumulator bit-identical (see spmm_kernel.cuh).
                            uint32_t idx = static_cast<uint32_t>(cols);
                            const uint32_t e = static_cast<uint32_t>(STEPS * c + t);
                            const bool real = br >= 0 && e < nnz[br];
                            const uint32_t blk = real ? row_ptr[br] + e : 0;
                            if (real) idx = col_idx[blk];
                            uint32_t* w = idx_word(cur, s, t / 2);
                            *w |= (t & 1) ? (idx << 16) : idx;
                            for (int i = 0; i < BH; ++i)
                                *val_word(cur, s, t * BH + i) =
                                    real ? values[static_cast<size_t>(blk) * BH + i] : -0.0f;
                        }
                    }
                }
            }
        }
        out.bin_beg[kBins] = static_cast<uint32_t>(cur);
        out.nchunks = cur;
    };
    Built bs, bf;
    build(steps_strict, bs);
    if (steps_fast != steps_strict) build(steps_fast, bf);
    if (bs.nchunks > 0xFFFFFFF0ull || bf.nchunks > 0xFFFFFFF0ull)
        return fail(SPCV_ERR_UNSUPPORTED, "spcv_cu_pack: stream too large");

    auto* w = new (std::nothrow) spcv_cu_weights;
    if (!w) return fail(SPCV_ERR_CUDA, "spcv_cu_pack: out of host memory");
    w->rows = rows;
    w->cols = cols;
    w->block_h = block_h;
    w->brows = brows;
    w->G = G;
    w->STEPS = steps_strict;
    w->STEPS_fast = steps_fast;
    w->LPR = lay.LPR;
    w->NF = lay.NF;
    w->T = T;
    w->nblocks = nblocks;
    w->nchunks = bs.nchunks;
    w->knobs = kn;
    cudaGetDevice(&w->device);
    // Small-K matrices also get a weight-specialised kernel (jit.cu), compiled
    // on first use. SPCV_JIT=0 disables it, so the tile kernel runs everywhere.
    {
        w->jit_eligible = kn.jit && nvalues <= kJitMaxWeights;
        if (w->jit_eligible) {
            w->h_row_ptr.assign(row_ptr, row_ptr + brows + 1);
            w->h_col_idx.assign(col_idx, col_idx + nblocks);
            w->h_values.assign(values, values + nvalues);
        }
    }
    // head table of the few-column kernel: each block row's first 32 blocks
    const size_t head_rows = kn.small_head ? static_cast<size_t>(brows) : 0;
    std::vector<uint32_t> head_col(head_rows * 32, ~0u);
    std::vector<float> head_val(head_rows * 32 * BH, 0.0f);
    for (int r = 0; r < static_cast<int>(head_rows); ++r)
        for (uint32_t b = row_ptr[r], i = 0; b < row_ptr[r + 1] && i < 32; ++b, ++i) {
            head_col[static_cast<size_t>(r) * 32 + i] = col_idx[b];
            for (int j = 0; j < BH; ++j)
                head_val[(static_cast<size_t>(r) * 32 + i) * BH + j] = values[static_cast<size_t>(b) * BH + j];
        }
    int rc = SPCV_OK;
    if ((head_rows && ((rc = upload(&w->d_head_col, head_col.data(), head_col.size())) ||
                       (rc = upload(&w->d_head_val, head_val.data(), head_val.size())))) ||
        (rc = upload(&w->d_nnz, nnz.data(), nnz.size())) ||
        (rc = upload(&w->d_delta, delta.data(), delta.size())) ||
        (rc = upload(&w->d_values, values, nvalues)) ||
        (rc = upload(&w->d_stream, reinterpret_cast<const uint4*>(bs.stream.data()), bs.stream.size() / 16)) ||
        (rc = upload(&w->d_bin_beg, bs.bin_beg.data(), bs.bin_beg.size())) ||
        (rc = upload(&w->d_row_ptr, row_ptr, static_cast<size_t>(brows) + 1)) ||
        (rc = upload(&w->d_col_idx, col_idx, nblocks)) ||
        (steps_fast != steps_strict &&
         ((rc = upload(&w->d_stream_fast, reinterpret_cast<const uint4*>(bf.stream.data()),
                       bf.stream.size() / 16)) ||
          (rc = upload(&w->d_bin_beg_fast, bf.bin_beg.data(), bf.bin_beg.size()))))) {
        free_weights(w);
        return rc;
    }
    *out = w;
    return SPCV_OK;
}

}  // namespace

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

extern "C" int spcv_cu_weights_kernel(spcv_cu_weights* w, int mode, int* kernel) {
    g_last_error.clear();
    // probe with the plain spmm_into shape (bias, clamp, all rows)
    if (!w || !kernel) return fail(SPCV_ERR_INVALID, "spcv_cu_weights_kernel: null argument");
    if (mode != SPCV_MODE_STRICT && mode != SPCV_MODE_FAST)
        return fail(SPCV_ERR_INVALID, "spcv_cu_weights_kernel: unknown arithmetic mode");
    *kernel = SPCV_KERNEL_TILE;
    if (w->jit_eligible) {
        int prev = 0;
        cudaGetDevice(&prev);
        SPCV_CUDA(cudaSetDevice(w->device));
        JitKey key;
        key.strict = mode == SPCV_MODE_STRICT;
        key.clamp = true;
        key.bias = true;
        key.vec = true;
        key.m_out = w->rows;
        key.sms = props_for(w->device).sms;
        jit_geometry(key, w->knobs);
        if (jit_prepare(w, key)) *kernel = SPCV_KERNEL_JIT;
        cudaSetDevice(prev);
    }
    return SPCV_OK;
}

#ifdef SPCV_TIMELINE
// Timeline builds only (tools/timeline.py): device buffer of 8 u64 per CTA of the next tile-kernel launches.
static unsigned long long* g_timeline = nullptr;
extern "C" void spcvx_set_timeline(unsigned long long* buf) { g_timeline = buf; }
#endif

// ------------------------------------------------------------------- launch
namespace {
int pick_kernel(const spcv_cu_weights* w, long long N, long long S, long long ntiles, int sms, bool vec, bool pass,
                bool strict, bool clamp, bool has_bias, const float* residual, uintptr_t act, uintptr_t out,
                int m_out, const JitVariant** jv);
}  // namespace

extern "C" int spcv_cu_weights_kernel_for(spcv_cu_weights* w, int mode, int images, int act_h, int act_w,
                                          int* kernel) {
    g_last_error.clear();
    if (!w || !kernel) return fail(SPCV_ERR_INVALID, "spcv_cu_weights_kernel_for: null argument");
    if (mode != SPCV_MODE_STRICT && mode != SPCV_MODE_FAST)
        return fail(SPCV_ERR_INVALID, "spcv_cu_weights_kernel_for: unknown arithmetic mode");
    if (images < 0 || act_h < 1 || act_w < 1) return fail(SPCV_ERR_SHAPE, "spcv_cu_weights_kernel_for: bad dims");
    *kernel = SPCV_KERNEL_TILE;
    if (!w->parts.empty()) return SPCV_OK;  // channel passes: the tile kernel
    int prev = 0;
    cudaGetDevice(&prev);
    SPCV_CUDA(cudaSetDevice(w->device));
    const long long S = static_cast<long long>(act_h) * act_w;
    const long long N = S * images;
    const long long ntiles = (N + w->T - 1) / w->T;
    const int sms = props_for(w->device).sms;
    const JitVariant* jv = nullptr;
    // the spmm_into call shape on 16 B-aligned tensors: bias, clamp, all rows
    int k = pick_kernel(w, N, S, ntiles, sms, S % 4 == 0, false, mode == SPCV_MODE_STRICT, true, true, nullptr,
                        0, 0, w->rows, &jv);
    if (k == SPCV_KERNEL_JIT && !jit_build(w, jv)) k = SPCV_KERNEL_TILE;  // launch()'s fallback after a failed compile
    *kernel = k;
    cudaSetDevice(prev);
    return SPCV_OK;
}

namespace {

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

// Autotuned launch geometry. The last, partial round of column tiles can run
// unsplit or split 2 or 4 ways by rows; with few tiles (fewer than two per SM:
// small batches, the per-GPU shards of a batch partitioned over GPUs) the
// number of CTAs sharing every tile (row split) matters too. Which is fastest
// depends on the layer (measured: c3 at 2-3 tiles per SM 7 % faster unsplit,
// MBv1 pw12 at the same tile count 25 % slower; MBv1 at 32 images per GPU the
// best row split differs per layer, 9 % over the heuristic), and every choice
// gives the same bits (the per-row arithmetic does not depend on the split).
// The first call of a (weights, columns, mode, layout) shape times the
// candidates with events on its stream (two launches each after one warm-up)
// and caches the winner in the weights. Not tuned (heuristic) when
// SPCV_AUTOTUNE=0 or SPCV_TAIL is set; a shape first seen with an output
// overlapping its residual (a repeated launch would re-add it) or inside a
// stream capture uses the heuristic until an eligible call has tuned it.
struct TunedGeometry {
    int tail = -1;   // -1: heuristic
    int split = 0;   // 0: heuristic
    int coal = 0;    // 1: the coalesced-epilogue build (unaligned layouts)
};

template <typename Run>
TunedGeometry tuned_geometry(const spcv_cu_weights* w, const spcvk::KernelArgs& a, long long N, long long ntiles,
                             int sms, bool strict, bool vec, bool coal_ok, cudaStream_t st, Run&& run) {
    TunedGeometry none;
    none.coal = coal_ok && w->knobs.coal == 2;
    if (!w->knobs.autotune || w->knobs.tail >= 0) return none;
    const long long key = N * 8 + (strict ? 4 : 0) + (vec ? 2 : 0);
    {
        std::lock_guard<std::mutex> lk(w->tune_mu);
        for (const auto& kv : w->tuned_tail)
            if (kv.first == key)  // also inside a capture
                return TunedGeometry{kv.second % 64 - 1, kv.second / 64 % 64, coal_ok ? kv.second / 4096 : 0};
    }
    if (a.acc_in) return none;  // a later channel pass reads out: not repeatable in place
    if (a.residual) {  // repeated launches are idempotent unless out overlaps the residual
        const size_t bytes = static_cast<size_t>(N / a.S) * a.M_out * a.S * sizeof(float);
        const char* r0 = reinterpret_cast<const char*>(a.residual);
        const char* o0 = reinterpret_cast<const char*>(a.out);
        if (r0 < o0 + bytes && o0 < r0 + bytes) return none;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return none;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        if (e0) cudaEventDestroy(e0);
        return none;
    }
    std::vector<TunedGeometry> cands = {{-1, 0, none.coal}, {0, 0, none.coal}, {2, 0, none.coal}, {4, 0, none.coal}};
    if (ntiles < 2LL * sms && w->knobs.split == 0)  // few tiles: the row split too
        for (int sp : {1, 2, 4, 8}) cands.push_back(TunedGeometry{-1, sp, none.coal});
    if (coal_ok && w->knobs.coal == 1) {  // unaligned layout: each geometry with the coalesced epilogue too
        const size_t n = cands.size();
        for (size_t i = 0; i < n; ++i) cands.push_back(TunedGeometry{cands[i].tail, cands[i].split, 1});
    }
    TunedGeometry best;
    float best_ms = 0.0f;
    uint64_t runs = 0;  // tuning launches are not the caller's work: not counted
    for (const TunedGeometry& cand : cands) {
        spcvk::KernelArgs t = a;
        t.tail_pref = cand.tail;
        t.split_pref = cand.split;
        t.coal = cand.coal;
        if (run(t) != SPCV_OK) continue;  // warm-up (geometry, L2)
        ++runs;
        cudaEventRecord(e0, st);
        const int r1 = run(t), r2 = run(t);
        runs += (r1 == SPCV_OK) + (r2 == SPCV_OK);
        cudaEventRecord(e1, st);
        float ms = 0.0f;
        if (r1 != SPCV_OK || r2 != SPCV_OK || cudaEventSynchronize(e1) != cudaSuccess ||
            cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess)
            continue;
        if (best_ms == 0.0f || ms < best_ms * 0.98f) best = cand, best_ms = ms;  // 2 %: stay with the heuristic on ties
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    g_launches.fetch_sub(runs, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lk(w->tune_mu);
    w->tuned_tail.emplace_back(key, best.coal * 4096 + best.split * 64 + best.tail + 1);
    return best;
}

// Which kernel serves a call (spcv_cu_weights_kernel_for reports the same choice):
//  * JIT — weight-specialised code (small K; the k-major variant only with
//    enough column groups for its persistent CTAs: below that the other
//    kernels' finer work units win — measured: c1, 784 columns, 24 vs 17 us;
//    MBv2 384->64 @14x14 x128, 25088 columns in 2 segments, 53 vs 38 us);
//    decided from the plan, so a variant that would not run is never compiled;
//  * SMALL — fewer column tiles than SMs and at most kSmallMaxProducts
//    products (batch 1, small planes): a warp per block row x 32 columns,
//    gathers from global memory (small.cu);
//  * TILE — everything else (any K, any layout, channel passes).
int pick_kernel(const spcv_cu_weights* w, long long N, long long S, long long ntiles, int sms, bool vec, bool pass,
                bool strict, bool clamp, bool has_bias, const float* residual, uintptr_t act, uintptr_t out,
                int m_out, const JitVariant** jv) {
    *jv = nullptr;
    const Knobs& kn = w->knobs;
    if (w->jit_eligible) {
        JitKey key;
        key.strict = strict;
        key.clamp = clamp;
        key.bias = has_bias;
        key.res = residual != nullptr;
        key.vec = S % 4 == 0 && act % 16 == 0 && out % 8 == 0 && reinterpret_cast<uintptr_t>(residual) % 8 == 0;
        key.m_out = m_out;
        key.sms = sms;
        jit_geometry(key, kn);
        if (const JitVariant* p = jit_plan(w, key)) {
            const long long min_cols = kn.kmajor_min_cols >= 0
                                           ? kn.kmajor_min_cols
                                           : 32LL * p->cpl * sms * key.warps / std::max(1, p->segments);
            if (p->direct || N >= min_cols) {
                *jv = p;
                return SPCV_KERNEL_JIT;
            }
        }
    }
    // (products bound: the few-column kernel gathers through L1/L2 without
    // reuse; beyond a few million products the staged tiles win — measured:
    // MBv2 160->960 @7x7 x128, 144 M products, 133 vs 53 us)
    if (!pass && kn.small && w->d_row_ptr && w->brows <= 65535 * 4 &&
        (kn.small > 1 || (ntiles < sms && static_cast<double>(w->nblocks) * w->block_h * N <= kSmallMaxProducts)))
        return SPCV_KERNEL_SMALL;
    return SPCV_KERNEL_TILE;
}

int launch(const spcv_cu_weights* w, const float* act, int images, int act_h, int act_w,
           const float* bias, int act_kind, float lo, float hi, float* out, int mode,
           cudaStream_t st, int out_rows = -1, const float* residual = nullptr,
           const float* acc_in = nullptr, int k_img = -1) {
    const long long S = static_cast<long long>(act_h) * act_w;
    const long long N = S * images;
    if (N == 0) return SPCV_OK;
    if (S > 0x7FFFFFFFLL) return fail(SPCV_ERR_UNSUPPORTED, "spmm: spatial extent too large");
    if (!act || !out) return fail(SPCV_ERR_INVALID, "spmm: null tensor pointer");
    if (!w->parts.empty()) {
        // Channel passes in order: the first starts from the bias and stores raw
        // sums into out, each next continues from out; the clamp and the
        // residual belong to the last. Every output still sums its terms in the
        // reference order (bias, channels ascending): bit-exact in strict mode.
        const size_t P = w->parts.size();
        for (size_t p = 0; p < P; ++p) {
            const bool last = p + 1 == P;
            const int rc = launch(w->parts[p], act + static_cast<long long>(w->part_k0[p]) * S, images, act_h,
                                  act_w, p == 0 ? bias : nullptr, last ? act_kind : SPCV_ACT_NONE, lo, hi, out,
                                  mode, st, out_rows, last ? residual : nullptr, p == 0 ? nullptr : out, w->cols);
            if (rc != SPCV_OK) return rc;
        }
        return SPCV_OK;
    }
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
    const bool fast_stream = mode == SPCV_MODE_FAST && w->d_stream_fast != nullptr;
    a.stream = fast_stream ? w->d_stream_fast : w->d_stream;
    a.bin_beg = fast_stream ? w->d_bin_beg_fast : w->d_bin_beg;
    a.steps = mode == SPCV_MODE_FAST ? w->STEPS_fast : w->STEPS;
    a.N = N;
    a.K = w->cols;
    a.K_img = k_img < 0 ? w->cols : k_img;
    a.acc_in = acc_in;
    a.M = w->rows;
    a.M_out = out_rows < 0 ? w->rows : out_rows;
    a.residual = residual;
    a.S = static_cast<int>(S);
    a.act_kind = act_kind;
    a.lo = lo;
    a.hi = hi;
    a.tail_start = 0x7FFFFFFFFFFFFFFFLL;
    a.tail_split = 1;
    a.tail_pref = -1;
    a.split_pref = 0;
    a.one2 = 0x3f8000003f800000ULL;
    a.coal = 0;
#ifdef SPCV_TIMELINE
    a.tl = g_timeline;
#endif
    const long long ntiles = (N + w->T - 1) / w->T;
    if (ntiles > 0x7FFFFFFFLL) return fail(SPCV_ERR_UNSUPPORTED, "spmm: too many column tiles");
    const int sms = props_for(dev).sms;
    const bool vec = (S % 4 == 0) && (reinterpret_cast<uintptr_t>(act) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(residual) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(acc_in) % 16 == 0);
    const bool strict = mode == SPCV_MODE_STRICT;
    const JitVariant* jv = nullptr;
    const int kind = pick_kernel(w, N, S, ntiles, sms, vec, acc_in != nullptr || a.K_img != a.K, strict,
                                 act_kind == SPCV_ACT_CLAMP, bias != nullptr, residual,
                                 reinterpret_cast<uintptr_t>(act), reinterpret_cast<uintptr_t>(out), a.M_out, &jv);
    if (kind == SPCV_KERNEL_JIT) {
        // A failed compile (recorded, never retried) falls back to the other kernels.
        if (const JitVariant* v = jit_build(w, jv)) return jit_launch(v, a, st);
    }
    if (kind == SPCV_KERNEL_SMALL) {
        const int rc = launch_small(w, a, strict, st);
        if (rc != SPCV_ERR_UNSUPPORTED) return rc;
        g_last_error.clear();
    }
    auto run = [&](const spcvk::KernelArgs& args) {
        switch (w->block_h) {
            case 1: return launch_bh1(args, w, ntiles, sms, strict, vec, st);
            case 2: return launch_bh2(args, w, ntiles, sms, strict, vec, st);
            default: return launch_bh4(args, w, ntiles, sms, strict, vec, st);
        }
    };
    // Unaligned layouts (H*W % 4 != 0 or unaligned tensors): the coalesced-epilogue
    // build is a candidate while its per-warp scratch fits next to the tile.
    const bool coal_ok = !vec && w->knobs.coal != 0 && !acc_in && a.K_img == a.K &&
                         smem_bytes(w->cols, (w->rows + 3) & ~3, w->T) +
                                 16 * sizeof(float) * spcvk::coal_scratch_floats(w->G, w->T) <=
                             kSmemLimit;
    const TunedGeometry tg = tuned_geometry(w, a, N, ntiles, sms, strict, vec, coal_ok, st, run);
    a.tail_pref = tg.tail;
    a.split_pref = tg.split;
    a.coal = tg.coal;
    return run(a);
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

size_t host_chunk_bytes() {
    static const size_t b = [] {
        const char* e = std::getenv("SPCV_HOST_CHUNK_MB");
        const long v = e ? std::atol(e) : 0;
        return v > 0 ? static_cast<size_t>(v) << 20 : kHostChunkBytes;
    }();
    return b;
}

bool host_ramp() {
    static const bool r = [] {
        const char* e = std::getenv("SPCV_HOST_RAMP");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return r;
}

// Image chunks of the host-buffer entry point: chunk = as many images as fit
// `budget` bytes (at least 1). With the ramp, the schedule starts and ends
// with 1/8, 1/4, 1/2 of a chunk (the first kernel starts early, the last
// download is short) when a chunk is large enough for those to be real
// fractions. The sizes are positive and always sum to `images`.
std::vector<int> host_chunks(int images, size_t per_image, size_t budget, bool ramp) {
    std::vector<int> sizes;
    if (images <= 0) return sizes;
    const int chunk = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>(static_cast<size_t>(images), budget / std::max<size_t>(per_image, 1))));
    std::vector<int> head;
    if (ramp && chunk >= 8 && images >= 4 * chunk)
        for (int f : {8, 4, 2}) head.push_back(chunk / f);
    int left = images;
    for (int n : head) left -= 2 * n;  // ramp-up and the mirrored ramp-down
    sizes = head;
    while (left > 0) {
        const int n = std::min(chunk, left);
        sizes.push_back(n);
        left -= n;
    }
    sizes.insert(sizes.end(), head.rbegin(), head.rend());
    return sizes;
}

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

extern "C" int spcv_cu_spmm_layer(const spcv_cu_weights* w, const float* act, int images,
                                  int act_c, int act_h, int act_w, const float* bias,
                                  size_t bias_len, int act_kind, float lo, float hi,
                                  const float* residual, float* out, int out_c, int mode,
                                  void* stream) {
    g_last_error.clear();
    if (!w) return fail(SPCV_ERR_INVALID, "spmm_layer: null weights");
    if (act_kind != SPCV_ACT_NONE && act_kind != SPCV_ACT_CLAMP)
        return fail(SPCV_ERR_INVALID, "spmm_layer: unknown activation kind");
    if (act_kind == SPCV_ACT_CLAMP && !(lo < hi)) return fail(SPCV_ERR_INVALID, "clamp requires lo < hi");
    if (mode != SPCV_MODE_STRICT && mode != SPCV_MODE_FAST)
        return fail(SPCV_ERR_INVALID, "spmm_layer: unknown arithmetic mode");
    if (w->cols != act_c)
        return fail(SPCV_ERR_SHAPE, "spmm_layer: weight cols " + std::to_string(w->cols) +
                                        " != activation channels " + std::to_string(act_c));
    // padded rows: the stored weights may have up to block_h-1 rows beyond
    // the layer's logical output channels (netdef.cpp:496-505)
    if (out_c < 1 || out_c > w->rows || w->rows - out_c >= w->block_h)
        return fail(SPCV_ERR_SHAPE, "spmm_layer: out channels " + std::to_string(out_c) +
                                        " incompatible with " + std::to_string(w->rows) +
                                        " weight rows of block height " + std::to_string(w->block_h));
    if (bias_len != 0 && bias_len != static_cast<size_t>(out_c))
        return fail(SPCV_ERR_SHAPE, "spmm_layer: bias length != out channels");
    if (images < 0 || act_h < 1 || act_w < 1) return fail(SPCV_ERR_SHAPE, "spmm_layer: bad dims");
    return launch(w, act, images, act_h, act_w, bias_len ? bias : nullptr, act_kind, lo, hi, out, mode,
                  static_cast<cudaStream_t>(stream), out_c, residual);
}

namespace spcv_detail {

int spmm_dw_fused(const spcv_cu_weights* w, const JitDwArgs& dw, int dw_stride, const float* dw_w_host,
                  const float* dw_b_host, bool dw_clamp, int images, int out_h, int out_w,
                  const float* bias, int act_kind, float lo, float hi, const float* residual,
                  float* out, int out_c, int mode, cudaStream_t st) {
    if (!w || !w->jit_eligible) return SPCV_ERR_UNSUPPORTED;
    // Opt-in (SPCV_FUSE_DW=1): measured slower than the two separate kernels
    // on MBv1-1.0 (dw1+pw1 507 vs 550 us, dw2+pw2 392 vs 323 us): the fused
    // producer recomputes each depthwise output per 1x1 column thread and
    // becomes issue-bound.
    if (!w->knobs.fuse_dw) return SPCV_ERR_UNSUPPORTED;
    const long long S = static_cast<long long>(out_h) * out_w;
    const long long N = S * images;
    if (N == 0) return SPCV_OK;
    int dev = 0;
    SPCV_CUDA(cudaGetDevice(&dev));
    if (dev != w->device) return SPCV_ERR_UNSUPPORTED;
    JitKey key;
    key.strict = mode == SPCV_MODE_STRICT;
    key.clamp = act_kind == SPCV_ACT_CLAMP;
    key.bias = bias != nullptr;
    key.res = residual != nullptr;
    key.m_out = out_c;
    key.sms = props_for(dev).sms;
    jit_geometry(key, w->knobs);
    key.dw = true;
    key.dw_clamp = dw_clamp;
    key.dw_stride = dw_stride;
    key.dw_w = dw_w_host;
    key.dw_b = dw_b_host;
    const JitVariant* v = jit_prepare(w, key);
    if (!v || !v->direct) return SPCV_ERR_UNSUPPORTED;
    spcvk::KernelArgs a{};
    a.out = out;
    a.bias = bias;
    a.residual = residual;
    a.N = N;
    a.S = static_cast<int>(S);
    a.M_out = out_c;
    a.act_kind = act_kind;
    a.lo = key.clamp ? lo : 0.0f;
    a.hi = key.clamp ? hi : 0.0f;
    return jit_launch(v, a, st, &dw);
}

}  // namespace spcv_detail

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
    // Every exit after this point goes through done(): all three streams are
    // drained (no copy may still write the caller's `out` after we return) and
    // the caller's device is restored.
    auto done = [&](int code) {
        for (cudaStream_t s : {hs.h2d, hs.k, hs.d2h})
            if (s) cudaStreamSynchronize(s);
        cudaSetDevice(prev);
        return code;
    };
#define SPCV_HOST_CUDA(call)                                        \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return done(cuda_fail(e_, #call));   \
    } while (0)
    if (hs.device != w->device) {
        hs.release();
        for (cudaStream_t* st : {&hs.h2d, &hs.k, &hs.d2h})
            SPCV_HOST_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
        hs.device = w->device;  // only once every stream exists
    }
    // 16 B-aligned sub-buffers: act | out | bias
    auto up4 = [](size_t n) { return (n + 3) & ~static_cast<size_t>(3); };
    const size_t need = up4(n_in) + up4(n_out) + up4(n_bias);
    if (need > hs.cap) {
        if (hs.buf) cudaFree(hs.buf);
        hs.buf = nullptr;
        hs.cap = 0;
        SPCV_HOST_CUDA(cudaMalloc(&hs.buf, need * sizeof(float)));
        hs.cap = need;
    }
    float* d_act = hs.buf;
    float* d_out = d_act + up4(n_in);
    float* d_bias = n_bias ? d_out + up4(n_out) : nullptr;

    const size_t per_image = S * (static_cast<size_t>(act_c) + out_c) * sizeof(float);
    const std::vector<int> sizes = host_chunks(images, per_image, host_chunk_bytes(), host_ramp());
    const int nchunks = static_cast<int>(sizes.size());
    while (static_cast<int>(hs.ev_in.size()) < nchunks) {
        cudaEvent_t a = nullptr, b = nullptr;
        SPCV_HOST_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        hs.ev_in.push_back(a);
        SPCV_HOST_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        hs.ev_done.push_back(b);
    }
    const size_t in_img = S * act_c, out_img = S * out_c;
    if (n_bias)
        SPCV_HOST_CUDA(cudaMemcpyAsync(d_bias, bias, n_bias * sizeof(float), cudaMemcpyHostToDevice, hs.h2d));
    for (int c = 0, i0 = 0; c < nchunks; i0 += sizes[c], ++c) {
        const size_t ni = static_cast<size_t>(sizes[c]), o = static_cast<size_t>(i0);
        SPCV_HOST_CUDA(cudaMemcpyAsync(d_act + o * in_img, act + o * in_img, ni * in_img * sizeof(float),
                                       cudaMemcpyHostToDevice, hs.h2d));
        SPCV_HOST_CUDA(cudaEventRecord(hs.ev_in[c], hs.h2d));
        SPCV_HOST_CUDA(cudaStreamWaitEvent(hs.k, hs.ev_in[c], 0));
        rc = launch(w, d_act + o * in_img, sizes[c], act_h, act_w, d_bias, act_kind, lo, hi,
                    d_out + o * out_img, mode, hs.k);
        if (rc) return done(rc);
        SPCV_HOST_CUDA(cudaEventRecord(hs.ev_done[c], hs.k));
        SPCV_HOST_CUDA(cudaStreamWaitEvent(hs.d2h, hs.ev_done[c], 0));
        SPCV_HOST_CUDA(cudaMemcpyAsync(out + o * out_img, d_out + o * out_img, ni * out_img * sizeof(float),
                                       cudaMemcpyDeviceToHost, hs.d2h));
    }
    SPCV_HOST_CUDA(cudaStreamSynchronize(hs.d2h));
    SPCV_HOST_CUDA(cudaStreamSynchronize(hs.k));
#undef SPCV_HOST_CUDA
    return done(SPCV_OK);
}

// ------------------------------------------------- the reference call shape
// spmm_into(const BcsrMatrix&, ...) with host tensors, as one call. The
// reference takes the matrix by const& on every call (kernels.cpp:304); here
// it is packed once per distinct content and device and kept in a small LRU
// cache, so a caller that loops spmm_into over layers and images (run_network,
// bench_layers) never repacks, reschedules or recompiles. A hit is verified
// byte for byte against the cached host copy (the hash only finds the entry).
namespace {

struct CachedWeights {
    uint64_t hash = 0;
    int device = 0, rows = 0, cols = 0, block_h = 0;
    std::vector<uint32_t> row_ptr, col_idx;
    std::vector<float> values;
    std::shared_ptr<spcv_cu_weights> w;
    size_t bytes() const { return (row_ptr.size() + col_idx.size() + values.size()) * 4; }
};

struct WeightCache {
    std::mutex mu;
    std::list<CachedWeights> lru;  // most recently used first
    size_t bytes = 0;
    uint64_t hits = 0, misses = 0;
};
WeightCache& weight_cache() {
    static WeightCache* c = new WeightCache;  // never destroyed: no CUDA calls at exit
    return *c;
}

size_t weight_cache_limit() {
    static const size_t b = [] {
        const char* e = std::getenv("SPCV_WEIGHT_CACHE_MB");
        const long v = e ? std::atol(e) : 256;
        return static_cast<size_t>(std::max(0L, v)) << 20;
    }();
    return b;
}

uint64_t hash_words(uint64_t h, const void* data, size_t bytes) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        uint64_t v;
        std::memcpy(&v, p + i, 8);
        h = (h ^ v) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 32;
    }
    for (; i < bytes; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
    return h ^ bytes;
}

}  // namespace

extern "C" int spcv_cu_spmm_bcsr_into_host(int rows, int cols, int block_h, const uint32_t* row_ptr,
                                           size_t row_ptr_len, const uint32_t* col_idx, size_t nblocks,
                                           const float* values, size_t nvalues, const float* act,
                                           int act_layout, int images, int act_c, int act_h, int act_w,
                                           const float* bias, size_t bias_len, int act_kind, float lo,
                                           float hi, float* out, int out_layout, int out_c, int out_h,
                                           int out_w, int cfg_m, int cfg_n, int mode) {
    g_last_error.clear();
    {
        // argument checks first, in the reference order, before the matrix is read
        spcv_cu_weights shape;
        shape.rows = rows;
        shape.cols = cols;
        shape.block_h = block_h;
        const int rc = check_args(&shape, act_layout, images, act_c, act_h, act_w, bias_len, act_kind, lo, hi,
                                  out_layout, out_c, out_h, out_w, cfg_m, cfg_n, mode);
        if (rc) return rc;
    }
    int dev = 0;
    SPCV_CUDA(cudaGetDevice(&dev));
    const bool shapes_ok = row_ptr && row_ptr_len >= 1 && (nblocks == 0 || (col_idx && values));
    uint64_t h = hash_words(0x243F6A8885A308D3ull ^ static_cast<uint64_t>(dev), &rows, sizeof rows);
    h = hash_words(h, &cols, sizeof cols);
    h = hash_words(h, &block_h, sizeof block_h);
    if (shapes_ok) {
        h = hash_words(h, row_ptr, row_ptr_len * 4);
        h = hash_words(h, col_idx, nblocks * 4);
        h = hash_words(h, values, nvalues * 4);
    }
    std::shared_ptr<spcv_cu_weights> w;
    WeightCache& c = weight_cache();
    if (shapes_ok) {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.lru.begin(); it != c.lru.end(); ++it)
            if (it->hash == h && it->device == dev && it->rows == rows && it->cols == cols &&
                it->block_h == block_h && it->row_ptr.size() == row_ptr_len && it->col_idx.size() == nblocks &&
                it->values.size() == nvalues && std::memcmp(it->row_ptr.data(), row_ptr, row_ptr_len * 4) == 0 &&
                (nblocks == 0 || std::memcmp(it->col_idx.data(), col_idx, nblocks * 4) == 0) &&
                (nvalues == 0 || std::memcmp(it->values.data(), values, nvalues * 4) == 0)) {
                c.lru.splice(c.lru.begin(), c.lru, it);
                w = it->w;
                ++c.hits;
                break;
            }
    }
    if (!w) {
        spcv_cu_weights* raw = nullptr;
        const int rc = spcv_cu_pack(rows, cols, block_h, row_ptr, row_ptr_len, col_idx, nblocks, values,
                                    nvalues, &raw);
        if (rc) return rc;  // FormatError: a malformed matrix (never cached)
        w = std::shared_ptr<spcv_cu_weights>(raw, [](spcv_cu_weights* p) { spcv_cu_free(p); });
        CachedWeights e;
        e.hash = h;
        e.device = dev;
        e.rows = rows;
        e.cols = cols;
        e.block_h = block_h;
        e.row_ptr.assign(row_ptr, row_ptr + row_ptr_len);
        e.col_idx.assign(col_idx, col_idx + nblocks);
        e.values.assign(values, values + nvalues);
        e.w = w;
        std::lock_guard<std::mutex> lk(c.mu);
        ++c.misses;
        const size_t limit = weight_cache_limit();
        if (e.bytes() <= limit) {
            c.bytes += e.bytes();
            c.lru.push_front(std::move(e));
            while (c.bytes > limit && !c.lru.empty()) {  // evict the least recently used
                c.bytes -= c.lru.back().bytes();
                c.lru.pop_back();  // in-flight callers hold their own reference
            }
        }
    }
    return spcv_cu_spmm_into_host(w.get(), act, act_layout, images, act_c, act_h, act_w, bias, bias_len,
                                  act_kind, lo, hi, out, out_layout, out_c, out_h, out_w, cfg_m, cfg_n, mode);
}

extern "C" void spcv_cu_weight_cache_clear(void) {
    WeightCache& c = weight_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.lru.clear();
    c.bytes = 0;
}

extern "C" int spcv_cu_cache_stats(size_t* entries, uint64_t* hits, uint64_t* misses, uint64_t* jit_compiles,
                                   uint64_t* jit_disk_hits) {
    WeightCache& c = weight_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (entries) *entries = c.lru.size();
    if (hits) *hits = c.hits;
    if (misses) *misses = c.misses;
    if (jit_compiles) *jit_compiles = g_jit_compiles.load();
    if (jit_disk_hits) *jit_disk_hits = g_jit_cache_hits.load();
    return SPCV_OK;
}

extern "C" uint64_t spcv_cu_launch_count(void) { return g_launches.load(); }

extern "C" const char* spcv_cu_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* spcv_cu_version(void) {
    return "spcv_cu 0.1 sm_100a (strict+fast, block_h 1/2/4, row slots 1/2/4)";
}
