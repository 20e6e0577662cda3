// launch.cuh — kernel selection and launch geometry, instantiated per block
// height and staging width by launch_bh{1,2,4}.cu / launch_bh{1,2,4}u.cu (parallel compilation).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <string>

#include "spcv_internal.h"

namespace spcv_detail {

using spcvk::kBins;

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
Geometry geometry(Kern kern, const spcv_cu_weights* w, long long ntiles, int sms, int tail_pref, int split_pref,
                  int max_threads, size_t scratch_per_warp);

template <int BH, int LPR, int NF, int STEPS, bool STRICT, bool VEC, bool RES, bool ACC = false, bool CAP = false,
          bool COAL = false>
int launch_one_r(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                 cudaStream_t st) {
    auto kern = spcvk::spmm_bcsr_kernel<BH, LPR, NF, STEPS, STRICT, VEC, RES, ACC, CAP, COAL>;
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
    // Geometry depends only on (kernel, weights, tile count) and the tuning
    // knobs: cache the last one.
    static thread_local long long key[7] = {-1, -1, -1, -1, -1, -1, -2};
    static thread_local Geometry g;
    const long long k[7] = {ntiles, dev, w->cols, w->rows, w->T, w->knobs.geometry_key(),
                            a.tail_pref * 64LL + a.split_pref};
    if (!std::equal(k, k + 7, key)) {
        g = geometry(kern, w, ntiles, sms, a.tail_pref, a.split_pref, CAP ? spcvk::kCapThreads : spcvk::kThreads,
                     COAL ? sizeof(float) * spcvk::coal_scratch_floats(32 / LPR, LPR * NF * 4) : 0);
        std::copy(k, k + 7, key);
    }
    dim3 grid(static_cast<unsigned>(g.grid_x), static_cast<unsigned>(g.split));
    spcvk::KernelArgs at = a;
    at.tail_start = g.tail_start;
    at.tail_split = g.tail_split;
    SPCV_CUDA(launch_kernel(kern, grid, dim3(g.nwarps * 32), g.smem, st, at));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

// Residual-add epilogue as a separate instantiation (the plain path keeps
// its register budget).
template <int BH, int LPR, int NF, int STEPS, bool STRICT, bool VEC>
int launch_one(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
               cudaStream_t st) {
    if (a.acc_in || a.K_img != a.K) {
        // Channel passes (spcv_cu.cu: pack_passes) are packed with one layout,
        // so the continuing-sum instantiations exist only for it.
        if constexpr (STEPS == 4 && LPR == (BH == 4 ? 4 : 2) && NF == (BH == 4 ? 2 : 4))
            return a.residual ? launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, true, true>(a, w, ntiles, sms, st)
                              : launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, false, true>(a, w, ntiles, sms, st);
        else
            return fail(SPCV_ERR_UNSUPPORTED, "spmm: channel pass with an unexpected layout");
    }
    // The register-capped build (three 8-warp CTAs per SM) of the unstructured
    // 2-step kernels, where three tiles fit in shared memory and the CTA size is free.
    if constexpr (BH == 1 && STEPS == 2 && VEC && STRICT) {
        const Knobs& kn = w->knobs;
        if (kn.regcap && (kn.nwarps == 0 || kn.nwarps <= 8) &&
            3 * smem_bytes(w->cols, w->rows, w->T) <= kSmemLimit)
            return a.residual ? launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, true, false, true>(a, w, ntiles, sms, st)
                              : launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, false, false, true>(a, w, ntiles, sms, st);
    }
    // Unaligned layouts: the build whose epilogue stores row by row through a
    // per-warp scratch, where the call's first launches measured it faster
    // (spcv_cu.cu: tuned_geometry) or SPCV_COAL=2 forces it.
    if constexpr (!VEC) {
        if (a.coal)
            return a.residual
                       ? launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, true, false, false, true>(a, w, ntiles, sms, st)
                       : launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, false, false, false, true>(a, w, ntiles, sms, st);
    }
    return a.residual ? launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, true>(a, w, ntiles, sms, st)
                      : launch_one_r<BH, LPR, NF, STEPS, STRICT, VEC, false>(a, w, ntiles, sms, st);
}

// VEC (16 B-aligned layouts) and !VEC kernels live in separate translation
// units (launch_bh{1,2,4}.cu / launch_bh{1,2,4}u.cu): half the compile time each.
template <int BH, int LPR, int NF, int STEPS, bool VEC>
int launch_g(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long nt, int sms,
             bool strict, cudaStream_t st) {
    return strict ? launch_one<BH, LPR, NF, STEPS, true, VEC>(a, w, nt, sms, st)
                  : launch_one<BH, LPR, NF, STEPS, false, VEC>(a, w, nt, sms, st);
}

template <int BH, int LPR, int NF, bool VEC>
int launch_s(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long nt, int sms,
             bool strict, cudaStream_t st) {
    return a.steps == 2 ? launch_g<BH, LPR, NF, 2, VEC>(a, w, nt, sms, strict, st)
                         : launch_g<BH, LPR, NF, 4, VEC>(a, w, nt, sms, strict, st);
}

template <int BH, bool VEC>
int launch_bh(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long nt, int sms,
              bool strict, cudaStream_t st) {
    if (BH == 4 || w->NF == 2) {
        switch (w->LPR) {
            case 16: return launch_s<BH, 16, 2, VEC>(a, w, nt, sms, strict, st);
            case 8: return launch_s<BH, 8, 2, VEC>(a, w, nt, sms, strict, st);
            default: return launch_s<BH, 4, 2, VEC>(a, w, nt, sms, strict, st);
        }
    }
    if constexpr (BH != 4) {
        switch (w->LPR) {
            case 8: return launch_s<BH, 8, 4, VEC>(a, w, nt, sms, strict, st);
            case 4: return launch_s<BH, 4, 4, VEC>(a, w, nt, sms, strict, st);
            default: return launch_s<BH, 2, 4, VEC>(a, w, nt, sms, strict, st);
        }
    }
    return fail(SPCV_ERR_UNSUPPORTED, "spmm: no kernel for this layout");
}

// Warps per CTA and CTAs per tile. Among 4/8/16 warps per CTA, take the
// one with the most resident warps per SM (occupancy API: shared memory and
// the kernel's real register count), preferring more, smaller CTAs on ties:
// each CTA stages its own tile, so more CTAs keep more bytes in flight. Then
// split tiles across CTAs (row split) until the grid covers the GPU.
template <typename Kern>
Geometry geometry(Kern kern, const spcv_cu_weights* w, long long ntiles, int sms, int tail_pref, int split_pref,
                  int max_threads, size_t scratch_per_warp) {
    Geometry g;
    g.ntiles = ntiles;
    // (the per-warp output scratch of the coalesced epilogue sits after the bias, 16 B-aligned)
    const size_t base = scratch_per_warp ? smem_bytes(w->cols, (w->rows + 3) & ~3, w->T)
                                         : smem_bytes(w->cols, w->rows, w->T);
    g.smem = base + 16 * scratch_per_warp;
    int best = 0, per_sm = 1;
    g.nwarps = std::min(16, max_threads / 32);
    const Knobs& kn = w->knobs;
    for (int nw : {4, 8, 16}) {
        if (nw * 32 > max_threads) continue;
        if (kn.nwarps && kn.nwarps != nw) continue;
        int ctas = 0;
        const size_t smem_nw = base + nw * scratch_per_warp;
        if (smem_nw > kSmemLimit ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, kern, nw * 32, smem_nw) != cudaSuccess)
            ctas = 0;
        if (ctas * nw > best) {
            best = ctas * nw;
            per_sm = ctas;
            g.nwarps = nw;
            g.smem = smem_nw;
        }
    }
    g.split = 1;
    while (g.nwarps * g.split * 2 <= kBins && ntiles * g.split < static_cast<long long>(sms) * per_sm)
        g.split *= 2;
    if (split_pref > 0 && g.nwarps * split_pref <= kBins && (split_pref & (split_pref - 1)) == 0)
        g.split = split_pref;  // autotuned (spcv_cu.cu)
    if (kn.split) {
        const int want = kn.split;
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
    if (full_rounds >= 1 && left > 0 && kn.tail != 0) {
        int ts = 1;
        if (per_sm == 1) {
            // One CTA per SM (K ~ 1024): split the partial round's tiles ts ways
            // (row slices) where that shortens it most: ceil(left * ts / sms)
            // sub-rounds of 1/ts of a tile, plus kStage of a tile per staging.
            // (measured: MBv1 pw13 242.9 -> 232.0 us at 4 slices; 8 slices lose:
            // pw13 +17 %, c5 +4 %)
            constexpr double kStage = 0.05;
            double best = 1.0 + kStage;
            for (int t = 2; t <= 4 && g.nwarps * g.split * t <= kBins; t *= 2) {
                const double rounds = static_cast<double>((left * t + resident - 1) / resident);
                const double cost = rounds * (1.0 / t + kStage);
                if (cost < best - 1e-9) best = cost, ts = t;
            }
        } else {
            // several CTAs share each SM: split while the tail stays under 3/4
            // of a round (measured best for the 2-3 CTA/SM layers)
            while (ts < 8 && g.nwarps * g.split * ts * 2 <= kBins && left * ts * 4 < resident * 3) ts *= 2;
        }
        if (tail_pref >= 0) ts = std::max(1, tail_pref);                      // autotuned (spcv_cu.cu)
        if (kn.tail > 1) ts = kn.tail;  // tuning aid
        if (ts > 1 && g.nwarps * g.split * ts <= kBins) {
            g.tail_split = ts;
            g.tail_start = ntiles - left / g.split;
        }
    }
    g.grid_x = g.tail_start + (ntiles - g.tail_start) * g.tail_split;
    return g;
}


}  // namespace spcv_detail
