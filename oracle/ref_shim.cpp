// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference library.
//
// TEST/BASELINE INFRASTRUCTURE ONLY. oracle/Makefile compiles this file together
// with /root/reference/proj/src/{tensor,sparse,kernels}.cpp (read in place,
// never copied) into oracle/_ref/libspcv_ref.so. Tests use it to pin the
// oracle restatement; bench.py uses it as the CPU baseline ("kind":
// "reference") and as the `--impl reference` arm.
//
// Error mapping (same codes as include/spcv_cu.h):
//   LayoutError -> 1, ShapeError -> 2, FormatError -> 3,
//   other std::invalid_argument -> 4, anything else -> 5.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "spcv/kernels.hpp"
#include "spcv/model_io.hpp"
#include "spcv/netdef.hpp"
#include "spcv/sparse.hpp"
#include "spcv/tensor.hpp"

namespace {

int code_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const spcv::BadMagicError&) {
        return 8;
    } catch (const spcv::UnsupportedVersionError&) {
        return 9;
    } catch (const spcv::TruncatedError&) {
        return 10;
    } catch (const spcv::ChecksumError&) {
        return 11;
    } catch (const spcv::ModelFormatError&) {
        return 12;
    } catch (const spcv::ModelIoError&) {
        return 7;
    } catch (const spcv::LayoutError&) {
        return 1;
    } catch (const spcv::ShapeError&) {
        return 2;
    } catch (const spcv::FormatError&) {
        return 3;
    } catch (const std::invalid_argument&) {
        return 4;
    } catch (...) {
        return 5;
    }
}

spcv::BcsrMatrix make_bcsr(int rows, int cols, int block_h, const std::uint32_t* row_ptr,
                           std::size_t nrp, const std::uint32_t* col_idx, std::size_t nblk,
                           const float* values, std::size_t nval) {
    spcv::BcsrMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.block_h = block_h;
    m.row_ptr.assign(row_ptr, row_ptr + nrp);
    m.col_idx.assign(col_idx, col_idx + nblk);
    m.values.assign(values, values + nval);
    return m;
}

spcv::Activation make_act(int kind, float lo, float hi) {
    return kind == 0 ? spcv::Activation::none() : spcv::Activation::clamp(lo, hi);
}

spcv::Tier tier_of(int t) {
    return t == 0 ? spcv::Tier::Scalar : (t == 1 ? spcv::Tier::Vector : spcv::Tier::Auto);
}

}  // namespace

extern "C" {

// spcv::spmm_into over `images` independent CHW images (act [images][cols][H*W],
// out [images][rows][H*W]). act_layout 1 = HWC (to exercise LayoutError).
int ref_spmm(int rows, int cols, int block_h, const std::uint32_t* row_ptr, std::size_t nrp,
             const std::uint32_t* col_idx, std::size_t nblk, const float* values,
             std::size_t nval, int images, int act_channels, int H, int W, int act_layout,
             const float* act, const float* bias, std::size_t bias_len, int act_kind, float lo,
             float hi, int out_channels, float* out, int cfg_m, int cfg_n, int prefetch,
             int tier) {
    try {
        const spcv::BcsrMatrix m =
            make_bcsr(rows, cols, block_h, row_ptr, nrp, col_idx, nblk, values, nval);
        const spcv::Activation fn = make_act(act_kind, lo, hi);
        spcv::MicrokernelConfig cfg;
        cfg.m = cfg_m;
        cfg.n = cfg_n;
        cfg.prefetch = prefetch != 0;
        cfg.tier = tier_of(tier);
        const std::size_t in_sz = static_cast<std::size_t>(act_channels) * H * W;
        const std::size_t out_sz = static_cast<std::size_t>(out_channels) * H * W;
        std::span<const float> b(bias, bias ? bias_len : 0);
        for (int i = 0; i < images; ++i) {
            spcv::Tensor a(act_channels, H, W,
                           act_layout == 1 ? spcv::Layout::HWC : spcv::Layout::CHW);
            std::memcpy(a.data.data(), act + i * in_sz, in_sz * sizeof(float));
            spcv::Tensor o(out_channels, H, W, spcv::Layout::CHW);
            spcv::spmm_into(m, a, b, fn, o, cfg);
            std::memcpy(out + i * out_sz, o.data.data(), out_sz * sizeof(float));
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_matmul_reference(int rows, int cols, int H, int W, const float* w, const float* act,
                         const float* bias, int act_kind, float lo, float hi, float* out) {
    try {
        spcv::DenseMatrix dm(rows, cols);
        std::memcpy(dm.data.data(), w, sizeof(float) * dm.data.size());
        spcv::Tensor a(cols, H, W, spcv::Layout::CHW);
        std::memcpy(a.data.data(), act, sizeof(float) * a.data.size());
        std::span<const float> b(bias, bias ? static_cast<std::size_t>(rows) : 0);
        const spcv::Tensor o = spcv::matmul_reference(dm, a, b, make_act(act_kind, lo, hi));
        std::memcpy(out, o.data.data(), sizeof(float) * o.data.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// spcv::depthwise_conv_chw (kernels.cpp:385-422) per image: in [images][C][H][W],
// w [C][3][3], bias [C] or null -> out [images][C][OH][OW].
int ref_depthwise(int images, int C, int H, int W, int stride, const float* w, const float* bias,
                  int act_kind, float lo, float hi, const float* in, float* out, int* OH, int* OW) {
    try {
        spcv::DepthwiseWeights dw(C);
        std::memcpy(dw.data.data(), w, sizeof(float) * dw.data.size());
        std::span<const float> b(bias, bias ? static_cast<std::size_t>(C) : 0);
        const std::size_t in_sz = static_cast<std::size_t>(C) * H * W;
        std::size_t out_sz = 0;
        for (int i = 0; i < images; ++i) {
            spcv::Tensor a(C, H, W, spcv::Layout::CHW);
            std::memcpy(a.data.data(), in + i * in_sz, in_sz * sizeof(float));
            const spcv::Tensor o = spcv::depthwise_conv_chw(a, dw, stride, b, make_act(act_kind, lo, hi));
            out_sz = o.data.size();
            *OH = o.height;
            *OW = o.width;
            if (out) std::memcpy(out + i * out_sz, o.data.data(), out_sz * sizeof(float));
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// spcv::entry_conv_hwc_to_chw (kernels.cpp:424-474) per image: in [images][H][W][C]
// (HWC), w [CO][C][3][3], bias [CO] or null -> out [images][CO][OH][OW].
int ref_entry_conv(int images, int C, int H, int W, int CO, int stride, const float* w, const float* bias,
                   int act_kind, float lo, float hi, const float* in, float* out, int* OH, int* OW) {
    try {
        spcv::ConvWeights cw(CO, C, 3, 3);
        std::memcpy(cw.data.data(), w, sizeof(float) * cw.data.size());
        std::span<const float> b(bias, bias ? static_cast<std::size_t>(CO) : 0);
        const std::size_t in_sz = static_cast<std::size_t>(C) * H * W;
        for (int i = 0; i < images; ++i) {
            spcv::Tensor a(C, H, W, spcv::Layout::HWC);
            std::memcpy(a.data.data(), in + i * in_sz, in_sz * sizeof(float));
            const spcv::Tensor o = spcv::entry_conv_hwc_to_chw(a, cw, stride, b, make_act(act_kind, lo, hi));
            *OH = o.height;
            *OW = o.width;
            if (out) std::memcpy(out + i * o.data.size(), o.data.data(), o.data.size() * sizeof(float));
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_encode_bcsr(int rows, int cols, int block_h, const float* w, std::uint32_t* row_ptr,
                    std::uint32_t* col_idx, float* values, std::size_t* nblocks) {
    try {
        spcv::DenseMatrix dm(rows, cols);
        std::memcpy(dm.data.data(), w, sizeof(float) * dm.data.size());
        const spcv::BcsrMatrix m = spcv::encode_bcsr(dm, block_h);
        std::copy(m.row_ptr.begin(), m.row_ptr.end(), row_ptr);
        std::copy(m.col_idx.begin(), m.col_idx.end(), col_idx);
        std::copy(m.values.begin(), m.values.end(), values);
        *nblocks = m.col_idx.size();
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_validate_bcsr(int rows, int cols, int block_h, const std::uint32_t* row_ptr,
                      std::size_t nrp, const std::uint32_t* col_idx, std::size_t nblk,
                      const float* values, std::size_t nval) {
    try {
        make_bcsr(rows, cols, block_h, row_ptr, nrp, col_idx, nblk, values, nval).validate();
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

int ref_generate_mask(int rows, int cols, double sparsity, int out_block, int in_block,
                      std::uint32_t seed, std::uint8_t* keep) {
    try {
        const spcv::SparsityMask mk =
            spcv::generate_mask(rows, cols, sparsity, spcv::BlockConfig(out_block, in_block), seed);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c)
                keep[static_cast<std::size_t>(r) * cols + c] = mk.get(r, c) ? 1 : 0;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// Timed CPU baseline: spmm_into over `images` images split contiguously over
// `nthreads` std::threads (reentrant per /root/reference/SPEC.md:290), default
// MicrokernelConfig with n = block_h (Auto tier -> vector, 16xN strips).
// Tensors are built once outside the timed region. Runs `warmups` untimed
// passes then `reps` timed passes; writes the per-pass seconds to secs[reps].
int ref_bench_spmm(int rows, int cols, int block_h, const std::uint32_t* row_ptr,
                   std::size_t nrp, const std::uint32_t* col_idx, std::size_t nblk,
                   const float* values, std::size_t nval, int images, int H, int W,
                   const float* act, const float* bias, int act_kind, float lo, float hi,
                   float* out, int nthreads, int warmups, int reps, double* secs) {
    try {
        const spcv::BcsrMatrix m =
            make_bcsr(rows, cols, block_h, row_ptr, nrp, col_idx, nblk, values, nval);
        const spcv::Activation fn = make_act(act_kind, lo, hi);
        spcv::MicrokernelConfig cfg;
        cfg.n = block_h;
        const std::size_t in_sz = static_cast<std::size_t>(cols) * H * W;
        const std::size_t out_sz = static_cast<std::size_t>(rows) * H * W;
        std::vector<spcv::Tensor> ins, outs;
        ins.reserve(images);
        outs.reserve(images);
        for (int i = 0; i < images; ++i) {
            ins.emplace_back(cols, H, W, spcv::Layout::CHW);
            std::memcpy(ins.back().data.data(), act + i * in_sz, in_sz * sizeof(float));
            outs.emplace_back(rows, H, W, spcv::Layout::CHW);
        }
        std::span<const float> b(bias, bias ? static_cast<std::size_t>(rows) : 0);
        if (nthreads < 1) nthreads = 1;
        nthreads = std::min(nthreads, std::max(images, 1));
        auto pass = [&] {
            std::vector<std::thread> th;
            th.reserve(nthreads);
            for (int t = 0; t < nthreads; ++t) {
                const int i0 = static_cast<int>(static_cast<long>(images) * t / nthreads);
                const int i1 = static_cast<int>(static_cast<long>(images) * (t + 1) / nthreads);
                th.emplace_back([&, i0, i1] {
                    for (int i = i0; i < i1; ++i) spcv::spmm_into(m, ins[i], b, fn, outs[i], cfg);
                });
            }
            for (auto& t : th) t.join();
        };
        for (int i = 0; i < warmups; ++i) pass();
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            pass();
            const auto t1 = std::chrono::steady_clock::now();
            secs[r] = std::chrono::duration<double>(t1 - t0).count();
        }
        if (out)
            for (int i = 0; i < images; ++i)
                std::memcpy(out + i * out_sz, outs[i].data.data(), out_sz * sizeof(float));
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// One layer of a multi-layer CPU benchmark (plain data, filled from Python).
struct RefLayer {
    int rows, cols, block_h;
    const std::uint32_t* row_ptr;
    std::size_t nrp;
    const std::uint32_t* col_idx;
    std::size_t nblk;
    const float* values;
    std::size_t nval;
    int images, H, W;
    const float* act;   // [images][cols][H*W]
    const float* bias;  // [rows] or null
    int act_kind;
    float lo, hi;
};

// Timed CPU workload: every (layer, image) pair is one spmm_into call (default
// MicrokernelConfig, n = block_h); `nthreads` std::threads pull units, longest
// first, from a shared counter. Objects are built once, outside the timing.
int ref_bench_layers(const RefLayer* L, int nlayers, int nthreads, int warmups, int reps,
                     double* secs) {
    try {
        struct Unit {
            int layer, image;
            double cost;
        };
        std::vector<spcv::BcsrMatrix> mats;
        std::vector<spcv::Activation> fns;
        std::vector<std::vector<spcv::Tensor>> ins(nlayers), outs(nlayers);
        std::vector<Unit> units;
        for (int l = 0; l < nlayers; ++l) {
            const RefLayer& x = L[l];
            mats.push_back(make_bcsr(x.rows, x.cols, x.block_h, x.row_ptr, x.nrp, x.col_idx, x.nblk,
                                     x.values, x.nval));
            fns.push_back(make_act(x.act_kind, x.lo, x.hi));
            const std::size_t in_sz = static_cast<std::size_t>(x.cols) * x.H * x.W;
            for (int i = 0; i < x.images; ++i) {
                ins[l].emplace_back(x.cols, x.H, x.W, spcv::Layout::CHW);
                std::memcpy(ins[l].back().data.data(), x.act + i * in_sz, in_sz * sizeof(float));
                outs[l].emplace_back(x.rows, x.H, x.W, spcv::Layout::CHW);
                units.push_back({l, i, static_cast<double>(x.nval) * x.H * x.W});
            }
        }
        std::stable_sort(units.begin(), units.end(),
                         [](const Unit& a, const Unit& b) { return a.cost > b.cost; });
        if (nthreads < 1) nthreads = 1;
        auto pass = [&] {
            std::atomic<std::size_t> next{0};
            std::vector<std::thread> th;
            for (int t = 0; t < nthreads; ++t)
                th.emplace_back([&] {
                    for (std::size_t u; (u = next.fetch_add(1)) < units.size();) {
                        const Unit& x = units[u];
                        const RefLayer& ly = L[x.layer];
                        spcv::MicrokernelConfig cfg;
                        cfg.n = ly.block_h;
                        std::span<const float> b(ly.bias, ly.bias ? static_cast<std::size_t>(ly.rows) : 0);
                        spcv::spmm_into(mats[x.layer], ins[x.layer][x.image], b, fns[x.layer],
                                        outs[x.layer][x.image], cfg);
                    }
                });
            for (auto& t : th) t.join();
        };
        for (int i = 0; i < warmups; ++i) pass();
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            pass();
            secs[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// ---------------------------------------------------------------- model files
// serialize_model(build_network(arch, width, default_plan(arch, sparsity)),
// instantiate_weights(seed)) (model_io.cpp:146-227, netdef.cpp:234-404).
// Two-call: with buf == null (or too small) only *n is written.
int ref_model_bytes(const char* arch, double width, double sparsity, std::uint32_t seed,
                    std::uint8_t* buf, std::size_t cap, std::size_t* n) {
    try {
        const spcv::NetworkSpec net =
            spcv::build_network(arch, width, spcv::default_plan(arch, sparsity));
        const spcv::WeightSet ws = spcv::instantiate_weights(net, seed);
        const std::vector<std::uint8_t> bytes = spcv::serialize_model(net, ws);
        *n = bytes.size();
        if (buf && cap >= bytes.size()) std::memcpy(buf, bytes.data(), bytes.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// parse_model (model_io.cpp:238-381): 0 or the typed-error code.
int ref_model_parse(const std::uint8_t* data, std::size_t size, int* layers) {
    try {
        const auto parsed = spcv::parse_model(data, size);
        if (layers) *layers = static_cast<int>(parsed.first.layers.size());
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// Layer i of a parsed model: kind, cout, storage and (two-call) the BCSR
// arrays of a sparse layer. meta = {kind, cin, cout, is_sparse, rows, cols,
// block_h, nrp, nblk, nval, nbias, residual_src}.
int ref_model_layer(const std::uint8_t* data, std::size_t size, int i, int* meta,
                    std::uint32_t* row_ptr, std::uint32_t* col_idx, float* values, float* bias) {
    try {
        const auto parsed = spcv::parse_model(data, size);
        const spcv::LayerSpec& L = parsed.first.layers.at(static_cast<std::size_t>(i));
        const spcv::LayerWeights& w = parsed.second.layers.at(static_cast<std::size_t>(i));
        const int m[12] = {static_cast<int>(L.kind), L.cin, L.cout, w.is_sparse ? 1 : 0,
                           w.sparse.rows, w.sparse.cols, w.sparse.block_h,
                           static_cast<int>(w.sparse.row_ptr.size()),
                           static_cast<int>(w.sparse.col_idx.size()),
                           static_cast<int>(w.sparse.values.size()),
                           static_cast<int>(w.bias.size()), L.residual_src};
        std::copy(m, m + 12, meta);
        if (row_ptr) std::copy(w.sparse.row_ptr.begin(), w.sparse.row_ptr.end(), row_ptr);
        if (col_idx) std::copy(w.sparse.col_idx.begin(), w.sparse.col_idx.end(), col_idx);
        if (values) std::copy(w.sparse.values.begin(), w.sparse.values.end(), values);
        if (bias) std::copy(w.bias.begin(), w.bias.end(), bias);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// run_network (netdef.cpp:456-524; which == 0, default ExecOptions) or
// run_network_reference (netdef.cpp:526-; which == 1) over `images` HWC images
// [images][H][W][C] of a model file; logits [images][num_classes]. Two-call
// on *classes (logits may be null).
int ref_run_model(const std::uint8_t* data, std::size_t size, const float* input, int images,
                  int which, float* logits, int* classes) {
    try {
        const auto parsed = spcv::parse_model(data, size);
        const spcv::NetworkSpec& net = parsed.first;
        if (classes) *classes = net.num_classes;
        if (!logits) return 0;
        const std::size_t per = static_cast<std::size_t>(net.input_h) * net.input_w * net.input_c;
        for (int i = 0; i < images; ++i) {
            spcv::Tensor t(net.input_c, net.input_h, net.input_w, spcv::Layout::HWC);
            std::copy(input + i * per, input + (i + 1) * per, t.data.begin());
            const std::vector<float> out = which == 0
                                               ? spcv::run_network(net, parsed.second, t, spcv::ExecOptions{})
                                               : spcv::run_network_reference(net, parsed.second, t);
            std::copy(out.begin(), out.end(), logits + static_cast<std::size_t>(i) * out.size());
        }
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

}  // extern "C"
