// The reference's hot-path tests (/root/reference/proj/tests/test_kernels.cpp),
// re-expressed against the C++ drop-in (include/spcv_b200/spcv.hpp) — the same
// calls a reference user makes, served by the B200 kernel. Built and run by
// tests/test_cpp_dropin.py on a GPU box. Prints "ok <name>" per case and exits
// non-zero on the first failure.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "spcv_b200/spcv.hpp"

using namespace spcv;

static int g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            std::exit(1);                                                        \
        }                                                                        \
    } while (0)

template <typename E, typename F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static DenseMatrix random_matrix(int rows, int cols, std::mt19937& rng) {
    DenseMatrix m(rows, cols);
    for (float& v : m.data) v = static_cast<float>(rng() % 2000) / 999.0f - 1.0f;
    return m;
}
static Tensor random_chw(int c, int h, int w, std::mt19937& rng) {
    Tensor t(c, h, w, Layout::CHW);
    for (float& v : t.data) v = static_cast<float>(rng() % 1000) / 999.0f;
    return t;
}
static std::vector<float> random_bias(int n, std::mt19937& rng) {
    std::vector<float> b(static_cast<std::size_t>(n));
    for (float& v : b) v = static_cast<float>(rng() % 200) / 99.0f - 1.0f;
    return b;
}

// Mask without the libstdc++-specific generator: keep each entry with
// probability 1-sparsity, whole blocks (input preparation only).
static BcsrMatrix masked(DenseMatrix& w, double sparsity, int block_h, std::mt19937& rng) {
    for (int br = 0; br < w.rows / block_h; ++br)
        for (int c = 0; c < w.cols; ++c)
            if ((rng() % 1000) < sparsity * 1000)
                for (int i = 0; i < block_h; ++i) w(br * block_h + i, c) = 0.0f;
    return encode_bcsr(w, block_h);
}

// Dense oracle: bias first, ascending k, separate multiply and add
// (tensor.cpp:38-62). Built with -ffp-contract=off.
static std::vector<float> dense_ref(const DenseMatrix& w, const Tensor& a,
                                    const std::vector<float>& bias, const Activation& f) {
    const int S = a.spatial();
    std::vector<float> out(static_cast<std::size_t>(w.rows) * S);
    for (int r = 0; r < w.rows; ++r) {
        for (int s = 0; s < S; ++s) {
            float acc = bias.empty() ? 0.0f : bias[r];
            for (int k = 0; k < w.cols; ++k) {
                const float p = w(r, k) * a.data[static_cast<std::size_t>(k) * S + s];
                acc = acc + p;
            }
            out[static_cast<std::size_t>(r) * S + s] = f.apply(acc);
        }
    }
    return out;
}

int main() {
    {  // test_kernels.cpp:55-68
        DenseMatrix eye(8, 8);
        for (int i = 0; i < 8; ++i) eye(i, i) = 1.0f;
        std::mt19937 rng(3);
        const Tensor act = random_chw(8, 5, 7, rng);
        const std::vector<float> bias(8, 0.0f);
        for (int bh : {1, 2, 4}) {
            MicrokernelConfig cfg;
            cfg.n = bh;
            CHECK(spmm(encode_bcsr(eye, bh), act, bias, Activation::none(), cfg).data == act.data);
        }
        std::puts("ok identity");
    }
    {  // test_kernels.cpp:70-89
        DenseMatrix w(2, 3);
        w(0, 1) = 2.0f;
        w(1, 1) = -3.0f;
        const BcsrMatrix m = encode_bcsr(w, 2);
        CHECK(m.nnz_blocks() == 1);
        Tensor act(3, 1, 2, Layout::CHW);
        act.data = {9.0f, 9.0f, 1.0f, 4.0f, 9.0f, 9.0f};
        MicrokernelConfig cfg;
        cfg.n = 2;
        const Tensor out = spmm(m, act, std::vector<float>{1.0f, -1.0f}, Activation::relu6(), cfg);
        CHECK(out.data == (std::vector<float>{3.0f, 6.0f, 0.0f, 0.0f}));
        std::puts("ok hand_case");
    }
    {  // test_kernels.cpp:91-126: variants and remainders, exact against the dense oracle
        std::mt19937 rng(17);
        for (int mw : {4, 8, 16})
            for (int bh : {1, 2, 4}) {
                DenseMatrix w = random_matrix(64, 64, rng);
                const BcsrMatrix m = masked(w, 0.9, bh, rng);
                const Tensor act = random_chw(64, 14, 14, rng);
                const std::vector<float> bias = random_bias(64, rng);
                MicrokernelConfig cfg;
                cfg.m = mw;
                cfg.n = bh;
                CHECK(spmm(m, act, bias, Activation::relu6(), cfg).data ==
                      dense_ref(w, act, bias, Activation::relu6()));
            }
        for (int S : {1, 3, 5, 7, 13, 197}) {
            DenseMatrix w = random_matrix(16, 12, rng);
            const BcsrMatrix m = masked(w, 0.7, 2, rng);
            const Tensor act = random_chw(12, 1, S, rng);
            const std::vector<float> bias = random_bias(16, rng);
            MicrokernelConfig cfg;
            cfg.n = 2;
            CHECK(spmm(m, act, bias, Activation::none(), cfg).data ==
                  dense_ref(w, act, bias, Activation::none()));
        }
        std::puts("ok variants_and_remainders");
    }
    {  // test_kernels.cpp:151-175: prefetch + fused clamp
        std::mt19937 rng(29);
        DenseMatrix w = random_matrix(24, 32, rng);
        const BcsrMatrix m = masked(w, 0.75, 2, rng);
        const Tensor act = random_chw(32, 9, 9, rng);
        const std::vector<float> bias = random_bias(24, rng);
        MicrokernelConfig on;
        on.n = 2;
        MicrokernelConfig off = on;
        off.prefetch = false;
        CHECK(spmm(m, act, bias, Activation::none(), on).data ==
              spmm(m, act, bias, Activation::none(), off).data);
        Tensor plain = spmm(m, act, bias, Activation::none(), on);
        for (float& v : plain.data) v = Activation::relu6().apply(v);
        CHECK(spmm(m, act, bias, Activation::relu6(), on).data == plain.data);
        std::puts("ok prefetch_and_clamp");
    }
    {  // test_kernels.cpp:177-214: error classes
        std::mt19937 rng(37);
        DenseMatrix w = random_matrix(8, 8, rng);
        const BcsrMatrix m = masked(w, 0.5, 2, rng);
        const Tensor act = random_chw(8, 2, 2, rng);
        const std::vector<float> bias(8, 0.0f);
        MicrokernelConfig c4;
        c4.n = 4;
        CHECK(throws_as<FormatError>([&] { (void)spmm(m, act, bias, Activation::none(), c4); }));
        MicrokernelConfig c2;
        c2.n = 2;
        CHECK(throws_as<ShapeError>(
            [&] { (void)spmm(m, random_chw(9, 2, 2, rng), bias, Activation::none(), c2); }));
        CHECK(throws_as<LayoutError>(
            [&] { (void)spmm(m, Tensor(8, 2, 2, Layout::HWC), bias, Activation::none(), c2); }));
        MicrokernelConfig c5 = c2;
        c5.m = 5;
        CHECK(throws_as<std::invalid_argument>(
            [&] { (void)spmm(m, act, bias, Activation::none(), c5); }));
        CHECK(throws_as<ShapeError>([&] {
            (void)spmm(m, act, std::vector<float>(3, 0.0f), Activation::none(), c2);
        }));
        std::puts("ok validation");
    }
    {  // test_kernels.cpp:216-239: dense baseline (cuBLAS here: fp32 rounding, not bit-exact)
        std::mt19937 rng(43);
        const DenseMatrix w = random_matrix(16, 16, rng);
        const Tensor act = random_chw(16, 6, 6, rng);
        const std::vector<float> bias = random_bias(16, rng);
        const Tensor d = dense_gemm_baseline(w, act, bias, Activation::relu6());
        const std::vector<float> want = dense_ref(w, act, bias, Activation::relu6());
        double dev = 0.0;
        for (std::size_t i = 0; i < want.size(); ++i)
            dev = std::max(dev, static_cast<double>(std::fabs(d.data[i] - want[i])));
        CHECK(dev <= 1e-5);
        std::puts("ok dense_baseline");
    }
    {  // device-resident batch + bit-exact unpack
        std::mt19937 rng(41);
        DenseMatrix w = random_matrix(96, 64, rng);
        const BcsrMatrix m = masked(w, 0.8, 4, rng);
        const DeviceBcsr dw(m);
        const BcsrMatrix back = dw.unpack();
        CHECK(back.row_ptr == m.row_ptr && back.col_idx == m.col_idx && back.values == m.values);
        std::puts("ok device_pack_roundtrip");
    }
    {  // run_network's pointwise step (netdef.cpp:494-512): padded rows, residual after the clamp
        std::mt19937 rng(41);
        const int rows = 10, K = 24, H = 6, W = 5, B = 2, S = H * W;
        DenseMatrix w = random_matrix(rows + 2, K, rng);  // 2 padded rows (block height 4)
        for (int c = 0; c < K; ++c) w(rows, c) = w(rows + 1, c) = 0.0f;
        const BcsrMatrix m = masked(w, 0.6, 4, rng);
        DenseMatrix logical(rows, K);
        const DenseMatrix dec = decode_bcsr(m);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < K; ++c) logical(r, c) = dec(r, c);
        std::vector<float> act(static_cast<std::size_t>(B) * K * S), res(static_cast<std::size_t>(B) * rows * S);
        for (float& v : act) v = static_cast<float>(rng() % 1000) / 999.0f;
        for (float& v : res) v = static_cast<float>(rng() % 2000) / 999.0f - 1.0f;
        const std::vector<float> bias = random_bias(rows, rng);
        float *da = nullptr, *db = nullptr, *dr = nullptr, *dout = nullptr;
        cudaMalloc(&da, act.size() * 4);
        cudaMalloc(&db, bias.size() * 4);
        cudaMalloc(&dr, res.size() * 4);
        cudaMalloc(&dout, res.size() * 4);
        cudaMemcpy(da, act.data(), act.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(db, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dr, res.data(), res.size() * 4, cudaMemcpyHostToDevice);
        DeviceBcsr dw(m);
        spmm_layer(dw, da, B, H, W, db, Activation::relu6(), dr, dout, rows);
        std::vector<float> got(res.size());
        cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
        bool same = true;
        for (int b = 0; b < B; ++b) {
            Tensor img(K, H, W, Layout::CHW);
            std::copy(act.begin() + b * K * S, act.begin() + (b + 1) * K * S, img.data.begin());
            const std::vector<float> want = dense_ref(logical, img, bias, Activation::relu6());
            for (int i = 0; i < rows * S; ++i) {
                const float v = want[i] + res[static_cast<std::size_t>(b) * rows * S + i];
                same = same && got[static_cast<std::size_t>(b) * rows * S + i] == v;
            }
        }
        CHECK(same);
        cudaFree(da);
        cudaFree(db);
        cudaFree(dr);
        cudaFree(dout);
        std::puts("ok spmm_layer_padded_residual");
    }
    std::printf("all %d checks passed\n", g_checks);
    return 0;
}
