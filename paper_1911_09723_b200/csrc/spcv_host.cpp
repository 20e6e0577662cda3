// spcv_host.cpp — the C++ mirror of the reference SpMM surface over the C-ABI.
//
// Reference behaviour mirrored (file:line in /root/reference/proj):
//   Tensor ctor dims check            include/spcv/tensor.hpp:37-42
//   Activation::clamp lo<hi            include/spcv/tensor.hpp:79-87
//   BcsrMatrix::validate               src/sparse.cpp:16-51
//   encode_bcsr / decode_bcsr          src/sparse.cpp:108-148
//   tier plumbing + variant names      src/kernels.cpp:240-300
//   spmm_into validation order         src/kernels.cpp:306-322
//   spmm allocating wrapper            src/kernels.cpp:336-341
#include "spcv_b200/spcv.hpp"

#include <cuda_runtime.h>

#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <random>
#include <string_view>

namespace spcv {

void throw_status(int status, const char* message) {
    const std::string msg = message ? message : "";
    switch (status) {
        case SPCV_OK: return;
        case SPCV_ERR_LAYOUT: throw LayoutError(msg);
        case SPCV_ERR_SHAPE: throw ShapeError(msg);
        case SPCV_ERR_FORMAT: throw FormatError(msg);
        case SPCV_ERR_INVALID: throw std::invalid_argument(msg);
        case SPCV_ERR_MODEL_IO: throw ModelIoError(msg);
        case SPCV_ERR_BAD_MAGIC: throw BadMagicError(msg);
        case SPCV_ERR_VERSION: throw UnsupportedVersionError(msg);
        case SPCV_ERR_TRUNCATED: throw TruncatedError(msg);
        case SPCV_ERR_CHECKSUM: throw ChecksumError(msg);
        case SPCV_ERR_MODEL_FORMAT: throw ModelFormatError(msg);
        default: throw DeviceError(msg.empty() ? "spcv_cu: device failure" : msg);
    }
}

static void check(int status) {
    if (status != SPCV_OK) throw_status(status, spcv_cu_last_error());
}

// ---------------------------------------------------------------- tensors

Tensor::Tensor(int c, int h, int w, Layout l) : channels(c), height(h), width(w), layout(l) {
    if (c < 1 || h < 1 || w < 1) throw ShapeError("tensor dims must be >= 1");
    data.assign(static_cast<std::size_t>(c) * h * w, 0.0f);
}

std::size_t Tensor::index(int c, int h, int w) const {
    const std::size_t hw = static_cast<std::size_t>(h) * width + w;
    return layout == Layout::CHW ? static_cast<std::size_t>(c) * height * width + hw
                                 : hw * channels + c;
}

DenseMatrix::DenseMatrix(int r, int c) : rows(r), cols(c) {
    if (r < 0 || c < 0) throw ShapeError("matrix dims must be >= 0");
    data.assign(static_cast<std::size_t>(r) * c, 0.0f);
}

Activation Activation::clamp(float lo, float hi) {
    if (!(lo < hi)) throw std::invalid_argument("clamp requires lo < hi");
    Activation a;
    a.kind = Kind::Clamp;
    a.lo = lo;
    a.hi = hi;
    return a;
}

// ------------------------------------------------------------------- BCSR

void BcsrMatrix::validate() const {
    if (rows < 1 || cols < 1) throw FormatError("bcsr: dims must be >= 1");
    if (block_h != 1 && block_h != 2 && block_h != 4)
        throw FormatError("bcsr: block height must be 1, 2 or 4");
    if (rows % block_h != 0) throw FormatError("bcsr: rows not divisible by block height");
    const std::size_t nbr = static_cast<std::size_t>(rows / block_h);
    if (row_ptr.size() != nbr + 1) throw FormatError("bcsr: row_ptr length != block rows + 1");
    if (row_ptr.front() != 0) throw FormatError("bcsr: row_ptr[0] != 0");
    for (std::size_t r = 0; r < nbr; ++r)
        if (row_ptr[r + 1] < row_ptr[r]) throw FormatError("bcsr: row_ptr not non-decreasing");
    if (row_ptr.back() != col_idx.size()) throw FormatError("bcsr: row_ptr[-1] != block count");
    if (values.size() != col_idx.size() * static_cast<std::size_t>(block_h))
        throw FormatError("bcsr: values length != block count * block height");
    for (std::size_t r = 0; r < nbr; ++r)
        for (std::uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
            if (col_idx[b] >= static_cast<std::uint32_t>(cols))
                throw FormatError("bcsr: column index out of range");
            if (b > row_ptr[r] && col_idx[b] <= col_idx[b - 1])
                throw FormatError("bcsr: column indices not strictly increasing");
        }
}

BcsrMatrix encode_bcsr(const DenseMatrix& w, int block_h) {
    if (block_h != 1 && block_h != 2 && block_h != 4)
        throw FormatError("encode_bcsr: block height must be 1, 2 or 4");
    if (w.rows % block_h != 0) throw ShapeError("encode_bcsr: rows not divisible by block height");
    BcsrMatrix m;
    m.rows = w.rows;
    m.cols = w.cols;
    m.block_h = block_h;
    m.row_ptr.assign(1, 0u);
    for (int br = 0; br < w.rows / block_h; ++br) {
        for (int c = 0; c < w.cols; ++c) {
            bool any = false;
            for (int i = 0; i < block_h; ++i) any = any || w(br * block_h + i, c) != 0.0f;
            if (!any) continue;
            m.col_idx.push_back(static_cast<std::uint32_t>(c));
            for (int i = 0; i < block_h; ++i) m.values.push_back(w(br * block_h + i, c));
        }
        m.row_ptr.push_back(static_cast<std::uint32_t>(m.col_idx.size()));
    }
    return m;
}

DenseMatrix decode_bcsr(const BcsrMatrix& m) {
    m.validate();
    DenseMatrix w(m.rows, m.cols);
    for (int br = 0; br < m.block_rows(); ++br)
        for (std::uint32_t b = m.row_ptr[br]; b < m.row_ptr[br + 1]; ++b)
            for (int i = 0; i < m.block_h; ++i)
                w(br * m.block_h + i, static_cast<int>(m.col_idx[b])) =
                    m.values[static_cast<std::size_t>(b) * m.block_h + i];
    return w;
}

// ---------------------------------------------------------- tier plumbing
// One CUDA path: "vector" always exists. Kept so callers of the reference
// plumbing (kernels.cpp:240-300) compile and behave the same.

bool vector_tier_available() { return true; }

Tier resolve_tier(Tier requested) {
    const char* env = std::getenv("SPCV_FORCE_SCALAR");
    if (env && *env && std::string_view(env) != "0") return Tier::Scalar;
    return requested == Tier::Auto ? Tier::Vector : requested;
}

const char* tier_name(Tier t) {
    return t == Tier::Scalar ? "scalar" : (t == Tier::Vector ? "vector" : "auto");
}

Tier parse_tier(const std::string& s) {
    if (s == "scalar") return Tier::Scalar;
    if (s == "vector") return Tier::Vector;
    if (s == "auto") return Tier::Auto;
    throw std::invalid_argument("unknown tier '" + s + "' (expected scalar|vector|auto)");
}

int default_strip_width(Tier t) { return resolve_tier(t) == Tier::Vector ? 16 : 8; }

std::string variant_name(int m, int n) { return std::to_string(m) + "x" + std::to_string(n); }

std::pair<int, int> parse_variant(const std::string& s) {
    const auto bad = [&] {
        return std::invalid_argument("bad variant '" + s + "' (expected MxN, e.g. 16x2)");
    };
    const std::size_t x = s.find('x');
    if (x == std::string::npos || x == 0 || x + 1 >= s.size()) throw bad();
    auto digits = [](std::string_view v) {
        if (v.empty() || v.size() > 6) return -1;
        int out = 0;
        for (char ch : v) {
            if (ch < '0' || ch > '9') return -1;
            out = out * 10 + (ch - '0');
        }
        return out;
    };
    const int m = digits(std::string_view(s).substr(0, x));
    const int n = digits(std::string_view(s).substr(x + 1));
    if (m < 0 || n < 0) throw bad();
    if (m != 4 && m != 8 && m != 16)
        throw std::invalid_argument("variant strip width must be 4, 8 or 16 (got " + s + ")");
    if (n != 1 && n != 2 && n != 4)
        throw std::invalid_argument("variant out_block must be 1, 2 or 4 (got " + s + ")");
    return {m, n};
}

// ------------------------------------------------------------ device weights

DeviceBcsr::DeviceBcsr(const BcsrMatrix& m) {
    check(spcv_cu_pack(m.rows, m.cols, m.block_h, m.row_ptr.data(), m.row_ptr.size(),
                       m.col_idx.data(), m.col_idx.size(), m.values.data(), m.values.size(), &h_));
}

DeviceBcsr& DeviceBcsr::operator=(DeviceBcsr&& o) noexcept {
    if (this != &o) {
        spcv_cu_free(h_);
        h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
}

DeviceBcsr::~DeviceBcsr() { spcv_cu_free(h_); }

int DeviceBcsr::rows() const {
    int r = 0;
    check(spcv_cu_weights_info(h_, &r, nullptr, nullptr, nullptr, nullptr, nullptr));
    return r;
}
int DeviceBcsr::cols() const {
    int c = 0;
    check(spcv_cu_weights_info(h_, nullptr, &c, nullptr, nullptr, nullptr, nullptr));
    return c;
}
int DeviceBcsr::block_h() const {
    int b = 0;
    check(spcv_cu_weights_info(h_, nullptr, nullptr, &b, nullptr, nullptr, nullptr));
    return b;
}

BcsrMatrix DeviceBcsr::unpack() const {
    BcsrMatrix m;
    std::size_t nb = 0;
    check(spcv_cu_weights_info(h_, &m.rows, &m.cols, &m.block_h, &nb, nullptr, nullptr));
    m.row_ptr.resize(static_cast<std::size_t>(m.rows / m.block_h) + 1);
    m.col_idx.resize(nb);
    m.values.resize(nb * static_cast<std::size_t>(m.block_h));
    check(spcv_cu_unpack(h_, m.row_ptr.data(), m.col_idx.data(), m.values.data()));
    return m;
}

// ----------------------------------------------------------------- spmm

static int act_kind(const Activation& a) {
    return a.kind == Activation::Kind::Clamp ? SPCV_ACT_CLAMP : SPCV_ACT_NONE;
}
static int layout_code(Layout l) { return l == Layout::CHW ? SPCV_LAYOUT_CHW : SPCV_LAYOUT_HWC; }

void spmm_into(const BcsrMatrix& w, const Tensor& act, std::span<const float> bias,
               const Activation& fused, Tensor& out, const MicrokernelConfig& cfg) {
    // The reference validates act/bias/out before touching the matrix
    // (kernels.cpp:306-322) and never validates the matrix itself; the
    // device packer does (FormatError on a malformed matrix). Run the
    // reference's argument checks first so error precedence is identical.
    if (act.layout != Layout::CHW) throw LayoutError("spmm: activation must be CHW");
    if (w.cols != act.channels) throw ShapeError("spmm: weight cols != activation channels");
    if (cfg.n != w.block_h) throw FormatError("spmm: cfg out_block != matrix block height");
    if (!bias.empty() && static_cast<int>(bias.size()) != w.rows)
        throw ShapeError("spmm: bias length != rows");
    if (out.layout != Layout::CHW || out.channels != w.rows || out.height != act.height ||
        out.width != act.width)
        throw ShapeError("spmm: output tensor shape/layout mismatch");
    const int m = cfg.m != 0 ? cfg.m : default_strip_width(cfg.tier);
    if (m != 4 && m != 8 && m != 16) throw std::invalid_argument("spmm: strip width must be 4, 8 or 16");

    // packed once per distinct matrix content (the C-ABI's weight cache): a
    // caller looping spmm_into over layers and images never repacks
    check(spcv_cu_spmm_bcsr_into_host(w.rows, w.cols, w.block_h, w.row_ptr.data(), w.row_ptr.size(),
                                      w.col_idx.data(), w.col_idx.size(), w.values.data(), w.values.size(),
                                      act.data.data(), layout_code(act.layout), 1, act.channels,
                                      act.height, act.width, bias.empty() ? nullptr : bias.data(),
                                      bias.size(), act_kind(fused), fused.lo, fused.hi, out.data.data(),
                                      layout_code(out.layout), out.channels, out.height, out.width,
                                      cfg.m, cfg.n, cfg.strict ? SPCV_MODE_STRICT : SPCV_MODE_FAST));
}

Tensor spmm(const BcsrMatrix& w, const Tensor& act, std::span<const float> bias,
            const Activation& fused, const MicrokernelConfig& cfg) {
    Tensor out(w.rows, act.height, act.width, Layout::CHW);
    spmm_into(w, act, bias, fused, out, cfg);
    return out;
}

void dense_gemm_into(const DenseMatrix& w, const Tensor& act, std::span<const float> bias,
                     const Activation& fused, Tensor& out, const MicrokernelConfig& cfg) {
    // kernels.cpp:347-360 order, checked here so errors precede any device work
    if (act.layout != Layout::CHW) throw LayoutError("dense_gemm: activation must be CHW");
    if (w.cols != act.channels) throw ShapeError("dense_gemm: weight cols != activation channels");
    if (!bias.empty() && static_cast<int>(bias.size()) != w.rows)
        throw ShapeError("dense_gemm: bias length != rows");
    if (out.layout != Layout::CHW || out.channels != w.rows || out.height != act.height ||
        out.width != act.width)
        throw ShapeError("dense_gemm: output tensor shape/layout mismatch");
    const int m = cfg.m != 0 ? cfg.m : default_strip_width(cfg.tier);
    if (m != 4 && m != 8 && m != 16)
        throw std::invalid_argument("dense_gemm: strip width must be 4, 8 or 16");
    float *dw = nullptr, *da = nullptr, *db = nullptr, *dout = nullptr;
    auto cleanup = [&] {
        cudaFree(dw);
        cudaFree(da);
        cudaFree(db);
        cudaFree(dout);
    };
    auto ck = [&](cudaError_t e) {
        if (e != cudaSuccess) {
            cleanup();
            throw DeviceError(std::string("dense_gemm: ") + cudaGetErrorString(e));
        }
    };
    ck(cudaMalloc(&dw, std::max<size_t>(w.data.size(), 1) * 4));
    ck(cudaMalloc(&da, act.data.size() * 4));
    ck(cudaMalloc(&dout, out.data.size() * 4));
    if (!bias.empty()) ck(cudaMalloc(&db, bias.size() * 4));
    ck(cudaMemcpy(dw, w.data.data(), w.data.size() * 4, cudaMemcpyHostToDevice));
    ck(cudaMemcpy(da, act.data.data(), act.data.size() * 4, cudaMemcpyHostToDevice));
    if (!bias.empty()) ck(cudaMemcpy(db, bias.data(), bias.size() * 4, cudaMemcpyHostToDevice));
    const int rc = spcv_cu_dense_gemm_into(
        dw, w.rows, w.cols, da, SPCV_LAYOUT_CHW, 1, act.channels, act.height, act.width, db,
        bias.size(), act_kind(fused), fused.lo, fused.hi, dout, SPCV_LAYOUT_CHW, out.channels,
        out.height, out.width, cfg.m, nullptr);
    if (rc != SPCV_OK) {
        const std::string msg = spcv_cu_last_error();
        cleanup();
        throw_status(rc, msg.c_str());
    }
    ck(cudaMemcpy(out.data.data(), dout, out.data.size() * 4, cudaMemcpyDeviceToHost));
    cleanup();
}

Tensor dense_gemm_baseline(const DenseMatrix& w, const Tensor& act, std::span<const float> bias,
                           const Activation& fused, const MicrokernelConfig& cfg) {
    Tensor out(w.rows, act.height, act.width, Layout::CHW);
    dense_gemm_into(w, act, bias, fused, out, cfg);
    return out;
}

void spmm_batched_into(const DeviceBcsr& w, const float* d_act, int images, int height, int width,
                       const float* d_bias, const Activation& fused, float* d_out,
                       const MicrokernelConfig& cfg, void* stream) {
    int rows = 0, cols = 0;
    check(spcv_cu_weights_info(w.handle(), &rows, &cols, nullptr, nullptr, nullptr, nullptr));
    check(spcv_cu_spmm_into(w.handle(), d_act, SPCV_LAYOUT_CHW, images, cols, height, width,
                            d_bias, d_bias ? static_cast<std::size_t>(rows) : 0, act_kind(fused),
                            fused.lo, fused.hi, d_out, SPCV_LAYOUT_CHW, rows, height, width, cfg.m,
                            cfg.n, cfg.strict ? SPCV_MODE_STRICT : SPCV_MODE_FAST, stream));
}

}  // namespace spcv

namespace spcv {

void spmm_layer(const DeviceBcsr& w, const float* d_act, int images, int height, int width,
                const float* d_bias, const Activation& fused, const float* d_residual, float* d_out,
                int out_channels, bool strict, void* stream) {
    check(spcv_cu_spmm_layer(w.handle(), d_act, images, w.cols(), height, width, d_bias,
                             d_bias ? static_cast<size_t>(out_channels) : 0,
                             fused.kind == Activation::Kind::Clamp ? SPCV_ACT_CLAMP : SPCV_ACT_NONE,
                             fused.lo, fused.hi, d_residual, d_out, out_channels,
                             strict ? SPCV_MODE_STRICT : SPCV_MODE_FAST, stream));
}

// ------------------------------------------------------------ model files

DeviceModel::DeviceModel(std::span<const std::uint8_t> bytes) {
    check(spcv_cu_model_load(bytes.data(), bytes.size(), &h_));
    int n = 0;
    check(spcv_cu_model_parse(bytes.data(), bytes.size(), &n));
    int first[12], last[12];
    check(spcv_cu_model_layer(h_, 0, first));
    check(spcv_cu_model_layer(h_, n - 1, last));
    // info = {kind, cin, cout, in_h, in_w, out_h, out_w, sparse, block_h, act, residual, stride}
    meta_[0] = n;
    meta_[1] = first[3];
    meta_[2] = first[4];
    meta_[3] = first[1];
    meta_[4] = last[2];
}

DeviceModel DeviceModel::load(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw ModelIoError("cannot open model file '" + path + "'");
    std::vector<std::uint8_t> bytes;
    std::uint8_t buf[1 << 16];
    std::size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) bytes.insert(bytes.end(), buf, buf + n);
    const bool err = std::ferror(f) != 0;
    std::fclose(f);
    if (err) throw ModelIoError("error reading model file '" + path + "'");
    return DeviceModel(std::span<const std::uint8_t>(bytes));
}

DeviceModel::~DeviceModel() { spcv_cu_model_free(h_); }

void DeviceModel::forward(const float* d_input, int images, float* d_logits, bool strict,
                          void* stream) const {
    check(spcv_cu_model_forward(h_, d_input, images, input_h(), input_w(), input_c(), d_logits,
                                strict ? SPCV_MODE_STRICT : SPCV_MODE_FAST, stream));
}

std::vector<float> run_network(const DeviceModel& model, const Tensor& input, bool strict) {
    if (input.layout != Layout::HWC || input.channels != model.input_c() ||
        input.height != model.input_h() || input.width != model.input_w())
        throw ShapeError("run: input must be HWC " + std::to_string(model.input_h()) + "x" +
                         std::to_string(model.input_w()) + "x" + std::to_string(model.input_c()));
    std::vector<float> logits(static_cast<std::size_t>(model.num_classes()));
    float *din = nullptr, *dout = nullptr;
    auto ck = [&](cudaError_t e) {
        if (e != cudaSuccess) {
            cudaFree(din);
            cudaFree(dout);
            throw DeviceError(std::string("run_network: ") + cudaGetErrorString(e));
        }
    };
    ck(cudaMalloc(&din, input.data.size() * sizeof(float)));
    ck(cudaMalloc(&dout, logits.size() * sizeof(float)));
    ck(cudaMemcpy(din, input.data.data(), input.data.size() * sizeof(float), cudaMemcpyHostToDevice));
    try {
        model.forward(din, 1, dout, strict, nullptr);
    } catch (...) {
        cudaFree(din);
        cudaFree(dout);
        throw;
    }
    ck(cudaMemcpy(logits.data(), dout, logits.size() * sizeof(float), cudaMemcpyDeviceToHost));
    cudaFree(din);
    cudaFree(dout);
    return logits;
}

// ------------------------------------------------------------ masks

BlockConfig::BlockConfig(int ob, int ib) : out_block(ob), in_block(ib) {
    if ((ob != 1 && ob != 2 && ob != 4) || (ib != 1 && ib != 2 && ib != 4))
        throw FormatError("block sizes must be 1, 2 or 4");
}

SparsityMask::SparsityMask(int r, int c)
    : rows(r), cols(c), bits((static_cast<std::size_t>(r) * c + 63) / 64, 0) {
    if (r < 1 || c < 1) throw ShapeError("mask dims must be >= 1");
}

bool SparsityMask::get(int r, int c) const {
    const std::size_t i = static_cast<std::size_t>(r) * cols + c;
    return (bits[i >> 6] >> (i & 63)) & 1u;
}

void SparsityMask::set(int r, int c, bool v) {
    const std::size_t i = static_cast<std::size_t>(r) * cols + c;
    const std::uint64_t m = std::uint64_t{1} << (i & 63);
    bits[i >> 6] = v ? (bits[i >> 6] | m) : (bits[i >> 6] & ~m);
}

std::int64_t SparsityMask::popcount() const {
    std::int64_t n = 0;
    for (std::uint64_t w : bits) n += __builtin_popcountll(w);
    return n;
}

SparsityMask generate_mask(int rows, int cols, double sparsity, BlockConfig block,
                           std::uint32_t seed) {
    if (sparsity < 0.0 || sparsity >= 1.0) throw std::invalid_argument("sparsity must be in [0, 1)");
    if (rows % block.out_block != 0) throw FormatError("generate_mask: rows not divisible by out_block");
    if (cols % block.in_block != 0) throw FormatError("generate_mask: cols not divisible by in_block");
    const int tcols = cols / block.in_block;
    const std::size_t tiles = static_cast<std::size_t>(rows / block.out_block) * tcols;
    const std::size_t zeroed = static_cast<std::size_t>(std::llround(static_cast<double>(tiles) * sparsity));
    // tile order after a partial shuffle: only the first `zeroed` positions matter
    std::vector<std::uint32_t> order(tiles);
    for (std::size_t i = 0; i < tiles; ++i) order[i] = static_cast<std::uint32_t>(i);
    std::mt19937 gen(seed);
    for (std::size_t i = 0; i < zeroed && i + 1 < tiles; ++i) {
        std::uniform_int_distribution<std::size_t> pick(i, tiles - 1);
        std::swap(order[i], order[pick(gen)]);
    }
    SparsityMask mask(rows, cols);
    for (auto& w : mask.bits) w = ~std::uint64_t{0};
    const std::size_t total = static_cast<std::size_t>(rows) * cols;
    if (total % 64) mask.bits.back() &= (std::uint64_t{1} << (total % 64)) - 1;  // unused tail bits clear
    for (std::size_t i = 0; i < zeroed; ++i) {
        const int tr = static_cast<int>(order[i] / tcols), tc = static_cast<int>(order[i] % tcols);
        for (int dr = 0; dr < block.out_block; ++dr)
            for (int dc = 0; dc < block.in_block; ++dc)
                mask.set(tr * block.out_block + dr, tc * block.in_block + dc, false);
    }
    return mask;
}

void apply_mask(DenseMatrix& w, const SparsityMask& mask) {
    if (w.rows != mask.rows || w.cols != mask.cols) throw ShapeError("apply_mask: matrix/mask shape mismatch");
    for (int r = 0; r < w.rows; ++r)
        for (int c = 0; c < w.cols; ++c)
            if (!mask.get(r, c)) w.data[static_cast<std::size_t>(r) * w.cols + c] = 0.0f;
}

}  // namespace spcv
