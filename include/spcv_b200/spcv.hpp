// spcv_b200/spcv.hpp — C++ drop-in for the reference SpMM operator surface.
//
// A caller of the reference library
//   #include "spcv/kernels.hpp"     (spmm_into / spmm / spconv_1x1, kernels.hpp:28-55)
//   #include "spcv/sparse.hpp"      (BcsrMatrix, FormatError, sparse.hpp:12-79)
//   #include "spcv/tensor.hpp"      (Tensor, Activation, ShapeError/LayoutError, tensor.hpp:11-97)
// switches to this header and links libspcv_b200.so. Names, argument meaning,
// validation order and exception classes are the reference's; the work runs
// on the B200 through the C-ABI in include/spcv_cu.h (no CPU fallback: with no
// usable CUDA device every call throws spcv::DeviceError).
//
// Additions for device-resident use (no reference counterpart):
// DeviceBcsr (weights packed once, kept on the GPU) and spmm_batched_into
// (NCHW batches on device memory, caller's stream).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../spcv_cu.h"

namespace spcv {

// ---------------------------------------------------------------- errors
// Same hierarchy as tensor.hpp:11-21 and sparse.hpp:12-15.
class ShapeError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class LayoutError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class FormatError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
/// CUDA failure or a shape beyond this build's device limits (no reference
/// counterpart: the reference cannot fail this way).
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- tensors
enum class Layout : std::uint8_t { CHW, HWC };

/// Single-image host tensor (tensor.hpp:30-54): dims >= 1, owns its floats.
struct Tensor {
    int channels = 0;
    int height = 0;
    int width = 0;
    Layout layout = Layout::CHW;
    std::vector<float> data;

    Tensor() = default;
    Tensor(int c, int h, int w, Layout l);

    int spatial() const { return height * width; }
    std::size_t size() const { return data.size(); }
    std::size_t index(int c, int h, int w) const;
    float at(int c, int h, int w) const { return data[index(c, h, w)]; }
    float& at(int c, int h, int w) { return data[index(c, h, w)]; }
};

/// Row-major dense weight matrix (tensor.hpp:57-70).
struct DenseMatrix {
    int rows = 0;
    int cols = 0;
    std::vector<float> data;

    DenseMatrix() = default;
    DenseMatrix(int r, int c);
    float operator()(int r, int c) const { return data[static_cast<std::size_t>(r) * cols + c]; }
    float& operator()(int r, int c) { return data[static_cast<std::size_t>(r) * cols + c]; }
};

/// Fused output activation (tensor.hpp:74-97). Clamp uses the ternary compare,
/// so NaN passes through and -0.0 is kept.
struct Activation {
    enum class Kind : std::uint8_t { None, Clamp } kind = Kind::None;
    float lo = 0.0f;
    float hi = 0.0f;

    static Activation none() { return {}; }
    static Activation clamp(float lo, float hi);
    static Activation relu6() { return clamp(0.0f, 6.0f); }
    float apply(float x) const {
        if (kind == Kind::Clamp) return x < lo ? lo : (x > hi ? hi : x);
        return x;
    }
};

// ------------------------------------------------------------ BCSR format
/// Nx1 block-CSR weights, exactly the reference layout (sparse.hpp:65-79).
struct BcsrMatrix {
    int rows = 0;
    int cols = 0;
    int block_h = 1;
    std::vector<std::uint32_t> row_ptr;
    std::vector<std::uint32_t> col_idx;
    std::vector<float> values;

    int block_rows() const { return rows / block_h; }
    std::size_t nnz_blocks() const { return col_idx.size(); }
    std::size_t nnz_values() const { return values.size(); }
    /// Same checks and order as sparse.cpp:16-51; throws FormatError.
    void validate() const;
};

/// encode_bcsr / decode_bcsr (sparse.cpp:108-148): host-side preparation.
/// sparse.hpp:20-28: tile shape of a sparsity mask.
struct BlockConfig {
    int out_block = 1;
    int in_block = 1;
    explicit BlockConfig(int ob = 1, int ib = 1);
};

/// sparse.hpp:30-57: bit-packed keep mask over a rows x cols matrix (row-major).
struct SparsityMask {
    int rows = 0;
    int cols = 0;
    std::vector<std::uint64_t> bits;
    SparsityMask() = default;
    SparsityMask(int r, int c);
    bool get(int r, int c) const;
    void set(int r, int c, bool v);
    std::int64_t popcount() const;
};

/// sparse.cpp:63-98: zero llround(tiles * sparsity) whole tiles chosen by a
/// partial Fisher-Yates shuffle with std::mt19937(seed); same checks.
SparsityMask generate_mask(int rows, int cols, double sparsity, BlockConfig block,
                           std::uint32_t seed);
/// sparse.cpp:100-106.
void apply_mask(DenseMatrix& w, const SparsityMask& mask);

BcsrMatrix encode_bcsr(const DenseMatrix& w, int block_h);
DenseMatrix decode_bcsr(const BcsrMatrix& m);

// ---------------------------------------------------------------- kernels
/// kernels.hpp:18. One CUDA path serves every tier; the tier is accepted for
/// source compatibility. SPCV_FORCE_SCALAR is honoured by resolve_tier only.
enum class Tier : std::uint8_t { Scalar, Vector, Auto };

/// kernels.hpp:28-33. `m` (CPU strip width) is validated as in the reference
/// ({0,4,8,16}) and otherwise ignored; `n` must equal the matrix block height;
/// `prefetch` is a hint. `strict` selects the bit-exact arithmetic (default)
/// versus FFMA contraction (within the north_star tolerance).
struct MicrokernelConfig {
    int m = 0;
    int n = 1;
    bool prefetch = true;
    Tier tier = Tier::Auto;
    bool strict = true;
};

bool vector_tier_available();
Tier resolve_tier(Tier requested);
const char* tier_name(Tier t);
Tier parse_tier(const std::string& s);
int default_strip_width(Tier resolved);
std::string variant_name(int m, int n);
std::pair<int, int> parse_variant(const std::string& s);

/// kernels.hpp:45-46: out[c,s] = fused(bias[c] + sum value*act[col,s]).
/// Host tensors: the call packs `w`, copies `act`/`bias` to the device, runs
/// the kernel and copies `out` back (synchronous).
void spmm_into(const BcsrMatrix& w, const Tensor& act, std::span<const float> bias,
               const Activation& fused, Tensor& out, const MicrokernelConfig& cfg = {});
Tensor spmm(const BcsrMatrix& w, const Tensor& act, std::span<const float> bias,
            const Activation& fused = {}, const MicrokernelConfig& cfg = {});
inline Tensor spconv_1x1(const BcsrMatrix& w, const Tensor& act, std::span<const float> bias,
                         const Activation& fused = {}, const MicrokernelConfig& cfg = {}) {
    return spmm(w, act, bias, fused, cfg);
}

/// kernels.hpp:85-90: dense baseline with the same contract (host tensors;
/// cuBLAS SGEMM in pedantic fp32 + bias/clamp epilogue, not bit-exact).
void dense_gemm_into(const DenseMatrix& w, const Tensor& act, std::span<const float> bias,
                     const Activation& fused, Tensor& out, const MicrokernelConfig& cfg = {});
Tensor dense_gemm_baseline(const DenseMatrix& w, const Tensor& act, std::span<const float> bias,
                           const Activation& fused = {}, const MicrokernelConfig& cfg = {});

// ------------------------------------------------------- device-resident
/// Weights packed once onto the current CUDA device (RAII over spcv_cu_weights).
class DeviceBcsr {
public:
    DeviceBcsr() = default;
    explicit DeviceBcsr(const BcsrMatrix& m);
    DeviceBcsr(const DeviceBcsr&) = delete;
    DeviceBcsr& operator=(const DeviceBcsr&) = delete;
    DeviceBcsr(DeviceBcsr&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    DeviceBcsr& operator=(DeviceBcsr&& o) noexcept;
    ~DeviceBcsr();

    const spcv_cu_weights* handle() const { return h_; }
    int rows() const;
    int cols() const;
    int block_h() const;
    /// Bit-exact device decode back to the reference format.
    BcsrMatrix unpack() const;

private:
    spcv_cu_weights* h_ = nullptr;
};

/// spmm_into over `images` CHW images in device memory (act [images][cols][H*W],
/// out [images][rows][H*W], bias device pointer or nullptr), asynchronous on
/// `stream` (a cudaStream_t). Same validation order as spmm_into.
void spmm_batched_into(const DeviceBcsr& w, const float* d_act, int images, int height, int width,
                       const float* d_bias, const Activation& fused, float* d_out,
                       const MicrokernelConfig& cfg = {}, void* stream = nullptr);

/// The executor's pointwise step (run_network, netdef.cpp:494-512) on device
/// tensors: `w` may carry up to block_h-1 padded rows beyond `out_channels`
/// (computed, never stored), `d_bias` has out_channels entries (or nullptr),
/// and `d_residual` (nullptr or [images][out_channels][H*W]) is added after the
/// activation. Asynchronous on `stream`.
void spmm_layer(const DeviceBcsr& w, const float* d_act, int images, int height, int width,
                const float* d_bias, const Activation& fused, const float* d_residual, float* d_out,
                int out_channels, bool strict = true, void* stream = nullptr);

// ------------------------------------------------------------ model files
/// model_io.hpp:13-41: the model-file error family.
class ModelIoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class BadMagicError : public ModelIoError {
public:
    using ModelIoError::ModelIoError;
};
class UnsupportedVersionError : public ModelIoError {
public:
    using ModelIoError::ModelIoError;
};
class TruncatedError : public ModelIoError {
public:
    using ModelIoError::ModelIoError;
};
class ChecksumError : public ModelIoError {
public:
    using ModelIoError::ModelIoError;
};
class ModelFormatError : public ModelIoError {
public:
    using ModelIoError::ModelIoError;
};

/// An SPCV model file (parse_model, model_io.cpp:238-381: same checks, same
/// typed errors) uploaded once onto the current CUDA device, and the executor
/// (run_network, netdef.cpp:456-524) over it with every activation on the device.
class DeviceModel {
public:
    explicit DeviceModel(std::span<const std::uint8_t> bytes);
    /// load_model (model_io.cpp): read the file, then as above.
    static DeviceModel load(const std::string& path);
    DeviceModel(const DeviceModel&) = delete;
    DeviceModel& operator=(const DeviceModel&) = delete;
    DeviceModel(DeviceModel&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {
        for (int i = 0; i < 5; ++i) meta_[i] = o.meta_[i];
    }
    ~DeviceModel();

    int num_layers() const { return meta_[0]; }
    int input_h() const { return meta_[1]; }
    int input_w() const { return meta_[2]; }
    int input_c() const { return meta_[3]; }
    int num_classes() const { return meta_[4]; }
    const spcv_cu_model* handle() const { return h_; }

    /// run_network over `images` HWC images in device memory: d_input
    /// [images][H][W][C] -> d_logits [images][num_classes], asynchronous on
    /// `stream`. strict = bit-identical to the reference executor.
    void forward(const float* d_input, int images, float* d_logits, bool strict = true,
                 void* stream = nullptr) const;

private:
    spcv_cu_model* h_ = nullptr;
    int meta_[5] = {0, 0, 0, 0, 0};
};

/// run_network(net, ws, input) for one host HWC image (netdef.cpp:456): copy
/// in, forward on the device, copy the logits out. Input checks as
/// check_run_inputs (netdef.cpp:433-441): ShapeError.
std::vector<float> run_network(const DeviceModel& model, const Tensor& input, bool strict = true);

/// Throws the reference exception class matching an spcv_status code.
void throw_status(int status, const char* message);

}  // namespace spcv
