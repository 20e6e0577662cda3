// model.cu — SPCV model file -> device upload.
//
// Parses the reference's model container (format: model_io.hpp:48-55,
// serialize_model model_io.cpp:146-227, parse_model model_io.cpp:238-381)
// with the same checks in the same order and the same typed errors, then
// packs every sparse 1x1 / classifier layer once onto the device
// (spcv_cu_pack) with its bias, and uploads dense ones as row-major
// matrices. Layer i of the loaded model then runs as the executor's
// pointwise step (run_network, netdef.cpp:494-512) via spcv_cu_model_run.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "model_internal.h"

using namespace spcv_detail;
using namespace spcv_model;

namespace {

// ------------------------------------------------------------------ errors
// Thrown inside the parser only; mapped to status codes at the C-ABI.
struct ParseError {
    int code;
    std::string msg;
};
[[noreturn]] void raise(int code, const std::string& msg) { throw ParseError{code, msg}; }
void check(bool ok, const std::string& what) {
    if (!ok) raise(SPCV_ERR_MODEL_FORMAT, "model file invalid: " + what);
}

// CRC-32 (IEEE 802.3, reflected 0xEDB88320): zlib's crc32(0, data, n), which
// the reference uses for the trailer (model_io.cpp:223-225, 370-373).
uint32_t crc32_ieee(const uint8_t* p, size_t n) {
    static uint32_t table[256];
    static bool ready = false;
    if (!ready) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        ready = true;
    }
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

// Little-endian reader that never trusts a length beyond the bytes present.
struct Reader {
    const uint8_t* p;
    size_t size, off = 0;
    void need(size_t n) const {
        if (n > size - off) raise(SPCV_ERR_TRUNCATED, "model file truncated at offset " + std::to_string(off));
    }
    uint8_t u8() {
        need(1);
        return p[off++];
    }
    uint16_t u16() {
        need(2);
        const uint16_t v = static_cast<uint16_t>(p[off] | (p[off + 1] << 8));
        off += 2;
        return v;
    }
    uint32_t u32() {
        need(4);
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[off + i]) << (8 * i);
        off += 4;
        return v;
    }
    uint64_t u64() {
        need(8);
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[off + i]) << (8 * i);
        off += 8;
        return v;
    }
    float f32() {
        const uint32_t b = u32();
        float v;
        std::memcpy(&v, &b, 4);
        return v;
    }
    double f64() {
        const uint64_t b = u64();
        double v;
        std::memcpy(&v, &b, 8);
        return v;
    }
    std::string str() {
        const uint32_t n = u32();
        need(n);
        std::string s(reinterpret_cast<const char*>(p + off), n);
        off += n;
        return s;
    }
    std::vector<float> f32s() {
        const uint32_t n = u32();
        need(static_cast<size_t>(n) * 4);
        std::vector<float> v(n);
        std::memcpy(v.data(), p + off, static_cast<size_t>(n) * 4);  // little-endian host
        off += static_cast<size_t>(n) * 4;
        return v;
    }
    std::vector<uint32_t> u32s() {
        const uint32_t n = u32();
        need(static_cast<size_t>(n) * 4);
        std::vector<uint32_t> v(n);
        std::memcpy(v.data(), p + off, static_cast<size_t>(n) * 4);
        off += static_cast<size_t>(n) * 4;
        return v;
    }
};

// BcsrMatrix::validate (sparse.cpp:16-51) -> message or "" when valid.
std::string bcsr_problem(const Layer& L) {
    if (L.rows < 1 || L.cols < 1) return "bcsr: dims must be >= 1";
    if (L.bh != 1 && L.bh != 2 && L.bh != 4) return "bcsr: block height must be 1, 2 or 4";
    if (L.rows % L.bh != 0) return "bcsr: rows not divisible by block height";
    const size_t brows = static_cast<size_t>(L.rows / L.bh);
    if (L.row_ptr.size() != brows + 1) return "bcsr: row_ptr length != block rows + 1";
    if (L.row_ptr.front() != 0) return "bcsr: row_ptr[0] != 0";
    for (size_t r = 0; r < brows; ++r)
        if (L.row_ptr[r] > L.row_ptr[r + 1]) return "bcsr: row_ptr not non-decreasing";
    if (L.row_ptr.back() != L.col_idx.size()) return "bcsr: row_ptr[-1] != block count";
    if (L.values.size() != L.col_idx.size() * static_cast<size_t>(L.bh))
        return "bcsr: values length != block count * block height";
    for (size_t r = 0; r < brows; ++r)
        for (uint32_t b = L.row_ptr[r]; b < L.row_ptr[r + 1]; ++b) {
            if (L.col_idx[b] >= static_cast<uint32_t>(L.cols)) return "bcsr: column index out of range";
            if (b > L.row_ptr[r] && L.col_idx[b] <= L.col_idx[b - 1])
                return "bcsr: column indices not strictly increasing";
        }
    return "";
}

// NetworkSpec::validate (netdef.cpp:27-67); failures are ModelFormatError
// in parse_model (model_io.cpp:375-379).
void validate_net(const Net& net) {
    auto bad = [](const std::string& m) { raise(SPCV_ERR_MODEL_FORMAT, "model file invalid: " + m); };
    const auto& Ls = net.layers;
    if (Ls.empty()) bad("network has no layers");
    if (Ls.front().kind != kEntryConv) bad("network must start with the entry convolution");
    if (Ls.back().kind != kFullyConnected) bad("network must end with the classifier");
    if (Ls.size() < 3 || Ls[Ls.size() - 2].kind != kGlobalPool) bad("classifier must follow global pooling");
    int c = net.input_c, h = net.input_h, w = net.input_w;
    for (size_t i = 0; i < Ls.size(); ++i) {
        const Layer& L = Ls[i];
        if (L.cin != c || L.in_h != h || L.in_w != w) bad("layer " + L.name + ": input does not chain");
        if (L.kind == kDepthwise && L.cout != L.cin) bad("layer " + L.name + ": depthwise must preserve channels");
        if (L.kind == kGlobalPool && (L.cout != L.cin || L.out_h != 1 || L.out_w != 1))
            bad("layer " + L.name + ": pooling must emit cin x 1 x 1");
        if (L.sparse && !(L.sparsity > 0.0 && L.sparsity < 1.0))
            bad("layer " + L.name + ": sparse layer needs sparsity in (0, 1)");
        if (!L.sparse && L.sparsity != 0.0) bad("layer " + L.name + ": dense layer must have sparsity 0");
        if (L.block_h != 1 && L.block_h != 2 && L.block_h != 4)
            bad("layer " + L.name + ": block height must be 1, 2 or 4");
        if (L.residual_src >= 0) {
            if (static_cast<size_t>(L.residual_src) >= i) bad("layer " + L.name + ": residual source must come earlier");
            const Layer& s = Ls[static_cast<size_t>(L.residual_src)];
            if (s.cout != L.cout || s.out_h != L.out_h || s.out_w != L.out_w)
                bad("layer " + L.name + ": residual source shape mismatch");
        }
        c = L.cout;
        h = L.out_h;
        w = L.out_w;
    }
    if (Ls.back().cout != net.num_classes) bad("classifier output does not match num_classes");
}

// parse_model (model_io.cpp:238-381), check for check.
Net parse(const uint8_t* data, size_t size) {
    Reader c{data, size};
    c.need(4);
    if (std::memcmp(data, "SPCV", 4) != 0) raise(SPCV_ERR_BAD_MAGIC, "not a model file (bad magic)");
    c.off = 4;
    const uint16_t version = c.u16();
    if (version != 1) raise(SPCV_ERR_VERSION, "unsupported model format version " + std::to_string(version));
    Net net;
    net.name = c.str();
    net.width_milli = static_cast<int>(c.u32());
    net.input_h = static_cast<int>(c.u32());
    net.input_w = static_cast<int>(c.u32());
    net.input_c = static_cast<int>(c.u32());
    net.num_classes = static_cast<int>(c.u32());
    net.plan_sparsity = c.f64();
    net.block_start = static_cast<int>(c.u32());
    net.block_h_after = static_cast<int>(c.u32());
    const uint32_t count = c.u32();
    for (uint32_t i = 0; i < count; ++i) {
        Layer L;
        L.kind = c.u8();
        check(L.kind <= kFullyConnected, "unknown layer kind " + std::to_string(L.kind));
        L.name = c.str();
        L.cin = static_cast<int>(c.u32());
        L.cout = static_cast<int>(c.u32());
        L.stride = static_cast<int>(c.u32());
        L.in_h = static_cast<int>(c.u32());
        L.in_w = static_cast<int>(c.u32());
        L.out_h = static_cast<int>(c.u32());
        L.out_w = static_cast<int>(c.u32());
        L.sparse = c.u8() != 0;
        L.sparsity = c.f64();
        L.block_h = static_cast<int>(c.u32());
        const uint8_t ak = c.u8();
        check(ak <= 1, "unknown activation kind");
        const float lo = c.f32(), hi = c.f32();
        if (ak == 1) {
            check(lo < hi, "activation clamp bounds");
            L.act_kind = 1;
            L.lo = lo;
            L.hi = hi;
        }
        L.residual_src = static_cast<int>(c.u32());
        L.bias = c.f32s();
        L.storage = c.u8();
        switch (L.kind) {
            case kGlobalPool:
                check(L.storage == kNone, "pooling layer carries weights");
                check(L.bias.empty(), "pooling layer carries a bias");
                break;
            case kEntryConv: {
                check(L.storage == kConv, "entry layer storage tag");
                const int co = static_cast<int>(c.u32()), ci = static_cast<int>(c.u32());
                const int kh = static_cast<int>(c.u32()), kw = static_cast<int>(c.u32());
                check(co == L.cout && ci == L.cin && kh == 3 && kw == 3, "entry convolution dims for layer " + L.name);
                if (co < 0 || ci < 0) raise(SPCV_ERR_CUDA, "entry convolution: allocation failure");
                L.other = c.f32s();
                check(L.other.size() == static_cast<size_t>(co) * ci * kh * kw,
                      "entry convolution value count for layer " + L.name);
                break;
            }
            case kDepthwise: {
                check(L.storage == kDw, "depthwise layer storage tag");
                const int ch = static_cast<int>(c.u32());
                check(ch == L.cout, "depthwise channel count for layer " + L.name);
                if (ch < 0) raise(SPCV_ERR_CUDA, "depthwise: allocation failure");
                L.other = c.f32s();
                check(L.other.size() == static_cast<size_t>(ch) * 9, "depthwise value count for layer " + L.name);
                break;
            }
            case kPointwise:
            case kFullyConnected: {
                if (L.storage == kDense) {
                    L.rows = static_cast<int>(c.u32());
                    L.cols = static_cast<int>(c.u32());
                    check(L.rows == L.cout && L.cols == L.cin, "dense matrix dims for layer " + L.name);
                    if (L.rows < 0 || L.cols < 0) raise(SPCV_ERR_SHAPE, "matrix dims must be >= 0");
                    L.values = c.f32s();
                    check(L.values.size() == static_cast<size_t>(L.rows) * L.cols, "dense value count for layer " + L.name);
                } else if (L.storage == kBcsr) {
                    L.rows = static_cast<int>(c.u32());
                    L.cols = static_cast<int>(c.u32());
                    L.bh = static_cast<int>(c.u32());
                    L.row_ptr = c.u32s();
                    L.col_idx = c.u32s();
                    L.values = c.f32s();
                    const std::string prob = bcsr_problem(L);  // BcsrMatrix::validate
                    if (!prob.empty()) raise(SPCV_ERR_MODEL_FORMAT, "layer " + L.name + ": " + prob);
                    check(L.cols == L.cin, "sparse matrix cols for layer " + L.name);
                    check(L.bh == L.block_h, "sparse block height for layer " + L.name);
                    check(L.rows == (L.cout + L.block_h - 1) / L.block_h * L.block_h,
                          "sparse matrix rows for layer " + L.name);
                } else {
                    raise(SPCV_ERR_MODEL_FORMAT, "model file invalid: 1x1 layer storage tag");
                }
                check(L.bias.size() == static_cast<size_t>(L.cout), "bias length for layer " + L.name);
                break;
            }
        }
        if (L.kind == kEntryConv || L.kind == kDepthwise)
            check(L.bias.size() == static_cast<size_t>(L.cout), "bias length for layer " + L.name);
        net.layers.push_back(std::move(L));
    }
    const size_t body_end = c.off;
    const uint32_t stored = c.u32();
    if (c.off != size) raise(SPCV_ERR_MODEL_FORMAT, "model file invalid: trailing bytes after checksum");
    if (stored != crc32_ieee(data, body_end)) raise(SPCV_ERR_CHECKSUM, "model file checksum mismatch");
    validate_net(net);
    return net;
}

}  // namespace

namespace {

void free_model(spcv_cu_model* m) {
    if (!m) return;
    for (auto* w : m->w) spcv_cu_free(w);
    for (float* p : m->d_dense) cudaFree(p);
    for (float* p : m->d_bias) cudaFree(p);
    for (float* p : m->d_conv) cudaFree(p);
    if (m->pool || !m->graphs.empty()) cudaDeviceSynchronize();  // no forward may still run
    for (auto& g : m->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.done) cudaEventDestroy(g.done);
        for (float* p : g.ws) cudaFree(p);
    }
    if (m->pool) cudaMemPoolDestroy(m->pool);
    delete m;
}

int parse_status(const uint8_t* bytes, size_t size, Net* out) {
    if (!bytes && size) return fail(SPCV_ERR_INVALID, "model: null buffer");
    try {
        *out = parse(bytes, size);
        return SPCV_OK;
    } catch (const ParseError& e) {
        return fail(e.code, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(SPCV_ERR_CUDA, "model: out of host memory");
    }
}

}  // namespace

extern "C" int spcv_cu_model_parse(const uint8_t* bytes, size_t size, int* layers) {
    Net net;
    const int rc = parse_status(bytes, size, &net);
    if (rc == SPCV_OK && layers) *layers = static_cast<int>(net.layers.size());
    return rc;
}

extern "C" int spcv_cu_model_load(const uint8_t* bytes, size_t size, spcv_cu_model** out) {
    if (!out) return fail(SPCV_ERR_INVALID, "model: null out");
    *out = nullptr;
    auto* m = new (std::nothrow) spcv_cu_model;
    if (!m) return fail(SPCV_ERR_CUDA, "model: out of host memory");
    int rc = parse_status(bytes, size, &m->net);
    if (rc != SPCV_OK) {
        delete m;
        return rc;
    }
    cudaGetDevice(&m->device);
    const size_t n = m->net.layers.size();
    m->w.assign(n, nullptr);
    m->d_dense.assign(n, nullptr);
    m->d_bias.assign(n, nullptr);
    m->d_conv.assign(n, nullptr);
    auto upload = [&](float** dst, const std::vector<float>& v, const char* what) {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(v.size(), 1) * 4);
        if (e == cudaSuccess && !v.empty())
            e = cudaMemcpy(*dst, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
        return e == cudaSuccess ? SPCV_OK : cuda_fail(e, what);
    };
    for (size_t i = 0; i < n && rc == SPCV_OK; ++i) {
        Layer& L = m->net.layers[i];
        if (L.kind == kEntryConv) {
            // [co][ci][ky][kx] -> [co][ky][kx][ci]: every tap reads one HWC pixel
            // (the same repack as entry_conv_hwc_to_chw, kernels.cpp:433-441)
            std::vector<float> wp(L.other.size());
            for (int co = 0; co < L.cout; ++co)
                for (int ky = 0; ky < 3; ++ky)
                    for (int kx = 0; kx < 3; ++kx)
                        for (int ci = 0; ci < L.cin; ++ci)
                            wp[((static_cast<size_t>(co) * 3 + ky) * 3 + kx) * L.cin + ci] =
                                L.other[((static_cast<size_t>(co) * L.cin + ci) * 3 + ky) * 3 + kx];
            rc = upload(&m->d_conv[i], wp, "model: entry conv upload");
        } else if (L.kind == kDepthwise) {
            rc = upload(&m->d_conv[i], L.other, "model: depthwise upload");
        }
        if (L.kind == kEntryConv || L.kind == kDepthwise)
            L.zero_pad_exact = std::all_of(L.other.begin(), L.other.end(), [](float w) { return std::isfinite(w); }) &&
                               std::none_of(L.bias.begin(), L.bias.end(),
                                            [](float b) { return b == 0.0f && std::signbit(b); });
        if (rc == SPCV_OK && (L.kind == kEntryConv || L.kind == kDepthwise) && !L.bias.empty())
            rc = upload(&m->d_bias[i], L.bias, "model: bias upload");
        if (L.kind != kPointwise && L.kind != kFullyConnected) continue;
        if (L.storage == kBcsr) {
            rc = spcv_cu_pack(L.rows, L.cols, L.bh, L.row_ptr.data(), L.row_ptr.size(), L.col_idx.data(),
                              L.col_idx.size(), L.values.data(), L.values.size(), &m->w[i]);
        } else {
            cudaError_t e = cudaMalloc(&m->d_dense[i], std::max<size_t>(L.values.size(), 1) * 4);
            if (e == cudaSuccess && !L.values.empty())
                e = cudaMemcpy(m->d_dense[i], L.values.data(), L.values.size() * 4, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) rc = cuda_fail(e, "model: dense upload");
        }
        if (rc == SPCV_OK && !L.bias.empty()) {
            cudaError_t e = cudaMalloc(&m->d_bias[i], L.bias.size() * 4);
            if (e == cudaSuccess)
                e = cudaMemcpy(m->d_bias[i], L.bias.data(), L.bias.size() * 4, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) rc = cuda_fail(e, "model: bias upload");
        }
    }
    if (rc == SPCV_OK) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = m->device;
        cudaError_t e = cudaMemPoolCreate(&m->pool, &props);
        uint64_t keep = ~0ull;
        if (e == cudaSuccess) e = cudaMemPoolSetAttribute(m->pool, cudaMemPoolAttrReleaseThreshold, &keep);
        if (e != cudaSuccess) rc = cuda_fail(e, "model: workspace pool");
    }
    if (rc != SPCV_OK) {
        free_model(m);
        return rc;
    }
    *out = m;
    return SPCV_OK;
}

extern "C" int spcv_cu_model_layer(const spcv_cu_model* m, int i, int* info) {
    if (!m || !info) return fail(SPCV_ERR_INVALID, "model: null argument");
    if (i < 0 || static_cast<size_t>(i) >= m->net.layers.size())
        return fail(SPCV_ERR_INVALID, "model: layer index out of range");
    const Layer& L = m->net.layers[static_cast<size_t>(i)];
    const int v[12] = {L.kind, L.cin, L.cout, L.in_h, L.in_w, L.out_h, L.out_w,
                       L.storage == kBcsr ? 1 : 0, L.block_h, L.act_kind, L.residual_src, L.stride};
    std::copy(v, v + 12, info);
    return SPCV_OK;
}

extern "C" int spcv_cu_model_weights(const spcv_cu_model* m, int i, const spcv_cu_weights** w) {
    if (!m || !w) return fail(SPCV_ERR_INVALID, "model: null argument");
    if (i < 0 || static_cast<size_t>(i) >= m->net.layers.size())
        return fail(SPCV_ERR_INVALID, "model: layer index out of range");
    *w = m->w[static_cast<size_t>(i)];
    return *w ? SPCV_OK : fail(SPCV_ERR_INVALID, "model: layer is not a sparse 1x1 layer");
}

extern "C" int spcv_cu_model_run(const spcv_cu_model* m, int i, const float* act, int images,
                                 const float* residual, float* out, int mode, void* stream) {
    if (!m) return fail(SPCV_ERR_INVALID, "model: null model");
    if (i < 0 || static_cast<size_t>(i) >= m->net.layers.size())
        return fail(SPCV_ERR_INVALID, "model: layer index out of range");
    const size_t k = static_cast<size_t>(i);
    const Layer& L = m->net.layers[k];
    if (mode != SPCV_MODE_STRICT && mode != SPCV_MODE_FAST)
        return fail(SPCV_ERR_INVALID, "model: unknown arithmetic mode");
    if (L.kind == kEntryConv || L.kind == kDepthwise || L.kind == kGlobalPool) {
        if (images < 0) return fail(SPCV_ERR_SHAPE, "model: negative image count");
        if (images == 0) return SPCV_OK;
        if (!act || !out) return fail(SPCV_ERR_INVALID, "model: null tensor pointer");
        return run_spatial_layer(m, k, act, images, out, mode, static_cast<cudaStream_t>(stream));
    }
    if (L.kind != kPointwise && L.kind != kFullyConnected)
        return fail(SPCV_ERR_INVALID, "model: layer " + L.name + " is not a 1x1 / classifier layer");
    if (L.residual_src >= 0 && !residual)
        return fail(SPCV_ERR_INVALID, "model: layer " + L.name + " needs its residual input");
    if (m->w[k])
        return spcv_cu_spmm_layer(m->w[k], act, images, L.cin, L.in_h, L.in_w, m->d_bias[k],
                                  L.bias.size(), L.act_kind, L.lo, L.hi, L.residual_src >= 0 ? residual : nullptr,
                                  out, L.cout, mode, stream);
    if (L.residual_src >= 0)
        return fail(SPCV_ERR_UNSUPPORTED, "model: residual add on a dense layer is not supported");
    return spcv_cu_dense_gemm_into(m->d_dense[k], L.rows, L.cols, act, SPCV_LAYOUT_CHW, images, L.cin,
                                   L.in_h, L.in_w, m->d_bias[k], L.bias.size(), L.act_kind, L.lo, L.hi,
                                   out, SPCV_LAYOUT_CHW, L.cout, L.out_h, L.out_w, 0, stream);
}

extern "C" void spcv_cu_model_free(spcv_cu_model* m) { free_model(m); }
