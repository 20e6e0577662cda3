// C++ drop-in check of the model-file API: spcv::DeviceModel + spcv::run_network
// (include/spcv_b200/spcv.hpp) against logits the reference's run_network wrote.
//   test_model <model.spcv> <input_hwc.f32> <logits.f32>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <vector>

#include "spcv_b200/spcv.hpp"

static int failures = 0, checks = 0;
#define CHECK(cond)                                                    \
    do {                                                               \
        ++checks;                                                      \
        if (!(cond)) {                                                 \
            ++failures;                                                \
            std::printf("FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                              \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<std::uint8_t> slurp(const char* path) {
    std::ifstream f(path, std::ios::binary);
    return std::vector<std::uint8_t>(std::istreambuf_iterator<char>(f), {});
}

int main(int argc, char** argv) {
    if (argc != 4) {
        std::printf("usage: test_model <model> <input> <logits>\n");
        return 2;
    }
    const std::vector<std::uint8_t> bytes = slurp(argv[1]);
    const std::vector<std::uint8_t> in = slurp(argv[2]), want = slurp(argv[3]);

    spcv::DeviceModel m = spcv::DeviceModel::load(argv[1]);
    spcv::Tensor x(m.input_c(), m.input_h(), m.input_w(), spcv::Layout::HWC);
    CHECK(in.size() == x.data.size() * 4);
    std::memcpy(x.data.data(), in.data(), in.size());
    const std::vector<float> got = spcv::run_network(m, x);
    CHECK(got.size() * 4 == want.size());
    CHECK(std::memcmp(got.data(), want.data(), want.size()) == 0);  // bit-identical logits

    // typed errors, as parse_model / check_run_inputs raise them
    CHECK(throws<spcv::ModelIoError>([] { spcv::DeviceModel::load("/nonexistent/model.spcv"); }));
    std::vector<std::uint8_t> bad = bytes;
    bad[0] = 'X';
    CHECK(throws<spcv::BadMagicError>([&] { spcv::DeviceModel d{std::span<const std::uint8_t>(bad)}; }));
    std::vector<std::uint8_t> cut(bytes.begin(), bytes.begin() + bytes.size() / 2);
    CHECK(throws<spcv::TruncatedError>([&] { spcv::DeviceModel d{std::span<const std::uint8_t>(cut)}; }));
    std::vector<std::uint8_t> flip = bytes;
    flip[flip.size() - 1] ^= 0x55;
    CHECK(throws<spcv::ChecksumError>([&] { spcv::DeviceModel d{std::span<const std::uint8_t>(flip)}; }));
    spcv::Tensor wrong(m.input_c(), m.input_h() + 1, m.input_w(), spcv::Layout::HWC);
    CHECK(throws<spcv::ShapeError>([&] { spcv::run_network(m, wrong); }));

    std::printf("%s: %d/%d checks passed\n", failures ? "FAIL" : "all", checks - failures, checks);
    return failures ? 1 : 0;
}
