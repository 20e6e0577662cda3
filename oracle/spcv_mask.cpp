// spcv_mask.cpp — CPU restatement of the reference's seeded mask generator.
//
// TEST INFRASTRUCTURE ONLY (see spcv_oracle.c header). Used by tests and by
// input generation in the CPU-side checkers; never by the product path.
//
// generate_mask — /root/reference/proj/src/sparse.cpp:63-98. Zeroes
// llround(tiles * sparsity) whole out_block x in_block tiles chosen by a
// partial Fisher–Yates shuffle driven by std::mt19937(seed) and
// std::uniform_int_distribution<std::size_t>(i, tiles - 1). The distribution's
// algorithm is implementation-defined; this file and the reference are built
// by the same g++/libstdc++ here, so masks agree bit-for-bit (pinned by
// tests/test_oracle.py against oracle/_ref).
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>
#include <utility>
#include <vector>

extern "C" int oracle_generate_mask(int rows, int cols, double sparsity, int out_block,
                                    int in_block, std::uint32_t seed, std::uint8_t* keep) {
    if (sparsity < 0.0 || sparsity >= 1.0) return 4;  // std::invalid_argument
    if ((out_block != 1 && out_block != 2 && out_block != 4) ||
        (in_block != 1 && in_block != 2 && in_block != 4))
        return 3;  // FormatError (BlockConfig)
    if (rows < 1 || cols < 1) return 2;
    if (rows % out_block != 0 || cols % in_block != 0) return 3;

    const int trows = rows / out_block;
    const int tcols = cols / in_block;
    const std::size_t tiles = static_cast<std::size_t>(trows) * static_cast<std::size_t>(tcols);
    const std::size_t zeroed =
        static_cast<std::size_t>(std::llround(static_cast<double>(tiles) * sparsity));

    std::vector<std::uint32_t> pos(tiles);
    for (std::size_t i = 0; i < tiles; ++i) pos[i] = static_cast<std::uint32_t>(i);
    std::mt19937 rng(seed);
    for (std::size_t i = 0; i < zeroed && i + 1 < tiles; ++i) {
        std::uniform_int_distribution<std::size_t> d(i, tiles - 1);
        std::swap(pos[i], pos[d(rng)]);
    }
    const std::size_t n = static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols);
    for (std::size_t i = 0; i < n; ++i) keep[i] = 1;
    for (std::size_t i = 0; i < zeroed; ++i) {
        const int tr = static_cast<int>(pos[i] / static_cast<std::uint32_t>(tcols));
        const int tc = static_cast<int>(pos[i] % static_cast<std::uint32_t>(tcols));
        for (int dr = 0; dr < out_block; ++dr)
            for (int dc = 0; dc < in_block; ++dc)
                keep[static_cast<std::size_t>(tr * out_block + dr) * cols + tc * in_block + dc] = 0;
    }
    return 0;
}
