// Prints spcv::generate_mask (C++ mirror, include/spcv_b200/spcv.hpp) as 0/1
// rows for the cases given on the command line: rows cols sparsity ob ib seed.
#include <cstdio>
#include <cstdlib>

#include "spcv_b200/spcv.hpp"

int main(int argc, char** argv) {
    for (int a = 1; a + 5 < argc; a += 6) {
        const int rows = std::atoi(argv[a]), cols = std::atoi(argv[a + 1]);
        const double s = std::atof(argv[a + 2]);
        const int ob = std::atoi(argv[a + 3]), ib = std::atoi(argv[a + 4]);
        const unsigned seed = static_cast<unsigned>(std::strtoul(argv[a + 5], nullptr, 10));
        try {
            const spcv::SparsityMask m = spcv::generate_mask(rows, cols, s, spcv::BlockConfig(ob, ib), seed);
            std::printf("%lld ", static_cast<long long>(m.popcount()));
            for (int r = 0; r < rows; ++r)
                for (int c = 0; c < cols; ++c) std::putchar(m.get(r, c) ? '1' : '0');
            std::putchar('\n');
        } catch (const spcv::FormatError&) {
            std::printf("FormatError\n");
        } catch (const std::invalid_argument&) {
            std::printf("invalid_argument\n");
        }
    }
    return 0;
}
