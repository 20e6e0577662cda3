// launch_bh4u.cu — kernels for block height 4, unaligned layouts (4 B staging; separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh4_unaligned(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                         bool strict, cudaStream_t st) {
    return launch_bh<4, false>(a, w, ntiles, sms, strict, st);
}

}  // namespace spcv_detail
