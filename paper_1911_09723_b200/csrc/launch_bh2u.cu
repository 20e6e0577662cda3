// launch_bh2u.cu — kernels for block height 2, unaligned layouts (4 B staging; separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh2_unaligned(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                         bool strict, cudaStream_t st) {
    return launch_bh<2, false>(a, w, ntiles, sms, strict, st);
}

}  // namespace spcv_detail
