// launch_bh1u.cu — kernels for block height 1, unaligned layouts (4 B staging; separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh1_unaligned(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                         bool strict, cudaStream_t st) {
    return launch_bh<1, false>(a, w, ntiles, sms, strict, st);
}

}  // namespace spcv_detail
