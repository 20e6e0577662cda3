// launch_bh2.cu — kernels for block height 2 (separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh2(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t st) {
    return launch_bh<2>(a, w, ntiles, sms, strict, vec, st);
}

}  // namespace spcv_detail
