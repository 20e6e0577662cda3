// launch_bh2.cu — kernels for block height 2, 16 B-aligned layouts (separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh2_unaligned(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                         bool strict, cudaStream_t st);  // launch_bh2u.cu

int launch_bh2(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t st) {
    return vec ? launch_bh<2, true>(a, w, ntiles, sms, strict, st)
               : launch_bh2_unaligned(a, w, ntiles, sms, strict, st);
}

}  // namespace spcv_detail
