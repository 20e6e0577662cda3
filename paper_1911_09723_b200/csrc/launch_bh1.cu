// launch_bh1.cu — kernels for block height 1, 16 B-aligned layouts (separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh1_unaligned(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                         bool strict, cudaStream_t st);  // launch_bh1u.cu

int launch_bh1(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t st) {
    return vec ? launch_bh<1, true>(a, w, ntiles, sms, strict, st)
               : launch_bh1_unaligned(a, w, ntiles, sms, strict, st);
}

}  // namespace spcv_detail
