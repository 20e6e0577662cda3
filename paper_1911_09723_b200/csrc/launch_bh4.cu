// launch_bh4.cu — kernels for block height 4, 16 B-aligned layouts (separate TU: parallel build).
#include "launch.cuh"

namespace spcv_detail {

int launch_bh4_unaligned(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
                         bool strict, cudaStream_t st);  // launch_bh4u.cu

int launch_bh4(const spcvk::KernelArgs& a, const spcv_cu_weights* w, long long ntiles, int sms,
               bool strict, bool vec, cudaStream_t st) {
    return vec ? launch_bh<4, true>(a, w, ntiles, sms, strict, st)
               : launch_bh4_unaligned(a, w, ntiles, sms, strict, st);
}

}  // namespace spcv_detail
