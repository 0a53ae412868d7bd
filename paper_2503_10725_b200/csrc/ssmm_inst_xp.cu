// Explicit instantiations of the SSMM kernel with the in-smem row expansion of
// (N, 2N, 32) weights (split for parallel compilation).
#include "ssmm_kernel.cuh"

namespace smy {
template smy_status launch_t<16,1,2,1,1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<32,1,2,1,1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<64,1,2,1,1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<128,1,2,1,1>(const SsmmArgs&, cudaStream_t);
}  // namespace smy
