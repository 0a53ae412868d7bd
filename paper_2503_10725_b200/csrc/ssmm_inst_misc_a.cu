// Explicit instantiations of the SSMM kernel (split for parallel compilation).
#include "ssmm_kernel.cuh"

namespace smy {
template smy_status launch_t<32,1,2,2>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<32,2,2,2>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<32,1,4,1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<16,1,8,1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_t<16,1,16,1>(const SsmmArgs&, cudaStream_t);
}  // namespace smy
