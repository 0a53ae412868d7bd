// Explicit instantiations of the CTA-pair SSMM kernel.
#include "ssmm_pair.cuh"

namespace smy {
template smy_status launch_pair_t<64, 2, 2, 0>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<112, 2, 2, 0>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<128, 1, 2, 0>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<128, 1, 2, 1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<SMY_NT_WIDE, 1, 2, 0>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<SMY_NT_WIDE, 1, 2, 1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<128, 1, 1, 0>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<256, 1, 1, 0>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<224, 2, 1, 1>(const SsmmArgs&, cudaStream_t);
template smy_status launch_pair_t<SMY_MTP_NT, 2, 2, 1>(const SsmmArgs&, cudaStream_t);
}  // namespace smy
