// bwd_dk34.cu -- instantiation unit of the backward kernels for d_k = 3, 4
// (see bwd_kernels.cuh; split for parallel compilation).
#include "bwd_inst.cuh"

namespace onedf {
template void launch_bwd_query_dk<3>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_query_dk<4>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<3>(const KeyArgs&, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<4>(const KeyArgs&, int, int, unsigned, cudaStream_t);
}  // namespace onedf
