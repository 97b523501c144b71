// bwd_dk56.cu -- instantiation unit of the backward kernels for d_k = 5, 6
// (see bwd_kernels.cuh; split for parallel compilation).
#include "bwd_inst.cuh"

namespace onedf {
template void launch_bwd_query_dk<5>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_query_dk<6>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<5>(const KeyArgs&, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<6>(const KeyArgs&, int, int, unsigned, cudaStream_t);
}  // namespace onedf
