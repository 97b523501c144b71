// bwd_dk78.cu -- instantiation unit of the backward kernels for d_k = 7, 8
// (see bwd_kernels.cuh; split for parallel compilation).
#include "bwd_inst.cuh"

namespace onedf {
template void launch_bwd_query_dk<7>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_query_dk<8>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<7>(const KeyArgs&, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<8>(const KeyArgs&, int, int, unsigned, cudaStream_t);
}  // namespace onedf
