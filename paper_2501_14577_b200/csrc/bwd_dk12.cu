// bwd_dk12.cu -- instantiation unit of the backward kernels for d_k = 1, 2
// (see bwd_kernels.cuh; split for parallel compilation).
#include "bwd_inst.cuh"

namespace onedf {
template void launch_bwd_query_dk<1>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_query_dk<2>(const BwdArgs&, int, int, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<1>(const KeyArgs&, int, int, unsigned, cudaStream_t);
template void launch_bwd_key_dk<2>(const KeyArgs&, int, int, unsigned, cudaStream_t);
}  // namespace onedf
