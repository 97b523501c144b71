// fwd_inst.cu -- definition of the per-storage-type K6 launcher of
// fwd_kernels.cuh.  build.py compiles this file once per (value storage type,
// register rows R) unit (ONEDF_INST_TV = float or bf16, ONEDF_INST_R = 1, 2,
// 4, 8) so the instantiation sets compile in parallel.
#include "fwd_kernels.cuh"

#if !defined(ONEDF_INST_TV) || !defined(ONEDF_INST_R)
#error "fwd_inst.cu is compiled per unit with -DONEDF_INST_TV=float|bf16 -DONEDF_INST_R=1|2|4|8 (build.py)"
#endif

namespace onedf {

// The top-k attention launch for one (value storage type, register rows R) unit.
template <typename TV, int R>
void launch_fwd_tv(const FwdArgs& a, const onedf_problem* p, unsigned grid, cudaStream_t st) {
    if (!grid) return;
    ONEDF_DISPATCH_DK(p->d_k, {
        if (p->select) code_select_attn_kernel<DK, R, TV><<<grid, FWD_THREADS, 0, st>>>(a);
        else topk_attn_fwd_kernel<DK, R, TV><<<grid, FWD_THREADS, 0, st>>>(a);
    });
}

template void launch_fwd_tv<ONEDF_INST_TV, ONEDF_INST_R>(const FwdArgs&, const onedf_problem*, unsigned, cudaStream_t);

}  // namespace onedf

#if defined(ONEDF_FWD_STATS) && defined(ONEDF_INST_TV_FLOAT) && ONEDF_INST_R == 2
// tools only (variant builds): [queries, sum cnt, sum cnt^2, fallbacks] of the float k <= 64 kernels
// (without -rdc each unit has its own copy of g_fwd_stats), then reset
extern "C" int onedf_debug_fwd_stats(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, onedf::g_fwd_stats, 8 * sizeof(unsigned long long));
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(onedf::g_fwd_stats, z, sizeof(z));
    return 0;
}
#endif
