// bwd_inst.cu -- definitions of the per-(d_k, storage type) launchers of
// bwd_kernels.cuh.  build.py compiles this file once per instantiation unit
// (ONEDF_INST_DK_A/_B = two d_k values, ONEDF_INST_TV = float or bf16), so the
// many kernel instantiations compile in parallel.
#include "bwd_kernels.cuh"

#if !defined(ONEDF_INST_DK_A) || !defined(ONEDF_INST_DK_B) || !defined(ONEDF_INST_TV)
#error "bwd_inst.cu is compiled per unit with -DONEDF_INST_DK_A=.. -DONEDF_INST_DK_B=.. -DONEDF_INST_TV=.. (build.py)"
#endif

namespace onedf {

template <int DK, typename TV, int PV, int CHV, int RV>
static void bwd_query_launch(const BwdArgs& a, int nch, unsigned grid, cudaStream_t st) {
    if (PV * CHV == nch) bwd_query_kernel<DK, PV, CHV, RV, true, TV><<<grid, BWD_THREADS, 0, st>>>(a);
    else bwd_query_kernel<DK, PV, CHV, RV, false, TV><<<grid, BWD_THREADS, 0, st>>>(a);
}

template <int DK, typename TV, int PV, int RV>
static void bwd_query_launch_ch(const BwdArgs& a, int nch, int dv, unsigned grid, cudaStream_t st) {
    if (PV == 32 && dv > 128) bwd_query_launch<DK, TV, PV, 2, RV>(a, nch, grid, st);
    else bwd_query_launch<DK, TV, PV, 1, RV>(a, nch, grid, st);
}

template <int DK, typename TV, int PV>
static void bwd_query_launch_r(const BwdArgs& a, int nch, int dv, int k, unsigned grid, cudaStream_t st) {
    if (k <= 32) bwd_query_launch_ch<DK, TV, PV, 1>(a, nch, dv, grid, st);
    else if (k <= 64) bwd_query_launch_ch<DK, TV, PV, 2>(a, nch, dv, grid, st);
    else if (k <= 128) bwd_query_launch_ch<DK, TV, PV, 4>(a, nch, dv, grid, st);
    else bwd_query_launch_ch<DK, TV, PV, 8>(a, nch, dv, grid, st);
}

template <int DK, typename TV>
void launch_bwd_query_dk(const BwdArgs& a, int P, int nch, int dv, int k, unsigned grid, cudaStream_t st) {
    if (!grid) return;
    if (P == 4) bwd_query_launch_r<DK, TV, 4>(a, nch, dv, k, grid, st);
    else if (P == 8) bwd_query_launch_r<DK, TV, 8>(a, nch, dv, k, grid, st);
    else if (P == 16) bwd_query_launch_r<DK, TV, 16>(a, nch, dv, k, grid, st);
    else bwd_query_launch_r<DK, TV, 32>(a, nch, dv, k, grid, st);
}

// WHOLE: d_v == 4*P*CH (every lane chunk exists; d_v a compile-time constant in the gathers)
template <int DK, typename TV, int PV, int CHV>
static void bwd_key_launch(const KeyArgs& ka, int dv, unsigned grid, cudaStream_t st) {
    if (4 * PV * CHV == dv) bwd_key_kernel<DK, PV, CHV, true, TV><<<grid, BWD_THREADS, 0, st>>>(ka);
    else bwd_key_kernel<DK, PV, CHV, false, TV><<<grid, BWD_THREADS, 0, st>>>(ka);
}

template <int DK, typename TV>
void launch_bwd_key_dk(const KeyArgs& ka, int P, int dv, unsigned grid, cudaStream_t st) {
    if (!grid) return;
    if (P == 4) bwd_key_launch<DK, TV, 4, 1>(ka, dv, grid, st);
    else if (P == 8) bwd_key_launch<DK, TV, 8, 1>(ka, dv, grid, st);
    else if (P == 16) bwd_key_launch<DK, TV, 16, 1>(ka, dv, grid, st);
    else if (dv > 128) bwd_key_launch<DK, TV, 32, 2>(ka, dv, grid, st);
    else bwd_key_launch<DK, TV, 32, 1>(ka, dv, grid, st);
}

template void launch_bwd_query_dk<ONEDF_INST_DK_A, ONEDF_INST_TV>(const BwdArgs&, int, int, int, int, unsigned,
                                                                  cudaStream_t);
template void launch_bwd_key_dk<ONEDF_INST_DK_A, ONEDF_INST_TV>(const KeyArgs&, int, int, unsigned, cudaStream_t);
template void launch_bwd_query_dk<ONEDF_INST_DK_B, ONEDF_INST_TV>(const BwdArgs&, int, int, int, int, unsigned,
                                                                  cudaStream_t);
template void launch_bwd_key_dk<ONEDF_INST_DK_B, ONEDF_INST_TV>(const KeyArgs&, int, int, unsigned, cudaStream_t);

}  // namespace onedf
