// bwd_inst.cuh -- definitions of the per-d_k launchers of bwd_kernels.cuh;
// each bwd_dk*.cu includes this and instantiates its d_k values.
#pragma once

#include "bwd_kernels.cuh"

namespace onedf {

template <int DK, int PV, int CHV, int RV>
static void bwd_query_launch(const BwdArgs& a, int nch, unsigned grid, cudaStream_t st) {
    if (PV * CHV == nch) bwd_query_kernel<DK, PV, CHV, RV, true><<<grid, BWD_THREADS, 0, st>>>(a);
    else bwd_query_kernel<DK, PV, CHV, RV, false><<<grid, BWD_THREADS, 0, st>>>(a);
}

template <int DK, int PV, int RV>
static void bwd_query_launch_ch(const BwdArgs& a, int nch, int dv, unsigned grid, cudaStream_t st) {
    if (PV == 32 && dv > 128) bwd_query_launch<DK, PV, 2, RV>(a, nch, grid, st);
    else bwd_query_launch<DK, PV, 1, RV>(a, nch, grid, st);
}

template <int DK, int PV>
static void bwd_query_launch_r(const BwdArgs& a, int nch, int dv, int k, unsigned grid, cudaStream_t st) {
    if (k <= 32) bwd_query_launch_ch<DK, PV, 1>(a, nch, dv, grid, st);
    else if (k <= 64) bwd_query_launch_ch<DK, PV, 2>(a, nch, dv, grid, st);
    else if (k <= 128) bwd_query_launch_ch<DK, PV, 4>(a, nch, dv, grid, st);
    else bwd_query_launch_ch<DK, PV, 8>(a, nch, dv, grid, st);
}

template <int DK>
void launch_bwd_query_dk(const BwdArgs& a, int P, int nch, int dv, int k, unsigned grid, cudaStream_t st) {
    if (!grid) return;
    if (P == 4) bwd_query_launch_r<DK, 4>(a, nch, dv, k, grid, st);
    else if (P == 8) bwd_query_launch_r<DK, 8>(a, nch, dv, k, grid, st);
    else if (P == 16) bwd_query_launch_r<DK, 16>(a, nch, dv, k, grid, st);
    else bwd_query_launch_r<DK, 32>(a, nch, dv, k, grid, st);
}

template <int DK>
void launch_bwd_key_dk(const KeyArgs& ka, int P, int dv, unsigned grid, cudaStream_t st) {
    if (!grid) return;
    if (P == 4) bwd_key_kernel<DK, 4, 1><<<grid, BWD_THREADS, 0, st>>>(ka);
    else if (P == 8) bwd_key_kernel<DK, 8, 1><<<grid, BWD_THREADS, 0, st>>>(ka);
    else if (P == 16) bwd_key_kernel<DK, 16, 1><<<grid, BWD_THREADS, 0, st>>>(ka);
    else if (dv > 128) bwd_key_kernel<DK, 32, 2><<<grid, BWD_THREADS, 0, st>>>(ka);
    else bwd_key_kernel<DK, 32, 1><<<grid, BWD_THREADS, 0, st>>>(ka);
}

}  // namespace onedf
