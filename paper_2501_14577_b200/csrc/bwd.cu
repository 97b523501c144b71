// bwd.cu -- A8 backward query side (K7), A10 key side (K9), A12 eps reduce
// (K11).  The transpose (A9, K8) is in sort.cu and the mean-slot chain rule
// (A11, K10) in mean.cu.
//
// Appendix, with "dL/do_i . (v_j - o_i)/Z_i" read as a d_v-wide
// dot product (D15) and I held fixed (D16):
//   c_i   = dO_i . o_i,     g_ij = (dO_i . v_j - c_i)/Z_i,   delta = D_ij + eps
//   A_ij  = (1/delta)/Z_i,  w_ij = 2 g_ij / delta^2
//   dq_i  = -sum_j w_ij (q_i - k_j)
//   deps  = -sum_ij g_ij / delta^2
//   dv_j  = sum_{i: j in I_i} A_ij dO_i
//   dk_j  = sum_{i: j in I_i} w_ij (q_i - k_j)
// plus the mean slot as one more slot (its A, w go to the A11 scan).
//
// K7: one warp per query; a LANE per slot (each lane reads a whole v_j row
// as float4 bursts and dots it with dO_i broadcast from shared memory), so
// the 64-wide dot products need no shuffles; f64 arithmetic throughout.
// K9: one warp per key j walks its CSR segment of (query, slot) pairs in
// ascending slot order (the stable transpose fixes the order), with f64
// accumulators: a deterministic segment reduction, no float atomics.
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int BWD_WARPS = 8;
constexpr int BWD_THREADS = BWD_WARPS * 32;
constexpr int MAX_DV = 256;

void bwd_carve(const onedf_problem* p, Carver* c, BwdBufs* b) {
    const int64_t BH = p->B * p->H, total = BH * p->N;
    b->coeff = c->take<float2>((size_t)(total * p->k));
    b->muco = c->take<float2>((size_t)total);
    b->eps_blocks = (int)((total + BWD_WARPS - 1) / BWD_WARPS);
    b->eps_part = c->take<double>((size_t)b->eps_blocks);
}

struct BwdArgs {
    const float* Q; const float* K; const float* V; const float* eps;
    const float* O; const float* dO; const int32_t* idx; const float* Z;
    const float* Kbar; const float* Vbar;
    float* dQ; float2* coeff; float2* muco; double* eps_part;
    int64_t N, total;
    int k, dv, causal, mean_slot;
    void* ws;
};

template <int DK>
__global__ void __launch_bounds__(BWD_THREADS) bwd_query_kernel(const BwdArgs a) {
    __shared__ __align__(16) float s_dO[BWD_WARPS][MAX_DV];
    __shared__ double s_eps[BWD_WARPS];
    const int warp = threadIdx.x / 32, lane = lane_id();
    const int64_t gq = (int64_t)blockIdx.x * BWD_WARPS + warp;
    const int64_t N = a.N;
    double deps_w = 0.0;
    if (gq < a.total) {
        const int64_t bh = gq / N, i = gq % N;
        const float e = __ldg(a.eps);
        if (gq == 0 && lane == 0 && !(e > 0.f && isfinite(e))) set_flag(a.ws, FLAG_BAD_EPS);
        const double ed = (double)e;
        const int dv = a.dv, k = a.k;
        float q[DK];
#pragma unroll
        for (int d = 0; d < DK; ++d) q[d] = __ldg(a.Q + gq * DK + d);
        // dO_i to shared memory; c_i = dO_i . o_i (fixed-order warp tree)
        float* sdo = s_dO[warp];
        double cpart = 0.0;
        for (int d = lane; d < dv; d += 32) {
            const float g = __ldg(a.dO + gq * dv + d);
            sdo[d] = g;
            cpart = fma((double)g, (double)__ldg(a.O + gq * dv + d), cpart);
        }
        const double c = warp_sum(cpart);
        __syncwarp();
        const double Zi = (double)__ldg(a.Z + gq);
        const int64_t mrow = a.causal ? i : 0;
        double dq[DK];
#pragma unroll
        for (int d = 0; d < DK; ++d) dq[d] = 0.0;
        double deps = 0.0;
        float2* crow = a.coeff + gq * k;
        if (Zi > 0.0) {
            const double invZ = 1.0 / Zi;
            const float* Vb = a.V + bh * N * (int64_t)dv;
            for (int r = lane; r < k; r += 32) {
                const int32_t j = __ldg(a.idx + gq * k + r);
                if (j < 0) { crow[r] = make_float2(0.f, 0.f); continue; }
                float kj[DK];
#pragma unroll
                for (int d = 0; d < DK; ++d) kj[d] = __ldg(a.K + (bh * N + j) * DK + d);
                const double delta = dist64<DK>(q, kj) + ed;
                const double A = (1.0 / delta) * invZ;
                const float4* vr = reinterpret_cast<const float4*>(Vb + (int64_t)j * dv);
                const float4* dr = reinterpret_cast<const float4*>(sdo);
                double dot = 0.0;
                for (int v = 0; v < dv / 4; ++v) {
                    const float4 x = __ldg(vr + v);
                    const float4 y = dr[v];
                    dot = fma((double)x.x, (double)y.x, dot);
                    dot = fma((double)x.y, (double)y.y, dot);
                    dot = fma((double)x.z, (double)y.z, dot);
                    dot = fma((double)x.w, (double)y.w, dot);
                }
                const double g = (dot - c) * invZ;
                const double inv_d2 = 1.0 / (delta * delta);
                const double w = 2.0 * g * inv_d2;
                crow[r] = make_float2((float)A, (float)w);
#pragma unroll
                for (int d = 0; d < DK; ++d) dq[d] -= w * ((double)q[d] - (double)kj[d]);
                deps -= g * inv_d2;
            }
            if (a.mean_slot) {
                // mean slot: dims split over lanes for the dot product
                double dpart = 0.0;
                const float* vbar = a.Vbar + (bh * (a.causal ? N : 1) + mrow) * (int64_t)dv;
                for (int d = lane; d < dv; d += 32) dpart = fma((double)sdo[d], (double)__ldg(vbar + d), dpart);
                const double dot = warp_sum(dpart);
                float kb[DK];
#pragma unroll
                for (int d = 0; d < DK; ++d) kb[d] = __ldg(a.Kbar + (bh * (a.causal ? N : 1) + mrow) * DK + d);
                const double delta = dist64<DK>(q, kb) + ed;
                const double A = (1.0 / delta) * invZ;
                const double g = (dot - c) * invZ;
                const double inv_d2 = 1.0 / (delta * delta);
                const double w = 2.0 * g * inv_d2;
                if (lane == 0) {
#pragma unroll
                    for (int d = 0; d < DK; ++d) dq[d] -= w * ((double)q[d] - (double)kb[d]);
                    deps -= g * inv_d2;
                    a.muco[gq] = make_float2((float)A, (float)w);
                }
            } else if (lane == 0) {
                a.muco[gq] = make_float2(0.f, 0.f);
            }
        } else {
            for (int r = lane; r < k; r += 32) crow[r] = make_float2(0.f, 0.f);
            if (lane == 0) a.muco[gq] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int d = 0; d < DK; ++d) dq[d] = warp_sum(dq[d]);
        deps = warp_sum(deps);
        if (lane < DK) {
            double v = 0.0;
#pragma unroll
            for (int d = 0; d < DK; ++d) v = (lane == d) ? dq[d] : v;
            a.dQ[gq * DK + lane] = (float)v;
        }
        deps_w = deps;
    }
    if (lane == 0) s_eps[warp] = deps_w;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < BWD_WARPS; ++w) s += s_eps[w];
        a.eps_part[blockIdx.x] = s;
    }
}

struct KeyArgs {
    const float* Q; const float* K; const float* dO; const float2* coeff;
    const uint32_t* slots; const int32_t* offsets;
    float* dK; float* dV;
    int64_t N, L, total;
    int k, dv;
};

template <int DK>
__global__ void __launch_bounds__(BWD_THREADS) bwd_key_kernel(const KeyArgs a) {
    const int warp = threadIdx.x / 32, lane = lane_id();
    const int64_t gk = (int64_t)blockIdx.x * BWD_WARPS + warp;
    if (gk >= a.total) return;
    const int64_t N = a.N, bh = gk / N, j = gk % N;
    const int32_t* off = a.offsets + bh * (N + 1);
    const int32_t s0 = off[j], s1 = off[j + 1];
    const uint32_t* sl = a.slots + bh * a.L;
    const float2* cf = a.coeff + bh * a.L;
    const int dv = a.dv, k = a.k;
    const int nch = dv / 4;
    int P = 1;
    while (P < nch && P < 32) P <<= 1;
    const int G = 32 / P, grp = lane / P, ch_l = lane % P;
    float kj[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) kj[d] = __ldg(a.K + gk * DK + d);
    double dk[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) dk[d] = 0.0;
    const float* dOb = a.dO + bh * N * (int64_t)dv;
    const float* Qb = a.Q + bh * N * DK;
    float* dvrow = a.dV + gk * (int64_t)dv;
    for (int ch0 = 0; ch0 < nch; ch0 += P) {
        const int ch = ch0 + ch_l;
        const bool act = ch < nch;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        for (int32_t s = s0 + grp; s < s1; s += G) {
            const uint32_t slot = __ldg(sl + s);
            const int64_t iq = slot / (uint32_t)k;
            const float2 aw = __ldg(cf + slot);
            if (act) {
                const float4 g = __ldg(reinterpret_cast<const float4*>(dOb + iq * dv) + ch);
                const double A = (double)aw.x;
                acc0 = fma(A, (double)g.x, acc0);
                acc1 = fma(A, (double)g.y, acc1);
                acc2 = fma(A, (double)g.z, acc2);
                acc3 = fma(A, (double)g.w, acc3);
            }
            if (ch0 == 0 && ch_l == 0) {
#pragma unroll
                for (int d = 0; d < DK; ++d) dk[d] += (double)aw.y * ((double)__ldg(Qb + iq * DK + d) - (double)kj[d]);
            }
        }
        for (int o = P; o < 32; o <<= 1) {
            acc0 += __shfl_xor_sync(FULL, acc0, o);
            acc1 += __shfl_xor_sync(FULL, acc1, o);
            acc2 += __shfl_xor_sync(FULL, acc2, o);
            acc3 += __shfl_xor_sync(FULL, acc3, o);
        }
        if (grp == 0 && act)
            reinterpret_cast<float4*>(dvrow)[ch] = make_float4((float)acc0, (float)acc1, (float)acc2, (float)acc3);
    }
    // dK: group leaders (lanes 0, P, 2P, ...) hold partial sums over their slots
#pragma unroll
    for (int d = 0; d < DK; ++d)
        for (int o = P; o < 32; o <<= 1) dk[d] += __shfl_xor_sync(FULL, dk[d], o);
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < DK; ++d) a.dK[gk * DK + d] = (float)dk[d];
    }
}

__global__ void eps_reduce_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) acc += part[t];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

cudaError_t launch_bwd(const onedf_problem* p, const float* Q, const float* K, const float* V, const float* eps,
                       const float* O, const float* dO, const int32_t* idx, const float* Z, float* dQ, float* dK,
                       float* dV, double* d_eps, const MeanBufs* m, BwdBufs* b, TransposeBufs* t, void* ws,
                       cudaStream_t st, const Trace& tr) {
    const int64_t BH = p->B * p->H, N = p->N, total = BH * N;
    BwdArgs a;
    a.Q = Q; a.K = K; a.V = V; a.eps = eps; a.O = O; a.dO = dO; a.idx = idx; a.Z = Z;
    a.Kbar = m->Kbar; a.Vbar = m->Vbar; a.dQ = dQ; a.coeff = b->coeff; a.muco = b->muco; a.eps_part = b->eps_part;
    a.N = N; a.total = total; a.k = p->k; a.dv = p->d_v; a.causal = p->causal; a.mean_slot = p->mean_slot;
    a.ws = ws;
    ONEDF_DISPATCH_DK(p->d_k, { bwd_query_kernel<DK><<<(unsigned)b->eps_blocks, BWD_THREADS, 0, st>>>(a); });
    tr.mark(1, st);
    cudaError_t e = launch_transpose(p, idx, t, st);
    if (e != cudaSuccess) return e;
    tr.mark(2, st);
    KeyArgs ka;
    ka.Q = Q; ka.K = K; ka.dO = dO; ka.coeff = b->coeff; ka.slots = t->slots; ka.offsets = t->offsets;
    ka.dK = dK; ka.dV = dV; ka.N = N; ka.L = N * (int64_t)p->k; ka.total = total; ka.k = p->k; ka.dv = p->d_v;
    ONEDF_DISPATCH_DK(p->d_k, {
        bwd_key_kernel<DK><<<(unsigned)((total + BWD_WARPS - 1) / BWD_WARPS), BWD_THREADS, 0, st>>>(ka);
    });
    tr.mark(3, st);
    if (p->mean_slot) {
        e = launch_mean_grad_scan(p, Q, dO, reinterpret_cast<const float*>(b->muco), const_cast<MeanBufs*>(m), dK,
                                  dV, st);
        if (e != cudaSuccess) return e;
    }
    tr.mark(4, st);
    eps_reduce_kernel<<<1, 256, 0, st>>>(b->eps_part, b->eps_blocks, d_eps);
    tr.mark(5, st);
    return cudaGetLastError();
}

}  // namespace onedf
