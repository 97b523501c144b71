// fwd.cu -- A5-A7: causal candidate search, exact top-k, Cauchy weights and
// the value gather, fused in one kernel (K6), plus the sorted-record build (K4).
//
// One warp owns one query i of one (b,h) ("performed in parallel for
// every query"):
//  A5  lane c binary-searches run c (lower_bound on u64 codes, D3) for the
//      admissible runs c < floor(i/M) (D6) -- 32 runs per round, in parallel;
//      window w = min(W, len), s = clamp(p - W/2) (D1, D2).
//  A6  the warp streams every window as contiguous 16/32/48-B key records
//      (coords + original position, built by K4 in sorted order, so a window
//      is one coalesced burst), ranks each candidate by the f32 distance in
//      the pinned order (D23) packed with its position into a u64 key
//      (D bits << 32 | j; D >= 0 so the bit pattern is order-preserving), and
//      keeps the exact top-k: keys below the running k-th key are appended
//      (ballot + popc compaction) to a per-warp pending buffer in shared
//      memory; a full buffer is bitonic-sorted and merged into the sorted
//      top buffer (min(top[t], pend[K-1-t]) + half-cleaners), which then
//      lowers the admission threshold.
//  A7  S = 1/(D + eps) in f64, mean slot from the prefix means (D8), Z by a
//      fixed-order warp tree, and o = sum A v + A_mu Vbar with f64
//      accumulators; V rows are gathered as float4 bursts, lane groups split
//      the slots and are combined by a fixed shuffle tree (deterministic).
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int FWD_WARPS = 8;
constexpr int FWD_THREADS = FWD_WARPS * 32;
constexpr unsigned long long KEY_MAX = ~0ull;

void fwd_carve(const onedf_problem* p, Carver* c, FwdBufs* f) {
    const int64_t BH = p->B * p->H;
    const int rec = (p->d_k + 1 + 3) / 4 * 4;
    f->recs = c->take<float>((size_t)(BH * p->N * rec));
}

// ------------------------------------------------------------------ K4
template <int DK>
__global__ void build_records_kernel(const float* __restrict__ K, const int32_t* __restrict__ perm,
                                     float* __restrict__ recs, int64_t N, int64_t total) {
    constexpr int REC = RecW<DK>::value;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int64_t bh = t / N;
    const int32_t j = perm[t];
    float r[REC];
#pragma unroll
    for (int d = 0; d < REC; ++d) r[d] = 0.f;
#pragma unroll
    for (int d = 0; d < DK; ++d) r[d] = K[(bh * N + j) * DK + d];
    r[DK] = __int_as_float(j);
    float4* dst = reinterpret_cast<float4*>(recs + t * REC);
#pragma unroll
    for (int v = 0; v < REC / 4; ++v) dst[v] = make_float4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
}

// ------------------------------------------------------------------ warp top-k buffers
// Bitonic sort of buf[0..KC) ascending by one warp.
template <int KC>
__device__ __forceinline__ void warp_bitonic_sort(unsigned long long* buf) {
#pragma unroll
    for (int size = 2; size <= KC; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
            for (int t = lane_id(); t < KC / 2; t += 32) {
                const int i1 = 2 * stride * (t / stride) + (t % stride);
                const int i2 = i1 + stride;
                const unsigned long long a = buf[i1], b = buf[i2];
                const bool up = (i1 & size) == 0;
                if ((a > b) == up) { buf[i1] = b; buf[i2] = a; }
            }
            __syncwarp();
        }
    }
}

// Half-cleaner cascade: sorts a bitonic buf[0..KC) ascending.
template <int KC>
__device__ __forceinline__ void warp_bitonic_clean(unsigned long long* buf) {
#pragma unroll
    for (int stride = KC >> 1; stride > 0; stride >>= 1) {
#pragma unroll
        for (int t = lane_id(); t < KC / 2; t += 32) {
            const int i1 = 2 * stride * (t / stride) + (t % stride);
            const int i2 = i1 + stride;
            const unsigned long long a = buf[i1], b = buf[i2];
            if (a > b) { buf[i1] = b; buf[i2] = a; }
        }
        __syncwarp();
    }
}

// Merge pend[0..cnt) into the sorted top[0..KC); returns the new threshold top[k-1].
template <int KC>
__device__ __forceinline__ unsigned long long flush_pending(unsigned long long* top, unsigned long long* pend,
                                                            int cnt, int k) {
    for (int t = cnt + lane_id(); t < KC; t += 32) pend[t] = KEY_MAX;
    __syncwarp();
    warp_bitonic_sort<KC>(pend);
    for (int t = lane_id(); t < KC; t += 32) {
        const unsigned long long a = top[t], b = pend[KC - 1 - t];
        top[t] = a < b ? a : b;
    }
    __syncwarp();
    warp_bitonic_clean<KC>(top);
    return top[k - 1];
}

struct FwdArgs {
    const float* Q; const float* K; const float* V; const float* eps;
    const uint64_t* qcode; const uint64_t* scode; const float* recs;
    const float* Kbar; const float* Vbar;
    float* O; int32_t* idx; float* Z;
    int64_t N, M, total;
    int k, W, dv, causal, mean_slot;
    void* ws;
};

template <int DK, int KC>
__global__ void __launch_bounds__(FWD_THREADS) topk_attn_fwd_kernel(const FwdArgs a) {
    constexpr int REC = RecW<DK>::value;
    __shared__ __align__(16) unsigned long long s_top[FWD_WARPS][KC];
    __shared__ __align__(16) unsigned long long s_pend[FWD_WARPS][KC];
    const int warp = threadIdx.x / 32, lane = lane_id();
    const int64_t gq = (int64_t)blockIdx.x * FWD_WARPS + warp;
    if (gq >= a.total) return;
    const int64_t N = a.N, bh = gq / N, i = gq % N;
    unsigned long long* top = s_top[warp];
    unsigned long long* pend = s_pend[warp];
    const float e = __ldg(a.eps);
    if (gq == 0 && lane == 0 && !(e > 0.f && isfinite(e))) set_flag(a.ws, FLAG_BAD_EPS);

    float q[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) q[d] = __ldg(a.Q + gq * DK + d);
    const uint64_t qc = __ldg(a.qcode + gq);
    for (int t = lane; t < KC; t += 32) top[t] = KEY_MAX;
    __syncwarp();

    // ---------------- A5 + A6: candidate search and exact top-k
    const int64_t nruns = a.causal ? i / a.M : 1;
    const uint64_t* scode = a.scode + bh * N;
    const float* recs = a.recs + bh * N * REC;
    unsigned long long thresh = KEY_MAX;
    int cnt = 0;
    for (int64_t c0 = 0; c0 < nruns; c0 += 32) {
        const int64_t c = c0 + lane;
        int64_t base = 0;
        int w = 0;
        if (c < nruns) {
            const int64_t s0 = a.causal ? c * a.M : 0;
            const int64_t len = a.causal ? min64(a.M, N - s0) : N;
            int64_t lo = 0, hi = len;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (__ldg(scode + s0 + mid) < qc) lo = mid + 1; else hi = mid;
            }
            const int64_t ww = min64(a.W, len);
            int64_t s = lo - a.W / 2;
            s = s < 0 ? 0 : s;
            s = s > len - ww ? len - ww : s;
            base = s0 + s;
            w = (int)ww;
        }
        const int nc = (int)min64(32, nruns - c0);
        for (int cc = 0; cc < nc; ++cc) {
            const int64_t b = __shfl_sync(FULL, base, cc);
            const int ww = __shfl_sync(FULL, w, cc);
            for (int r0 = 0; r0 < ww; r0 += 32) {
                const int r = r0 + lane;
                const bool act = r < ww;
                unsigned long long key = KEY_MAX;
                if (act) {
                    const float4* rp = reinterpret_cast<const float4*>(recs + (b + r) * REC);
                    float rv[REC];
#pragma unroll
                    for (int v = 0; v < REC / 4; ++v) {
                        const float4 t4 = __ldg(rp + v);
                        rv[4 * v] = t4.x; rv[4 * v + 1] = t4.y; rv[4 * v + 2] = t4.z; rv[4 * v + 3] = t4.w;
                    }
                    const float D = rank_dist32<DK>(q, rv);
                    key = ((unsigned long long)__float_as_uint(D) << 32) | (unsigned)__float_as_int(rv[DK]);
                }
                bool pass = act && key < thresh;
                unsigned m = __ballot_sync(FULL, pass);
                int n = __popc(m);
                if (cnt + n > KC) {
                    thresh = flush_pending<KC>(top, pend, cnt, a.k);
                    cnt = 0;
                    pass = act && key < thresh;
                    m = __ballot_sync(FULL, pass);
                    n = __popc(m);
                }
                if (pass) pend[cnt + __popc(m & lanemask_lt())] = key;
                cnt += n;
                __syncwarp();
            }
        }
    }
    if (cnt > 0) flush_pending<KC>(top, pend, cnt, a.k);

    // ---------------- outputs: idx row
    const int k = a.k;
    int32_t* idx_row = a.idx + gq * k;
    int nsel = 0;
    for (int r = lane; r < k; r += 32) {
        const unsigned long long key = top[r];
        idx_row[r] = key == KEY_MAX ? -1 : (int32_t)(unsigned)(key & 0xffffffffull);
    }
    {
        // number of valid slots: top is ascending with KEY_MAX padding at the end
        unsigned vm = 0;
        for (int r0 = 0; r0 < k; r0 += 32) {
            const int r = r0 + lane;
            vm = __ballot_sync(FULL, r < k && top[r] != KEY_MAX);
            nsel += __popc(vm);
        }
    }

    // ---------------- A7: Cauchy weights (f64)
    double* Sbuf = reinterpret_cast<double*>(pend);   // reuse: KC doubles
    const double ed = (double)e;
    double zpart = 0.0;
    for (int r = lane; r < nsel; r += 32) {
        const int j = (int)(unsigned)(top[r] & 0xffffffffull);
        float kj[DK];
#pragma unroll
        for (int d = 0; d < DK; ++d) kj[d] = __ldg(a.K + (bh * N + j) * DK + d);
        const double S = 1.0 / (dist64<DK>(q, kj) + ed);
        Sbuf[r] = S;
        zpart += S;
    }
    double Zi = warp_sum(zpart);
    double Smu = 0.0;
    const int64_t mrow = a.causal ? i : 0;
    if (a.mean_slot) {
        float kb[DK];
#pragma unroll
        for (int d = 0; d < DK; ++d) kb[d] = __ldg(a.Kbar + (bh * (a.causal ? N : 1) + mrow) * DK + d);
        Smu = 1.0 / (dist64<DK>(q, kb) + ed);
        Zi += Smu;
    }
    __syncwarp();
    const double invZ = Zi > 0.0 ? 1.0 / Zi : 0.0;

    // ---------------- A7: value gather, float4 chunks, lane groups over slots
    const int nch = a.dv / 4;
    int P = 1;
    while (P < nch && P < 32) P <<= 1;
    const int G = 32 / P;                 // groups (1 when nch >= 32)
    const int grp = lane / P, ch_l = lane % P;
    const float* Vb = a.V + bh * N * (int64_t)a.dv;
    float* orow = a.O + gq * (int64_t)a.dv;
    const float* vbar = a.Vbar + (bh * (a.causal ? N : 1) + mrow) * (int64_t)a.dv;
    const double Amu = Smu * invZ;
    for (int ch0 = 0; ch0 < nch; ch0 += P) {
        const int ch = ch0 + ch_l;
        const bool act = ch < nch;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        for (int r = grp; r < nsel; r += G) {
            const int j = (int)(unsigned)(top[r] & 0xffffffffull);
            const double A = Sbuf[r] * invZ;
            if (act) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(Vb + (int64_t)j * a.dv) + ch);
                acc0 = fma(A, (double)v.x, acc0);
                acc1 = fma(A, (double)v.y, acc1);
                acc2 = fma(A, (double)v.z, acc2);
                acc3 = fma(A, (double)v.w, acc3);
            }
        }
        for (int o = P; o < 32; o <<= 1) {
            acc0 += __shfl_xor_sync(FULL, acc0, o);
            acc1 += __shfl_xor_sync(FULL, acc1, o);
            acc2 += __shfl_xor_sync(FULL, acc2, o);
            acc3 += __shfl_xor_sync(FULL, acc3, o);
        }
        if (grp == 0 && act) {
            if (a.mean_slot) {
                const float4 vb = __ldg(reinterpret_cast<const float4*>(vbar) + ch);
                acc0 = fma(Amu, (double)vb.x, acc0);
                acc1 = fma(Amu, (double)vb.y, acc1);
                acc2 = fma(Amu, (double)vb.z, acc2);
                acc3 = fma(Amu, (double)vb.w, acc3);
            }
            reinterpret_cast<float4*>(orow)[ch] = make_float4((float)acc0, (float)acc1, (float)acc2, (float)acc3);
        }
    }
    if (lane == 0) a.Z[gq] = (float)Zi;
}

cudaError_t launch_fwd(const onedf_problem* p, const float* Q, const float* K, const float* V, const float* eps,
                       const uint64_t* qcode, const uint64_t* scode, const int32_t* perm, float* O, int32_t* idx,
                       float* Z, const MeanBufs* m, FwdBufs* f, void* ws, cudaStream_t st, const Trace& tr) {
    const int64_t BH = p->B * p->H, N = p->N, total = BH * N;
    ONEDF_DISPATCH_DK(p->d_k, {
        build_records_kernel<DK><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(K, perm, f->recs, N, total);
    });
    tr.mark(1, st);
    FwdArgs a;
    a.Q = Q; a.K = K; a.V = V; a.eps = eps; a.qcode = qcode; a.scode = scode; a.recs = f->recs;
    a.Kbar = m->Kbar; a.Vbar = m->Vbar; a.O = O; a.idx = idx; a.Z = Z;
    a.N = N; a.M = p->causal ? p->chunk : N; a.total = total;
    a.k = p->k; a.W = effective_window(p); a.dv = p->d_v; a.causal = p->causal; a.mean_slot = p->mean_slot;
    a.ws = ws;
    const unsigned grid = (unsigned)((total + FWD_WARPS - 1) / FWD_WARPS);
#define ONEDF_FWD_KC(KCV)                                                        \
    ONEDF_DISPATCH_DK(p->d_k, { topk_attn_fwd_kernel<DK, KCV><<<grid, FWD_THREADS, 0, st>>>(a); })
    if (p->k <= 32) { ONEDF_FWD_KC(32) }
    else if (p->k <= 64) { ONEDF_FWD_KC(64) }
    else if (p->k <= 128) { ONEDF_FWD_KC(128) }
    else { ONEDF_FWD_KC(256) }
#undef ONEDF_FWD_KC
    tr.mark(2, st);
    return cudaGetLastError();
}

}  // namespace onedf
