// fwd.cu -- A5-A7: causal candidate search, exact top-k, Cauchy weights and
// the value gather, fused in one kernel (K6), plus the sorted-record build (K4).
//
// One warp owns one query i of one (b,h) ("performed in parallel for
// every query"); a CTA's 8 warps walk a contiguous stretch of the query
// SCHEDULE, which is the queries of each chunk sorted by Morton code (built by
// onedf's seg sort, K3).  Neighbouring warps therefore hold queries that are
// close in space: their windows into every run overlap and their neighbour
// sets share V rows, so the candidate records and gathered rows come from L1
// instead of L2 (L2 bandwidth, not HBM, is what bounds a gather on B200).
// The schedule only reorders work: every output row is computed by the same
// arithmetic whatever order it runs in, so results do not depend on it.
//
//  A5  lane c binary-searches run c (lower_bound on u64 codes, D3) for the
//      admissible runs c < floor(i/M) (D6) -- 32 runs per round, in parallel;
//      window w = min(W, len), s = clamp(p - W/2) (D1, D2).
//  A6  the warp streams every window as contiguous 16/32/48-B key records
//      (coords + original position, built by K4 in sorted order, so a window
//      is one coalesced burst) and ranks each candidate by the f32 distance in
//      the pinned order (D23) packed with its position into a u64 key
//      (D bits << 32 | j; D >= 0 so the bit pattern is order-preserving).
//      Two passes: (1) per-lane f32 min-lists of length 2*ceil(k/32) give a
//      bound T with #{D <= T} >= k (bisection over the union of the lists);
//      (2) every candidate with D <= T is appended to a per-warp shared-memory
//      buffer (integer cursor; ~1.4 k keys on average).  The collected keys
//      are unique, so their order is fixed by the keys alone: each 32-key row
//      is bitonic-sorted across the lanes with xor-shuffles, reversed,
//      min-merged into the register top list's last row (the lowest 32R of
//      both form a bitonic sequence) and a half-cleaner cascade restores
//      order.  If more than FWD_CAP keys tie at or below T, a streaming
//      selection with the same merges takes over.
//  A7  S = 1/(D + eps) in f64, mean slot from the prefix means (D8), Z by a
//      fixed-order warp tree, and o = sum A v + A_mu Vbar with f64
//      accumulators; V rows are gathered as float4 bursts (16 lanes per
//      64-float row), lane groups split the slots and are combined by a fixed
//      shuffle tree (deterministic).
#include "fwd_kernels.cuh"

namespace onedf {

void fwd_carve(const onedf_problem* p, Carver* c, FwdBufs* f) {
    const int64_t BH = p->B * p->H;
    const int rec = (p->d_k + 1 + 3) / 4 * 4;
    f->recs = c->take<float>((size_t)(BH * p->N * rec));
    f->qorder = c->take<int32_t>((size_t)(BH * p->N));
    sort_carve(p, c, &f->scr);

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

cudaError_t launch_fwd(const onedf_problem* p, const float* Q, const float* K, const void* V, const float* eps,
                       const uint64_t* qcode, const uint64_t* scode, const int32_t* perm, const int32_t* qorder,
                       void* O, int32_t* idx, float* Z, int32_t* indeg, const MeanBufs* m, FwdBufs* f, void* ws,
                       cudaStream_t st, const Trace& tr) {
    const int64_t BH = p->B * p->H, N = p->N, total = BH * N;
    ONEDF_DISPATCH_DK(p->d_k, {
        build_records_kernel<DK><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(K, perm, f->recs, N, total);
    });
    if (!qorder) {
        // no schedule from the caller: sort the query codes here (onedf_sort of qcode)
        const cudaError_t e = launch_query_order(p, qcode, f->qorder, f->scr, st);
        if (e != cudaSuccess) return e;
        qorder = f->qorder;
    }
    tr.mark(1, st);
    FwdArgs a;
    a.Q = Q; a.K = K; a.V = V; a.eps = eps; a.qcode = qcode; a.scode = scode; a.recs = f->recs;
    a.qorder = qorder;
    a.Kbar = m->Kbar; a.Vbar = m->Vbar; a.O = O; a.idx = idx; a.Z = Z;
    a.sh = make_shard(p);
    a.nq = a.sh.slots(N);
    a.N = N; a.M = p->causal ? p->chunk : N; a.total = BH * a.nq;
    a.k = p->k; a.W = effective_window(p); a.dv = p->d_v; a.causal = p->causal; a.mean_slot = p->mean_slot;
    a.score = p->score;
    a.indeg = indeg;
    if (indeg) {
        // A9's in-degree counts, accumulated by the top-k kernel (one integer RED per selected
        // slot) for the backward to reuse instead of re-reading idx
        const cudaError_t e = cudaMemsetAsync(indeg, 0, (size_t)(BH * N) * sizeof(int32_t), st);
        if (e != cudaSuccess) return e;
    }
    a.ws = ws;
    const int64_t per_cta = (int64_t)FWD_WARPS * FWD_QPW;
    const unsigned grid = (unsigned)((a.total + per_cta - 1) / per_cta);
    ONEDF_DISPATCH_TV(p->vdtype, {
        if (p->k <= 32) launch_fwd_tv<TV, 1>(a, p, grid, st);
        else if (p->k <= 64) launch_fwd_tv<TV, 2>(a, p, grid, st);
        else if (p->k <= 128) launch_fwd_tv<TV, 4>(a, p, grid, st);
        else launch_fwd_tv<TV, 8>(a, p, grid, st);
    });
    tr.mark(2, st);
    return cudaGetLastError();
}

}  // namespace onedf

