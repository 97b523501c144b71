// bwd.cu -- A8 backward query side (K7), A10 key side (K9), A12 eps reduce
// (K11).  The transpose (A9, K8: in-degree count + CSR offsets) is in csr.cu
// and the mean-slot chain rule (A11, K10) in mean.cu.
//
// Appendix, with "dL/do_i . (v_j - o_i)/Z_i" read as a d_v-wide
// dot product (D15) and I held fixed (D16):
//   c_i   = dO_i . o_i,     g_ij = (dO_i . v_j - c_i)/Z_i,   delta = D_ij + eps
//   A_ij  = (1/delta)/Z_i,  w_ij = 2 g_ij / delta^2
//   dq_i  = -sum_j w_ij (q_i - k_j)
//   deps  = -sum_ij g_ij / delta^2
//   dv_j  = sum_{i: j in I_i} A_ij dO_i
//   dk_j  = sum_{i: j in I_i} w_ij (q_i - k_j)
// plus the mean slot as one more slot (its A, w go to the A11 scan), and the
// score variants' weights and w (D24, slot_w).
//
// K7: one warp per query, queries visited in the Morton schedule (optional;
// see fwd.cu) so neighbouring warps gather overlapping V rows through L1.
// Phase 1: P lanes read one v_j row (P float4 chunks = one coalesced 256-B row
// at d_v = 64), each lane dots its chunk with its slice of dO_i (f64, exact
// f32 products); after T steps every lane holds T partial dots of T rows and a
// butterfly reduce-scatter (log2 P xor-shuffle levels, halving the live values
// each level) leaves each row's dot on one lane, which parks it in shared
// memory.  Phase 2, lane-parallel over the slots: Z_i and c_i = sum_j A_ij
// (dO_i.v_j) + A_imu dO_i.Vbar_i recomputed in f64 (reading R3), then g, A, w
// per slot, dq and deps in f64, and each (i, A, w) record appended to its
// key's CSR segment (integer cursor, csr.cu).
// K9: one warp per key j (keys visited in sorted-run order when perm is
// given) orders its CSR segment by query position (register bitonic sort of
// (i << 9 | position) keys up to KEY_REG_SEG = 512 entries; longer segments were ordered by
// csr.cu's bitmap counting sort after the query side), then
// walks it 32 entries at a time: lane groups of P gather the dO_i rows into
// f64 accumulators, a fixed shuffle tree at the end -- a deterministic
// segment reduction, no float atomics.  Every per-row result is independent
// of the visiting order and of the atomic interleaving.
#include "bwd_kernels.cuh"

namespace onedf {

void bwd_carve(const onedf_problem* p, Carver* c, BwdBufs* b) {
    const int64_t BH = p->B * p->H, total = BH * p->N;
    b->muco = c->take<float2>((size_t)total);
    b->eps_q = c->take<double>((size_t)total);
    b->eps_part = c->take<double>((size_t)EPS_PARTS);
    b->qorder = c->take<int32_t>((size_t)total);
    b->dV32 = p->vdtype == ONEDF_DTYPE_BF16 ? c->take<float>((size_t)(total * p->d_v)) : nullptr;
    sort_carve(p, c, &b->scr);
}

// A12: dε = Σ over all (b,h,i) of the per-query partials, in a fixed order:
// EPS_PARTS contiguous ranges summed by fixed block trees, then one block.
__global__ void __launch_bounds__(256) eps_partial_kernel(const double* __restrict__ eps_q, int64_t n,
                                                          double* __restrict__ part) {
    __shared__ double s[256];
    const int64_t per = (n + EPS_PARTS - 1) / EPS_PARTS;
    const int64_t a0 = (int64_t)blockIdx.x * per, a1 = min64(n, a0 + per);
    double acc = 0.0;
    for (int64_t t = a0 + threadIdx.x; t < a1; t += 256) acc += eps_q[t];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void __launch_bounds__(256) eps_final_kernel(const double* __restrict__ part, double* __restrict__ out) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int t = threadIdx.x; t < EPS_PARTS; t += 256) acc += part[t];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

static int lanes_per_row(int dv) {
    const int nch = dv / 4;
    int P = 4;
    while (P < nch && P < 32) P <<= 1;
    return P;
}

cudaError_t launch_bwd(const onedf_problem* p, const float* Q, const float* K, const void* V, const float* eps,
                       const void* dO, const int32_t* idx, const uint64_t* qcode, const int32_t* qorder,
                       const int32_t* perm, const int32_t* indeg, float* dQ, float* dK, void* dV, double* d_eps,
                       const MeanBufs* m, BwdBufs* b, CsrBufs* t, void* ws, cudaStream_t st, const Trace& tr) {
    const int64_t BH = p->B * p->H, N = p->N, total = BH * N;
    cudaError_t e = cudaSuccess;
    if (!qorder && qcode) {
        // schedule hint given as codes only: sort them here (the forward's qorder saves this)
        e = launch_query_order(p, qcode, b->qorder, b->scr, st);
        if (e != cudaSuccess) return e;
        qorder = b->qorder;
    }
    // A9 first: in-degree counts -> CSR offsets + insertion cursors (the query side appends into them)
    e = launch_csr_count(p, idx, qorder, indeg, t, st);
    if (e != cudaSuccess) return e;
    tr.mark(1, st);
    BwdArgs a;
    a.Q = Q; a.K = K; a.V = V; a.eps = eps; a.dO = dO; a.idx = idx;
    a.Kbar = m->Kbar; a.Vbar = m->Vbar; a.qorder = qorder;
    a.dQ = dQ; a.muco = b->muco; a.eps_q = b->eps_q;
    a.cursor = t->cursor; a.rec_i = t->rec_i; a.rec_aw = t->rec_aw; a.L = N * (int64_t)p->k;
    a.sh = make_shard(p);
    a.nq = a.sh.slots(N);
    a.N = N; a.total = BH * a.nq; a.k = p->k; a.dv = p->d_v; a.causal = p->causal; a.mean_slot = p->mean_slot;
    a.score = p->score;
    a.ws = ws;
    if (a.sh.on()) {
        // rows of queries this rank does not own stay zero: they enter the A11 scan and the eps sum
        e = cudaMemsetAsync(b->muco, 0, (size_t)total * sizeof(float2), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(b->eps_q, 0, (size_t)total * sizeof(double), st);
        if (e != cudaSuccess) return e;
    }
    const int P = lanes_per_row(p->d_v);
    const int nch = p->d_v / 4;
    const unsigned qgrid = (unsigned)((a.total + BWD_WARPS - 1) / BWD_WARPS);
    const unsigned kgrid = (unsigned)((total + BWD_WARPS - 1) / BWD_WARPS);
    ONEDF_DISPATCH_TV(p->vdtype, {
        ONEDF_DISPATCH_DK(p->d_k, { launch_bwd_query_dk<DK, TV>(a, P, nch, p->d_v, p->k, qgrid, st); });
    });
    tr.mark(2, st);
    // the ascending-i order of the long segments (hub keys), now that every record is in place
    e = launch_csr_long_order(p, t, st);
    if (e != cudaSuccess) return e;
    KeyArgs ka;
    ka.Q = Q; ka.K = K; ka.dO = dO; ka.offsets = t->offsets; ka.rec_i = t->rec_i; ka.rec_aw = t->rec_aw;
    ka.order = t->order;
    ka.korder = perm;
    // the key side's dV in f32: the output itself (float rows) or the f32 scratch of a BF16 problem
    float* dV32 = p->vdtype == ONEDF_DTYPE_BF16 ? b->dV32 : static_cast<float*>(dV);
    ka.dK = dK; ka.dV = dV32; ka.N = N; ka.L = N * (int64_t)p->k; ka.total = total; ka.k = p->k; ka.dv = p->d_v;
    ka.kt = p->score == SC_DOT ? 0.0 : 1.0;
    ONEDF_DISPATCH_TV(p->vdtype, {
        ONEDF_DISPATCH_DK(p->d_k, { launch_bwd_key_dk<DK, TV>(ka, P, p->d_v, kgrid, st); });
    });
    tr.mark(3, st);
    if (p->mean_slot) {
        e = launch_mean_grad_scan(p, Q, dO, reinterpret_cast<const float*>(b->muco), const_cast<MeanBufs*>(m), dK,
                                  dV32, dV, st);
        if (e != cudaSuccess) return e;
    } else if (p->vdtype == ONEDF_DTYPE_BF16) {
        e = launch_round_rows(dV32, static_cast<bf16*>(dV), total * p->d_v, st);
        if (e != cudaSuccess) return e;
    }
    tr.mark(4, st);
    eps_partial_kernel<<<EPS_PARTS, 256, 0, st>>>(b->eps_q, total, b->eps_part);
    eps_final_kernel<<<1, 256, 0, st>>>(b->eps_part, d_eps);
    tr.mark(5, st);
    return cudaGetLastError();
}

}  // namespace onedf
