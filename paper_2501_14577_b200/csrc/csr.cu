// csr.cu -- A9 the backward transpose as a key-major CSR (K8).
//
// north_star: "a deterministic backward that scatter-adds dK/dV through
// sorted-index segment reduction rather than float atomics".  The key side
// (A10) needs, for every key j, the (query i, A_ij, w_ij) records of the
// queries that selected it, in a FIXED order.  Built in three steps:
//   (1) in-degree count: cnt[j] += 1 for every valid idx entry (integer
//       atomics: the counts, and everything derived from them, are exact and
//       order-free);
//   (2) exclusive scan per (b,h) -> CSR offsets off[j] (and the insertion
//       cursors, a copy of off);
//   (3) the query side (bwd.cu K7) appends each record at
//       atomicAdd(&cursor[j], 1) -- an integer slot, so only the ORDER inside
//       a segment depends on scheduling, never a value;
// and the key side (K9) visits each segment in ascending query position
// (the records' i are distinct within a segment -- a query selects a key at
// most once; segments <= 128 are ordered by a register bitonic sort of
// (i, position) keys, longer ones by rank counting into the `order` scratch).  Every f64 sum
// therefore runs in the same order as a stable sort of (j, slot) would give,
// independent of the atomic interleaving: bitwise reproducible.
#include "common.cuh"
#include "internal.h"

namespace onedf {

void csr_carve(const onedf_problem* p, Carver* c, CsrBufs* t) {
    const int64_t BH = p->B * p->H, N = p->N, L = N * (int64_t)p->k;
    t->cursor = c->take<int32_t>((size_t)(BH * N));
    t->offsets = c->take<int32_t>((size_t)(BH * (N + 1)));
    t->rec = c->take<int4>((size_t)(BH * L));
    t->order = c->take<int32_t>((size_t)(BH * L));
}

// (1) count.  A CTA takes CSR_QPC consecutive slots of the query schedule (the
// Morton order of K6/K7 when given): neighbouring queries select largely the
// same keys, so the CTA first aggregates its CSR_QPC*k entries in a shared-
// memory hash table (open addressing, integer atomics) and then adds each
// distinct key's count to global memory once -- several times fewer global
// atomics than one per entry.  All counts are integers: order-free.
constexpr int CSR_QPC = 32;                    // queries per CTA
constexpr int CSR_THREADS = 256;
constexpr int CSR_TBL = 4096;                  // hash slots (>= 2 x the entries of a CTA at k <= 64)

__global__ void __launch_bounds__(CSR_THREADS) csr_count_kernel(const int32_t* __restrict__ idx,
                                                                const int32_t* __restrict__ qorder, int64_t N,
                                                                int64_t nq, int k, Shard sh,
                                                                int32_t* __restrict__ cnt) {
    __shared__ uint32_t tkey[CSR_TBL];
    __shared__ uint32_t tcnt[CSR_TBL];
    const int64_t bh = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * CSR_QPC;          // schedule slot of the CTA's first query
    const bool hashed = (int64_t)CSR_QPC * k * 2 <= CSR_TBL;
    if (hashed) {
        for (int t = threadIdx.x; t < CSR_TBL; t += CSR_THREADS) { tkey[t] = 0u; tcnt[t] = 0u; }
        __syncthreads();
    }
    int32_t* c = cnt + bh * N;
    const int64_t total = (int64_t)CSR_QPC * k;
    for (int64_t x = threadIdx.x; x < total; x += CSR_THREADS) {
        const int64_t qs = q0 + x / k;
        if (qs >= nq) break;
        int64_t pos;
        if (!sh.slot_pos(qs, N, pos)) continue;
        const int64_t i = qorder ? (int64_t)__ldg(qorder + bh * N + pos) : pos;
        const int32_t j = __ldg(idx + (bh * N + i) * k + x % k);
        if (j < 0) continue;
        if (!hashed) { atomicAdd(c + j, 1); continue; }
        uint32_t h = ((uint32_t)j * 2654435761u) >> (32 - 12);   // CSR_TBL = 2^12
        const uint32_t key = (uint32_t)j + 1u;
        while (true) {
            const uint32_t old = atomicCAS(&tkey[h], 0u, key);
            if (old == 0u || old == key) { atomicAdd(&tcnt[h], 1u); break; }
            h = (h + 1) & (CSR_TBL - 1);
        }
    }
    if (!hashed) return;
    __syncthreads();
    for (int t = threadIdx.x; t < CSR_TBL; t += CSR_THREADS) {
        const uint32_t key = tkey[t];
        if (key) atomicAdd(c + (key - 1u), (int32_t)tcnt[t]);
    }
}

// (2) one CTA per (b,h): exclusive scan of cnt -> off[0..N] and cursor = off[0..N)
constexpr int CSR_SCAN_THREADS = 1024;
__global__ void __launch_bounds__(CSR_SCAN_THREADS) csr_scan_kernel(int32_t* __restrict__ cnt_cursor,
                                                                    int32_t* __restrict__ off, int64_t N) {
    __shared__ int32_t wsum[CSR_SCAN_THREADS / 32];
    const int64_t bh = blockIdx.x;
    int32_t* c = cnt_cursor + bh * N;
    int32_t* o = off + bh * (N + 1);
    const int64_t per = (N + CSR_SCAN_THREADS - 1) / CSR_SCAN_THREADS;
    const int64_t a0 = (int64_t)threadIdx.x * per, a1 = min64(N, a0 + per);
    int32_t sum = 0;
    for (int64_t t = a0; t < a1; ++t) sum += c[t];
    const int lane = lane_id(), w = threadIdx.x / 32;
    int32_t inc = sum;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, inc, s);
        if (lane >= s) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int32_t v = wsum[lane];
        int32_t x = v;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int32_t y = __shfl_up_sync(FULL, x, s);
            if (lane >= s) x += y;
        }
        wsum[lane] = x - v;
        if (lane == 31) o[N] = x;
    }
    __syncthreads();
    int32_t run = wsum[w] + inc - sum;
    for (int64_t t = a0; t < a1; ++t) {
        const int32_t x = c[t];
        o[t] = run;
        c[t] = run;                                               // insertion cursor
        run += x;
    }
}

cudaError_t launch_csr_count(const onedf_problem* p, const int32_t* idx, const int32_t* qorder, CsrBufs* t,
                             cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N;
    cudaError_t e = cudaMemsetAsync(t->cursor, 0, (size_t)(BH * N) * sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    const Shard sh = make_shard(p);
    const int64_t nq = sh.slots(N);
    if (nq > 0) {
        const dim3 grid((unsigned)((nq + CSR_QPC - 1) / CSR_QPC), (unsigned)BH);
        csr_count_kernel<<<grid, CSR_THREADS, 0, st>>>(idx, qorder, N, nq, p->k, sh, t->cursor);
    }
    csr_scan_kernel<<<(unsigned)BH, CSR_SCAN_THREADS, 0, st>>>(t->cursor, t->offsets, N);
    return cudaGetLastError();
}

}  // namespace onedf
