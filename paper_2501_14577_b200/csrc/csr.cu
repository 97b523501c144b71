// csr.cu -- A9 the backward transpose as a key-major CSR (K8).
//
// north_star: "a deterministic backward that scatter-adds dK/dV through
// sorted-index segment reduction rather than float atomics".  The key side
// (A10) needs, for every key j, the (query i, A_ij, w_ij) records of the
// queries that selected it, in a FIXED order.  Built in three steps:
//   (1) in-degree count: cnt[j] += 1 for every valid idx entry (integer
//       atomics: the counts, and everything derived from them, are exact and
//       order-free) -- done by the forward's top-k kernel (one RED per selected
//       slot into the caller's indeg, copied here) or, without it, by the
//       counting pass over idx below;
//   (2) exclusive scan per (b,h) -> CSR offsets off[j] (and the insertion
//       cursors, a copy of off), multi-CTA;
//   (3) the query side (bwd.cu K7) appends each record at
//       atomicAdd(&cursor[j], 1) -- an integer slot, so only the ORDER inside
//       a segment depends on scheduling, never a value;
// and the key side (K9) visits each segment in ascending query position
// (the records' i are distinct within a segment -- a query selects a key at
// most once; segments <= KEY_REG_SEG (512) are ordered by the key side's register bitonic
// sort of (i, position) keys, longer ones by (4) below, a counting sort over a
// bitmap of query positions into the `order` scratch).  Records are stored as
// structure-of-arrays, i (4 B) and (A, w) (8 B): the ordering reads only i.  Every f64 sum
// therefore runs in the same order as a stable sort of (j, slot) would give,
// independent of the atomic interleaving: bitwise reproducible.
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int CSR_SCAN_THREADS = 256;
constexpr int CSR_SB = CSR_SCAN_THREADS * 16;          // counts per block of the offset scan (2)

void csr_carve(const onedf_problem* p, Carver* c, CsrBufs* t) {
    const int64_t BH = p->B * p->H, N = p->N, L = N * (int64_t)p->k;
    t->cursor = c->take<int32_t>((size_t)(BH * N));
    t->offsets = c->take<int32_t>((size_t)(BH * (N + 1)));
    t->rec_i = c->take<int32_t>((size_t)(BH * L));
    t->rec_aw = c->take<float2>((size_t)(BH * L));
    t->order = c->take<int32_t>((size_t)(BH * L));
    t->nlong = c->take<int32_t>(1);
    t->longseg = c->take<int2>((size_t)(BH * N));
    t->bsum = c->take<int32_t>((size_t)(BH * ((N + CSR_SB - 1) / CSR_SB + 1)));
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
#ifndef ONEDF_CSR_HASH
#define ONEDF_CSR_HASH 1
#endif
    const bool hashed = ONEDF_CSR_HASH && (int64_t)CSR_QPC * k * 2 <= CSR_TBL;
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

// (2) exclusive scan of cnt -> off[0..N] and cursor = off[0..N) per (b,h), in three launches so a
// long sequence is scanned by many CTAs: block sums of CSR_SB counts, a scan of the block sums per
// (b,h), and the apply pass (integer arithmetic: exact whatever the order).  Every long segment
// (csr_long_segment) is appended to the long-segment list.
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* s_w, int32_t& total) {
    const int lane = lane_id(), w = threadIdx.x / 32, nw = blockDim.x / 32;
    int32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    int32_t woff = 0, tot = 0;
    for (int x = 0; x < nw; ++x) {
        woff += x < w ? s_w[x] : 0;
        tot += s_w[x];
    }
    __syncthreads();
    total = tot;
    return woff + inc - v;
}

__global__ void __launch_bounds__(CSR_SCAN_THREADS) csr_blocksum_kernel(const int32_t* __restrict__ cnt, int64_t N,
                                                                        int32_t* __restrict__ bsum, int64_t nblk) {
    __shared__ int32_t s_w[CSR_SCAN_THREADS / 32];
    const int64_t bh = blockIdx.y, b0 = (int64_t)blockIdx.x * CSR_SB;
    int32_t sum = 0;
    for (int64_t t = b0 + threadIdx.x; t < min64(N, b0 + CSR_SB); t += CSR_SCAN_THREADS) sum += cnt[bh * N + t];
    int32_t total;
    block_excl_scan(sum, s_w, total);
    if (threadIdx.x == 0) bsum[bh * (nblk + 1) + blockIdx.x] = total;
}

__global__ void __launch_bounds__(CSR_SCAN_THREADS) csr_blockscan_kernel(int32_t* __restrict__ bsum, int64_t nblk,
                                                                         int32_t* __restrict__ off, int64_t N) {
    __shared__ int32_t s_w[CSR_SCAN_THREADS / 32];
    const int64_t bh = blockIdx.x;
    int32_t* b = bsum + bh * (nblk + 1);
    const int64_t per = (nblk + CSR_SCAN_THREADS - 1) / CSR_SCAN_THREADS;
    const int64_t u0 = min64(nblk, (int64_t)threadIdx.x * per), u1 = min64(nblk, u0 + per);
    int32_t sum = 0;
    for (int64_t u = u0; u < u1; ++u) sum += b[u];
    int32_t total;
    int32_t run = block_excl_scan(sum, s_w, total);
    for (int64_t u = u0; u < u1; ++u) { const int32_t x = b[u]; b[u] = run; run += x; }
    if (threadIdx.x == 0) off[bh * (N + 1) + N] = total;
}

__global__ void __launch_bounds__(CSR_SCAN_THREADS) csr_apply_kernel(int32_t* __restrict__ cnt_cursor,
                                                                     int32_t* __restrict__ off, int64_t N,
                                                                     const int32_t* __restrict__ bsum, int64_t nblk,
                                                                     int32_t* __restrict__ nlong,
                                                                     int2* __restrict__ longseg) {
    __shared__ int32_t s_w[CSR_SCAN_THREADS / 32];
    const int64_t bh = blockIdx.y, b0 = (int64_t)blockIdx.x * CSR_SB;
    int32_t* c = cnt_cursor + bh * N;
    int32_t* o = off + bh * (N + 1);
    constexpr int PER = CSR_SB / CSR_SCAN_THREADS;       // contiguous counts per thread
    const int64_t a0 = b0 + (int64_t)threadIdx.x * PER, a1 = min64(N, a0 + PER);
    int32_t v[PER];
    int32_t sum = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        v[u] = a0 + u < a1 ? c[a0 + u] : 0;
        sum += v[u];
    }
    int32_t total;
    int32_t run = bsum[bh * (nblk + 1) + blockIdx.x] + block_excl_scan(sum, s_w, total);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        if (a0 + u >= a1) break;
        o[a0 + u] = run;
        c[a0 + u] = run;                                           // insertion cursor
        if (v[u] > 0 && csr_long_segment(v[u], N)) longseg[atomicAdd(nlong, 1)] = make_int2((int)bh, (int)(a0 + u));
        run += v[u];
    }
}

// (4) after the query side: the ascending-i order of every long segment (hub keys of repeated-token
// inputs, thousands of records), as a counting sort over a bitmap of query positions: set bit i of
// every record, prefix-count the bits, and the rank of record e is the number of set bits below its
// i (the i of a segment are distinct: a query selects a key at most once).  O(len + N/32) per
// segment instead of ranking by comparisons.  One CTA per segment, CTAs loop over the list.
// Shared memory: the bitmap (N/32 words), per-word bit offsets within their 1024-bit block (u16),
// and per-block offsets.
constexpr int CSR_LONG_THREADS = 512;

__global__ void __launch_bounds__(CSR_LONG_THREADS) csr_long_order_kernel(const int32_t* __restrict__ nlong,
                                                                          const int2* __restrict__ longseg,
                                                                          const int32_t* __restrict__ offsets,
                                                                          const int32_t* __restrict__ rec_i,
                                                                          int32_t* __restrict__ order, int64_t N,
                                                                          int64_t L) {
    extern __shared__ uint32_t sm[];
    const int64_t nw = (N + 31) / 32, nb = (nw + 31) / 32;          // bitmap words, 1024-bit blocks
    uint32_t* bits = sm;
    int32_t* boff = reinterpret_cast<int32_t*>(sm + nw);              // [nb + 1]
    uint16_t* woff = reinterpret_cast<uint16_t*>(boff + nb + 1);      // [nw]
    __shared__ int32_t s_w[CSR_LONG_THREADS / 32];
    const int n = *nlong;
    for (int s = blockIdx.x; s < n; s += gridDim.x) {
        const int2 sj = longseg[s];
        const int64_t bh = sj.x, j = sj.y;
        const int32_t s0 = offsets[bh * (N + 1) + j], s1 = offsets[bh * (N + 1) + j + 1];
        const int32_t* ri = rec_i + bh * L;
        for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0u;
        __syncthreads();
        for (int32_t e = s0 + threadIdx.x; e < s1; e += blockDim.x) {
            const int32_t i = ri[e];
            atomicOr(&bits[i >> 5], 1u << (i & 31));
        }
        __syncthreads();
        // per-block popcounts -> exclusive offsets (one warp per block, then a block scan)
        const int lane = lane_id(), wid = threadIdx.x / 32, nwarps = blockDim.x / 32;
        for (int64_t b = wid; b < nb; b += nwarps) {
            const int64_t w = b * 32 + lane;
            const int c = w < nw ? __popc(bits[w]) : 0;
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += y;
            }
            if (w < nw) woff[w] = (uint16_t)(inc - c);
            if (lane == 31) boff[b] = inc;
        }
        __syncthreads();
        // exclusive scan of the nb block counts (sequential per thread chunk + warp scan of chunk sums)
        {
            const int64_t per = (nb + blockDim.x - 1) / blockDim.x;
            const int64_t b0 = threadIdx.x * per, b1 = min64(nb, b0 + per);
            int32_t sum = 0;
            for (int64_t b = b0; b < b1; ++b) sum += boff[b];
            int32_t inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s_w[wid] = inc;
            __syncthreads();
            if (wid == 0) {
                const int32_t v = lane < nwarps ? s_w[lane] : 0;
                int32_t x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                if (lane < nwarps) s_w[lane] = x - v;
            }
            __syncthreads();
            int32_t run = s_w[wid] + inc - sum;
            for (int64_t b = b0; b < b1; ++b) {
                const int32_t x = boff[b];
                boff[b] = run;
                run += x;
            }
        }
        __syncthreads();
        int32_t* go = order + bh * L + s0;
        for (int32_t e = s0 + threadIdx.x; e < s1; e += blockDim.x) {
            const int32_t i = ri[e];
            const int32_t w = i >> 5;
            const int32_t rank = boff[w >> 5] + woff[w] + __popc(bits[w] & ((1u << (i & 31)) - 1u));
            go[rank] = e - s0;
        }
        __syncthreads();
    }
}

// The same order by comparison counting (O(len^2) global loads): only for N too large for the
// shared-memory bitmap (N > ~1M positions per (b,h)).
__global__ void __launch_bounds__(CSR_LONG_THREADS) csr_long_rank_kernel(const int32_t* __restrict__ nlong,
                                                                         const int2* __restrict__ longseg,
                                                                         const int32_t* __restrict__ offsets,
                                                                         const int32_t* __restrict__ rec_i,
                                                                         int32_t* __restrict__ order, int64_t N,
                                                                         int64_t L) {
    const int n = *nlong;
    for (int s = blockIdx.x; s < n; s += gridDim.x) {
        const int2 sj = longseg[s];
        const int64_t bh = sj.x, j = sj.y;
        const int32_t s0 = offsets[bh * (N + 1) + j], s1 = offsets[bh * (N + 1) + j + 1];
        const int32_t* ri = rec_i + bh * L + s0;
        int32_t* go = order + bh * L + s0;
        for (int32_t e = threadIdx.x; e < s1 - s0; e += blockDim.x) {
            const int32_t mine = ri[e];
            int32_t rank = 0;
            for (int32_t x = 0; x < s1 - s0; ++x) rank += ri[x] < mine;
            go[rank] = e;
        }
    }
}

static size_t long_order_smem(int64_t N) {
    const int64_t nw = (N + 31) / 32, nb = (nw + 31) / 32;
    return (size_t)(nw * 4 + (nb + 1) * 4 + nw * 2 + 16);
}

// largest N whose bitmap fits in shared memory (N = 1M needs 192 KB)
constexpr size_t LONG_ORDER_SMEM_MAX = 200 * 1024;

cudaError_t launch_csr_long_order(const onedf_problem* p, CsrBufs* t, cudaStream_t st) {
    const size_t smem = long_order_smem(p->N);
    const int64_t L = p->N * (int64_t)p->k;
    if (smem > LONG_ORDER_SMEM_MAX) {
        csr_long_rank_kernel<<<2 * 148, CSR_LONG_THREADS, 0, st>>>(t->nlong, t->longseg, t->offsets, t->rec_i,
                                                                   t->order, p->N, L);
        return cudaGetLastError();
    }
    if (smem > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(csr_long_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    // a persistent grid: the number of long segments is only known on the device
    csr_long_order_kernel<<<2 * 148, CSR_LONG_THREADS, smem, st>>>(t->nlong, t->longseg, t->offsets, t->rec_i,
                                                                   t->order, p->N, L);
    return cudaGetLastError();
}

cudaError_t launch_csr_count(const onedf_problem* p, const int32_t* idx, const int32_t* qorder,
                             const int32_t* indeg, CsrBufs* t, cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N;
    cudaError_t e = indeg ? cudaMemcpyAsync(t->cursor, indeg, (size_t)(BH * N) * sizeof(int32_t),
                                            cudaMemcpyDeviceToDevice, st)
                          : cudaMemsetAsync(t->cursor, 0, (size_t)(BH * N) * sizeof(int32_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(t->nlong, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    const Shard sh = make_shard(p);
    const int64_t nq = sh.slots(N);
    if (nq > 0 && !indeg) {
        const dim3 grid((unsigned)((nq + CSR_QPC - 1) / CSR_QPC), (unsigned)BH);
        csr_count_kernel<<<grid, CSR_THREADS, 0, st>>>(idx, qorder, N, nq, p->k, sh, t->cursor);
    }
    const int64_t nblk = (N + CSR_SB - 1) / CSR_SB;
    const dim3 gb((unsigned)nblk, (unsigned)BH);
    csr_blocksum_kernel<<<gb, CSR_SCAN_THREADS, 0, st>>>(t->cursor, N, t->bsum, nblk);
    csr_blockscan_kernel<<<(unsigned)BH, CSR_SCAN_THREADS, 0, st>>>(t->bsum, nblk, t->offsets, N);
    csr_apply_kernel<<<gb, CSR_SCAN_THREADS, 0, st>>>(t->cursor, t->offsets, N, t->bsum, nblk, t->nlong, t->longseg);
    return cudaGetLastError();
}

}  // namespace onedf
