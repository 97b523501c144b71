// workload.cu -- the locality / recall workload on the
// same encode + sort kernels: Fig. 4 "overlap between the
// top-64 nearest neighbors before and after projection" and the k ablation
// (P:1583-1587).
//
// K12 code_knn: for every query, the k keys nearest in Morton code
// (|kcode - qcode|, u64; ties by position, D19), from the sorted run that
// onedf_sort built.  One thread per query: lower_bound of qcode in the run,
// then a two-cursor merge outward in (distance, position) order.  The right
// cursor walks up from the insertion point (codes >= q ascending, equal codes
// by ascending position).  The left side is consumed block by block (a block
// = the positions holding one code value, found by lower_bound), each block in
// ascending position, blocks from the nearest code outward -- so ties are
// broken by position exactly as the oracle's sort does.  O(k + blocks * log M)
// per query.
//
// K13 overlap: |A_r ∩ B_r| per row of two index lists (-1 entries and,
// optionally, the row's own position ignored) -- the locality metric.
#include "common.cuh"
#include "internal.h"

namespace onedf {

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t lo, int64_t hi, uint64_t x) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void code_knn_kernel(const uint64_t* __restrict__ qcode, const uint64_t* __restrict__ scode,
                                const int32_t* __restrict__ perm, int32_t* __restrict__ idx, int64_t N, int64_t M,
                                int64_t total, int k, int causal, int exclude_self) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int64_t bh = t / N, i = t % N;
    const uint64_t qc = __ldg(qcode + t);
    int32_t* out = idx + t * k;
    int n = 0;
    // one sorted run per admissible chunk (causal) or the whole row; runs are merged by
    // repeatedly taking the best head over all runs (the workload uses a single run)
    const int64_t nruns = causal ? i / M : 1;
    if (nruns == 1) {
        const int64_t s0 = 0, len = causal ? min64(M, N) : N;
        const uint64_t* run = scode + bh * N + s0;
        const int32_t* pm = perm + bh * N + s0;
        const int64_t p = lower_bound_u64(run, 0, len, qc);
        int64_t rc = p;                                   // right cursor
        int64_t lend = p, lbeg = p, lc = p;               // left block [lbeg, lend), cursor lc
        if (p > 0) { lbeg = lower_bound_u64(run, 0, p, __ldg(run + p - 1)); lc = lbeg; }
        while (n < k) {
            const bool hasL = lc < lend, hasR = rc < len;
            if (!hasL && !hasR) break;
            bool takeL;
            if (hasL && hasR) {
                const uint64_t dL = qc - __ldg(run + lc), dR = __ldg(run + rc) - qc;
                const int32_t jL = __ldg(pm + lc), jR = __ldg(pm + rc);
                takeL = dL < dR || (dL == dR && jL < jR);
            } else {
                takeL = hasL;
            }
            int32_t j;
            if (takeL) {
                j = __ldg(pm + lc);
                if (++lc == lend) {                       // next block to the left
                    lend = lbeg;
                    if (lend > 0) { lbeg = lower_bound_u64(run, 0, lend, __ldg(run + lend - 1)); lc = lbeg; }
                    else lc = lend;
                }
            } else {
                j = __ldg(pm + rc);
                ++rc;
            }
            if (exclude_self && j == (int32_t)i) continue;
            out[n++] = j;
        }
    }
    // nruns == 0 (a chunk-0 query) has nothing admissible; nruns > 1 is rejected by the ABI
    for (; n < k; ++n) out[n] = -1;
}

__global__ void overlap_kernel(const int32_t* __restrict__ a, int ka, const int32_t* __restrict__ b, int kb,
                               int64_t rows, int64_t self_period, int32_t* __restrict__ counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int32_t self = self_period > 0 ? (int32_t)(r % self_period) : -1;
    int c = 0;
    for (int x = 0; x < ka; ++x) {
        const int32_t v = __ldg(a + r * ka + x);
        if (v < 0 || v == self) continue;
        bool dup = false;                                  // count each index once
        for (int y = 0; y < x; ++y) dup |= __ldg(a + r * ka + y) == v;
        if (dup) continue;
        for (int y = 0; y < kb; ++y) {
            if (__ldg(b + r * kb + y) == v) { ++c; break; }
        }
    }
    counts[r] = c;
}

cudaError_t launch_code_knn(const onedf_problem* p, const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                            int exclude_self, int32_t* idx, cudaStream_t st) {
    const int64_t total = p->B * p->H * p->N;
    code_knn_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(qcode, scode, perm, idx, p->N, run_len_max(p),
                                                                     total, p->k, p->causal, exclude_self);
    return cudaGetLastError();
}

cudaError_t launch_overlap(const int32_t* a, int ka, const int32_t* b, int kb, int64_t rows, int64_t self_period,
                           int32_t* counts, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    overlap_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(a, ka, b, kb, rows, self_period, counts);
    return cudaGetLastError();
}

}  // namespace onedf
