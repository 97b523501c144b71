// sort.cu -- A3 segmented stable LSD radix sort of Morton codes (K3), also
// used for the Morton query schedule of the fwd/bwd kernels.
//
// A3 ("torch.sort", "radix sorted in O(N)", Alg. P:1786-1790,
// S:215-223): every run (chunk of M positions, or all N when non-causal) is
// sorted by (code, position).  One CTA owns one run; keys and 16-bit local
// positions live in shared memory (ping-pong), 8-bit digits, and each pass
// is a stable counting sort built from warp-level __match_any_sync
// histograms: per warp a digit histogram (leader lane adds popc(peers)), a
// CTA-wide exclusive scan in (digit, warp) order, and a scatter whose rank
// is popc(peers & lanemask_lt).  Digits that are constant across the run
// (AND/OR reduction) are skipped, so only the varying bits of the codes
// cost a pass.  The backward transpose (A9) is in csr.cu.
#include "common.cuh"
#include "internal.h"

#include <type_traits>

namespace onedf {

// ============================================================================ K3
constexpr int SEG_MAX_WARPS = 16;
constexpr int SEG_BIG_WARPS = 32;      // runs longer than SEG_SORT_MAX: keys stay in global scratch

// One CTA sorts one run.  SMEM: the run (<= SEG_SORT_MAX keys) lives in shared
// memory with 16-bit local positions; otherwise the ping-pong key/position
// buffers are global scratch (same algorithm, L2-resident per run) and only
// the digit histograms are in shared memory.
template <bool SMEM>
__global__ void __launch_bounds__((SMEM ? SEG_MAX_WARPS : SEG_BIG_WARPS) * 32) seg_sort_kernel(
    const uint64_t* __restrict__ kcode, uint64_t* __restrict__ scode, int32_t* __restrict__ perm,
    int64_t N, int64_t M, int64_t runs_per_bh, SortScratch scr, Shard sh) {
    using Pos = typename std::conditional<SMEM, uint16_t, uint32_t>::type;
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t bh = blockIdx.x / runs_per_bh;
    const int64_t c = blockIdx.x % runs_per_bh;
    if (sh.on() && Shard::owner(c, sh.world) != sh.rank) return;   // sharded: other ranks' runs arrive by all-gather
    const int64_t s0 = c * M;
    const int n = (int)min64(M, N - s0);
    const int nw = blockDim.x / 32;
    uint64_t *keys0, *keys1;
    Pos *vals0, *vals1;
    uint32_t* hist;
    if (SMEM) {
        const int nmax = (int)M;
        keys0 = reinterpret_cast<uint64_t*>(smem);
        keys1 = keys0 + nmax;
        const int npad = (nmax + 7) & ~7;       // keeps vals1 and hist 16-B aligned for odd run lengths
        vals0 = reinterpret_cast<Pos*>(keys1 + nmax);
        vals1 = vals0 + npad;
        hist = reinterpret_cast<uint32_t*>(reinterpret_cast<uint16_t*>(vals1) + npad);  // [256][nw]
    } else {
        const int64_t o = bh * N + s0;
        keys0 = scr.k[0] + o;
        keys1 = scr.k[1] + o;
        vals0 = reinterpret_cast<Pos*>(scr.v[0] + o);
        vals1 = reinterpret_cast<Pos*>(scr.v[1] + o);
        hist = reinterpret_cast<uint32_t*>(smem);
    }
    __shared__ unsigned long long s_and, s_or;

    const uint64_t* src = kcode + bh * N + s0;
    unsigned long long my_and = ~0ull, my_or = 0ull;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        uint64_t k = src[r];
        keys0[r] = k;
        vals0[r] = (Pos)r;
        my_and &= k;
        my_or |= k;
    }
    if (threadIdx.x == 0) { s_and = ~0ull; s_or = 0ull; }
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_and &= __shfl_xor_sync(FULL, my_and, o);
        my_or |= __shfl_xor_sync(FULL, my_or, o);
    }
    if (lane_id() == 0) { atomicAnd(&s_and, my_and); atomicOr(&s_or, my_or); }
    __syncthreads();
    const uint64_t varying = s_and ^ s_or;

    const int w = threadIdx.x / 32, lane = lane_id();
    const int per_warp = (n + nw - 1) / nw;
    const int w0 = min(n, w * per_warp), w1 = min(n, w0 + per_warp);
    uint64_t* ks = keys0; uint64_t* kd = keys1;
    Pos* vs = vals0; Pos* vd = vals1;

    for (int shift = 0; shift < 64; shift += 8) {
        if (((varying >> shift) & 0xffull) == 0) continue;   // uniform across threads
        for (int t = threadIdx.x; t < 256 * nw; t += blockDim.x) hist[t] = 0;
        __syncthreads();
        // phase A: per-warp digit counts
        for (int base = w0; base < w1; base += 32) {
            const int r = base + lane;
            const bool act = r < w1;
            const unsigned d = act ? (unsigned)((ks[r] >> shift) & 0xff) : 256u + lane;
            const unsigned peers = __match_any_sync(FULL, d);
            if (act && lane == __ffs(peers) - 1) hist[d * nw + w] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // exclusive scan over hist in (digit, warp) order -- 256*nw entries
        {
            const int total = 256 * nw;
            const int per = (total + blockDim.x - 1) / blockDim.x;
            const int a = threadIdx.x * per, b = min(total, a + per);
            uint32_t sum = 0;
            for (int t = a; t < b; ++t) sum += hist[t];
            __shared__ uint32_t wsum[SEG_BIG_WARPS];
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsum[w] = incl;
            __syncthreads();
            uint32_t woff = 0;
            for (int v = 0; v < w; ++v) woff += wsum[v];
            uint32_t run = woff + incl - sum;
            for (int t = a; t < b; ++t) { uint32_t h = hist[t]; hist[t] = run; run += h; }
        }
        __syncthreads();
        // phase B: stable scatter
        for (int base = w0; base < w1; base += 32) {
            const int r = base + lane;
            const bool act = r < w1;
            uint64_t key = act ? ks[r] : 0;
            const unsigned d = act ? (unsigned)((key >> shift) & 0xff) : 256u + lane;
            const unsigned peers = __match_any_sync(FULL, d);
            if (act) {
                const uint32_t dst = hist[d * nw + w] + __popc(peers & lanemask_lt());
                kd[dst] = key;
                vd[dst] = vs[r];
            }
            __syncwarp();
            if (act && lane == __ffs(peers) - 1) hist[d * nw + w] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        uint64_t* tk = ks; ks = kd; kd = tk;
        Pos* tv = vs; vs = vd; vd = tv;
    }
    uint64_t* outk = scode ? scode + bh * N + s0 : nullptr;
    int32_t* outp = perm + bh * N + s0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        if (scode) outk[r] = ks[r];
        outp[r] = (int32_t)(s0 + (int64_t)vs[r]);
    }
}

static size_t seg_sort_smem(int64_t M, int nw) {
    return (size_t)M * 8 * 2 + (size_t)((M + 7) & ~7ll) * 2 * 2 + 256 * (size_t)nw * 4;
}

void sort_carve(const onedf_problem* p, Carver* c, SortScratch* s) {
    const bool big = run_len_max(p) > SEG_SORT_MAX;
    const size_t n = big ? (size_t)(p->B * p->H * p->N) : 0;
    for (int b = 0; b < 2; ++b) {
        s->k[b] = big ? c->take<uint64_t>(n) : nullptr;
        s->v[b] = big ? c->take<uint32_t>(n) : nullptr;
    }
}

cudaError_t launch_seg_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm,
                            const SortScratch& scr, cudaStream_t st) {
    const int64_t N = p->N, BH = p->B * p->H;
    const int64_t M = run_len_max(p);
    const int64_t runs = num_runs(p);
    if (M > SEG_SORT_MAX) {
        const size_t smem = 256 * (size_t)SEG_BIG_WARPS * 4;
        seg_sort_kernel<false><<<(unsigned)(BH * runs), SEG_BIG_WARPS * 32, smem, st>>>(kcode, scode, perm, N, M,
                                                                                        runs, scr, make_shard(p));
        return cudaGetLastError();
    }
    int nw = (int)((M + 32 * 8 - 1) / (32 * 8));   // ~8 keys per lane
    nw = nw < 1 ? 1 : (nw > SEG_MAX_WARPS ? SEG_MAX_WARPS : nw);
    const size_t smem = seg_sort_smem(M, nw);
    cudaError_t e = cudaFuncSetAttribute(seg_sort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    seg_sort_kernel<true><<<(unsigned)(BH * runs), nw * 32, smem, st>>>(kcode, scode, perm, N, M, runs, scr,
                                                                       make_shard(p));
    return cudaGetLastError();
}

// The query schedule of K6/K7: the queries of every chunk (the same chunking
// as the key runs; all N when non-causal) sorted by (qcode, i).  Neighbouring
// schedule slots are then close in space, which is what lets a CTA's warps
// share candidate records and gathered rows through L1.  Pure reordering of
// work -- no output depends on it.
cudaError_t launch_query_order(const onedf_problem* p, const uint64_t* qcode, int32_t* qorder,
                               const SortScratch& scr, cudaStream_t st) {
    return launch_seg_sort(p, qcode, nullptr, qorder, scr, st);
}

}  // namespace onedf
