// sort.cu -- A3 segmented stable LSD radix sort of Morton codes (K3) and the
// A9 backward transpose: stable radix sort of (key j, slot s) pairs + CSR
// offsets (K8).
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
// cost a pass.
//
// A9 (north_star "sorted-index segment reduction rather than float atomics"):
// slot ids s = i*k + r sorted stably by j = idx[s] per (b,h) -- reduce-then-
// scan LSD radix with up to 9-bit digits: per-tile digit counts (upsweep),
// per-(b,h) exclusive scan in (digit, tile) order, and a warp-ranked stable
// scatter (downsweep).  Invalid slots (idx = -1) get key N and sort last.
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
    int64_t N, int64_t M, int64_t runs_per_bh, SortScratch scr) {
    using Pos = typename std::conditional<SMEM, uint16_t, uint32_t>::type;
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t bh = blockIdx.x / runs_per_bh;
    const int64_t c = blockIdx.x % runs_per_bh;
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
                                                                                        runs, scr);
        return cudaGetLastError();
    }
    int nw = (int)((M + 32 * 8 - 1) / (32 * 8));   // ~8 keys per lane
    nw = nw < 1 ? 1 : (nw > SEG_MAX_WARPS ? SEG_MAX_WARPS : nw);
    const size_t smem = seg_sort_smem(M, nw);
    cudaError_t e = cudaFuncSetAttribute(seg_sort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    seg_sort_kernel<true><<<(unsigned)(BH * runs), nw * 32, smem, st>>>(kcode, scode, perm, N, M, runs, scr);
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

// ============================================================================ K8
// Reduce-then-scan LSD radix sort of the (j, slot) pairs of every (b,h) by j,
// 8-bit digits, ceil(log2 N / 8) passes (2 at N = 64K).  Pass 0 reads idx
// directly (key j, value = slot id) and drops the invalid slots (j = -1).
// Per pass: (1) upsweep: per-tile digit counts -> hist[bh][digit][tile];
// (2) scan: one CTA per (bh, digit) turns its row into tile offsets within
// the digit and writes the digit total; (3) downsweep: each CTA ranks its
// tile stably (per-round __match_any_sync peers + per-warp running digit
// counts, then a (digit, warp)-ordered tile scan), stages the tile digit-
// sorted in shared memory, and writes each digit's run to its global slot
// with consecutive threads on consecutive addresses (coalesced).
#ifndef ONEDF_TR_THREADS
#define ONEDF_TR_THREADS 256
#endif
#ifndef ONEDF_TR_IPT
#define ONEDF_TR_IPT 8
#endif
#ifndef ONEDF_TR_MINB
#define ONEDF_TR_MINB 4
#endif
constexpr int TR_THREADS = ONEDF_TR_THREADS;
constexpr int TR_WARPS = TR_THREADS / 32;
constexpr int TR_IPT = ONEDF_TR_IPT;
constexpr int TR_TILE = TR_THREADS * TR_IPT;       // 2048 pairs per tile
constexpr int TR_RADIX = 256;

struct TrPlan {
    int64_t L;        // pairs per (b,h) = N*k
    int64_t tiles;    // per (b,h)
    int passes;
};

static TrPlan tr_plan(const onedf_problem* p) {
    TrPlan t;
    t.L = p->N * (int64_t)p->k;
    t.tiles = (t.L + TR_TILE - 1) / TR_TILE;
    int nb = 1;
    while ((1ll << nb) < p->N) ++nb;      // keys j in [0, N)
    t.passes = (nb + 7) / 8;
    return t;
}

void transpose_carve(const onedf_problem* p, Carver* c, TransposeBufs* t) {
    const int64_t BH = p->B * p->H;
    TrPlan pl = tr_plan(p);
    for (int b = 0; b < 2; ++b) {
        t->keys[b] = c->take<uint32_t>((size_t)(BH * pl.L));
        t->vals[b] = c->take<uint32_t>((size_t)(BH * pl.L));
    }
    t->hist = c->take<uint32_t>((size_t)(BH * TR_RADIX * pl.tiles));
    t->dtot = c->take<uint32_t>((size_t)(BH * TR_RADIX));
    t->nvalid = c->take<uint32_t>((size_t)BH);
    t->offsets = c->take<int32_t>((size_t)(BH * (p->N + 1)));
    t->slots = nullptr;
}

struct TrArgs {
    const int32_t* idx; const uint32_t* keys_in; const uint32_t* vals_in;
    uint32_t* keys_out; uint32_t* vals_out;
    uint32_t* hist; uint32_t* dtot; uint32_t* nvalid;
    int64_t L, tiles;
    int shift, first, k;
    Shard sh;            // sharded: only the owned queries' slots enter the transpose
};

__device__ __forceinline__ bool tr_load(const TrArgs& a, int64_t bh, int64_t pos, uint32_t nv, uint32_t& key,
                                        uint32_t& val) {
    if (a.first) {
        if (pos >= a.L) return false;
        if (a.sh.on() && !a.sh.owns_row(pos / a.k)) return false;
        const int32_t j = __ldg(a.idx + bh * a.L + pos);
        key = (uint32_t)j;
        val = (uint32_t)pos;
        return j >= 0;
    }
    if (pos >= (int64_t)nv) return false;
    key = __ldg(a.keys_in + bh * a.L + pos);
    val = __ldg(a.vals_in + bh * a.L + pos);
    return true;
}

// Exclusive scan of one value per thread over a TR_THREADS block; returns the total.
__device__ __forceinline__ uint32_t tr_block_scan(uint32_t v, uint32_t& excl, uint32_t* s_w) {
    const int lane = lane_id(), w = threadIdx.x / 32;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t woff = 0, tot = 0;
#pragma unroll
    for (int x = 0; x < TR_WARPS; ++x) {
        const uint32_t t = s_w[x];
        woff += x < w ? t : 0;
        tot += t;
    }
    excl = woff + inc - v;
    __syncthreads();
    return tot;
}

__global__ void __launch_bounds__(TR_THREADS) tr_upsweep_kernel(const TrArgs a) {
    __shared__ uint32_t h[TR_RADIX];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    const uint32_t nv = a.first ? 0u : __ldg(a.nvalid + bh);
#pragma unroll
    for (int r = 0; r < TR_IPT; ++r) {
        const int64_t pos = tile * TR_TILE + r * TR_THREADS + threadIdx.x;
        uint32_t key, val;
        if (tr_load(a, bh, pos, nv, key, val)) atomicAdd(&h[(key >> a.shift) & 0xffu], 1u);   // integer: order-free
    }
    __syncthreads();
    a.hist[(bh * TR_RADIX + threadIdx.x) * a.tiles + tile] = h[threadIdx.x];
}

// One CTA per (digit, bh): exclusive scan of the digit's tile counts.
__global__ void __launch_bounds__(1024) tr_scan_kernel(const TrArgs a) {
    const int64_t bh = blockIdx.y, d = blockIdx.x;
    uint32_t* h = a.hist + (bh * TR_RADIX + d) * a.tiles;
    const int64_t per = (a.tiles + 1023) / 1024;
    const int64_t t0 = threadIdx.x * per, t1 = min64(a.tiles, t0 + per);
    uint32_t sum = 0;
    for (int64_t t = t0; t < t1; ++t) sum += h[t];
    __shared__ uint32_t wsum[32];
    const int lane = lane_id(), w = threadIdx.x / 32;
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t v = wsum[lane];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        wsum[lane] = x - v;
        if (lane == 31) {
            a.dtot[bh * TR_RADIX + d] = x;
            if (a.first) atomicAdd(a.nvalid + bh, x);   // integer: order-free
        }
    }
    __syncthreads();
    uint32_t run = wsum[w] + inc - sum;
    for (int64_t t = t0; t < t1; ++t) { const uint32_t x = h[t]; h[t] = run; run += x; }
}

__global__ void __launch_bounds__(TR_THREADS, ONEDF_TR_MINB) tr_downsweep_kernel(const TrArgs a) {
    __shared__ uint32_t sk[TR_TILE], sv[TR_TILE];
    __shared__ uint32_t cnt[TR_WARPS * TR_RADIX];    // [warp][digit]: a warp's random digits hit distinct banks
    __shared__ uint32_t tstart[TR_RADIX], gbase[TR_RADIX];
    __shared__ uint32_t s_w[TR_WARPS];
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    const int w = threadIdx.x / 32, lane = lane_id();
    const uint32_t nv = a.first ? 0u : __ldg(a.nvalid + bh);
    for (int t = threadIdx.x; t < TR_RADIX * TR_WARPS; t += TR_THREADS) cnt[t] = 0;
    {
        // global base of each digit for this tile: digit start + tile offset within the digit
        const int d = threadIdx.x;
        uint32_t ex;
        tr_block_scan(__ldg(a.dtot + bh * TR_RADIX + d), ex, s_w);
        gbase[d] = ex + __ldg(a.hist + (bh * TR_RADIX + d) * a.tiles + tile);
    }
    __syncthreads();
    uint32_t key[TR_IPT], val[TR_IPT], rank[TR_IPT];
    bool act[TR_IPT];
#pragma unroll
    for (int r = 0; r < TR_IPT; ++r) {
        const int64_t pos = tile * TR_TILE + (int64_t)w * (32 * TR_IPT) + r * 32 + lane;
        act[r] = tr_load(a, bh, pos, nv, key[r], val[r]);
    }
#pragma unroll
    for (int r = 0; r < TR_IPT; ++r) {
        const uint32_t d = act[r] ? ((key[r] >> a.shift) & 0xffu) : (uint32_t)TR_RADIX + lane;
        const unsigned peers = __match_any_sync(FULL, d);
        uint32_t prev = 0;
        if (act[r]) prev = cnt[w * TR_RADIX + d];
        rank[r] = prev + __popc(peers & lanemask_lt());
        __syncwarp();
        if (act[r] && lane == __ffs(peers) - 1) cnt[w * TR_RADIX + d] = prev + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        // (digit, warp)-ordered exclusive scan of the tile: thread d owns digit d's warps
        const int d = threadIdx.x;
        uint32_t pw[TR_WARPS], td = 0;
#pragma unroll
        for (int x = 0; x < TR_WARPS; ++x) { pw[x] = td; td += cnt[x * TR_RADIX + d]; }
        uint32_t ex;
        tr_block_scan(td, ex, s_w);
        tstart[d] = ex;
#pragma unroll
        for (int x = 0; x < TR_WARPS; ++x) cnt[x * TR_RADIX + d] = ex + pw[x];
    }
    __syncthreads();
    int ntile = 0;
#pragma unroll
    for (int r = 0; r < TR_IPT; ++r) {
        if (act[r]) {
            const uint32_t d = (key[r] >> a.shift) & 0xffu;
            const uint32_t lp = cnt[w * TR_RADIX + d] + rank[r];
            sk[lp] = key[r];
            sv[lp] = val[r];
        }
        ntile += __syncthreads_count(act[r]);
    }
    for (int p = threadIdx.x; p < ntile; p += TR_THREADS) {
        const uint32_t k2 = sk[p];
        const uint32_t d = (k2 >> a.shift) & 0xffu;
        const int64_t g = (int64_t)gbase[d] + (p - (int)tstart[d]);
        a.keys_out[bh * a.L + g] = k2;
        a.vals_out[bh * a.L + g] = sv[p];
    }
}

// CSR offsets: off[j] = first sorted position with key >= j, off[N] = #valid.
__global__ void tr_offsets_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ nvalid,
                                  int32_t* __restrict__ off, int64_t L, uint32_t N) {
    const int64_t bh = blockIdx.y;
    const uint32_t* kk = keys + bh * L;
    int32_t* o = off + bh * ((int64_t)N + 1);
    const int64_t nv = __ldg(nvalid + bh);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= nv; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t prev = p == 0 ? 0u : __ldg(kk + p - 1) + 1u;     // first key not yet assigned
        const uint32_t cur = p == nv ? N : __ldg(kk + p);
        for (uint32_t j = prev; j <= cur; ++j) o[j] = (int32_t)p;
    }
}

cudaError_t launch_transpose(const onedf_problem* p, const int32_t* idx, TransposeBufs* t, cudaStream_t st) {
    const int64_t BH = p->B * p->H;
    const TrPlan pl = tr_plan(p);
    const dim3 grid((unsigned)pl.tiles, (unsigned)BH);
    cudaError_t e = cudaMemsetAsync(t->nvalid, 0, (size_t)BH * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    int cur = -1;   // -1: read from idx
    for (int ps = 0; ps < pl.passes; ++ps) {
        const int out = (cur + 1) & 1;
        TrArgs a;
        a.idx = idx;
        a.keys_in = cur < 0 ? nullptr : t->keys[cur];
        a.vals_in = cur < 0 ? nullptr : t->vals[cur];
        a.keys_out = t->keys[out];
        a.vals_out = t->vals[out];
        a.hist = t->hist; a.dtot = t->dtot; a.nvalid = t->nvalid;
        a.L = pl.L; a.tiles = pl.tiles; a.shift = 8 * ps; a.first = cur < 0;
        a.k = p->k; a.sh = make_shard(p);
        tr_upsweep_kernel<<<grid, TR_THREADS, 0, st>>>(a);
        tr_scan_kernel<<<dim3(TR_RADIX, (unsigned)BH), 1024, 0, st>>>(a);
        tr_downsweep_kernel<<<grid, TR_THREADS, 0, st>>>(a);
        cur = out;
    }
    const unsigned ob = (unsigned)min64((pl.L + 1 + 255) / 256, 4096);
    tr_offsets_kernel<<<dim3(ob, (unsigned)BH), 256, 0, st>>>(t->keys[cur], t->nvalid, t->offsets, pl.L,
                                                              (uint32_t)p->N);
    t->slots = t->vals[cur];
    return cudaGetLastError();
}

}  // namespace onedf
