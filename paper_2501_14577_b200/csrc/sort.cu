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

namespace onedf {

// ============================================================================ K3
constexpr int SEG_MAX_WARPS = 16;

__global__ void __launch_bounds__(SEG_MAX_WARPS * 32) seg_sort_kernel(
    const uint64_t* __restrict__ kcode, uint64_t* __restrict__ scode, int32_t* __restrict__ perm,
    int64_t N, int64_t M, int64_t runs_per_bh) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t bh = blockIdx.x / runs_per_bh;
    const int64_t c = blockIdx.x % runs_per_bh;
    const int64_t s0 = c * M;
    const int n = (int)min64(M, N - s0);
    const int nw = blockDim.x / 32;
    const int nmax = (int)M;
    uint64_t* keys0 = reinterpret_cast<uint64_t*>(smem);
    uint64_t* keys1 = keys0 + nmax;
    uint16_t* vals0 = reinterpret_cast<uint16_t*>(keys1 + nmax);
    uint16_t* vals1 = vals0 + nmax;
    uint32_t* hist = reinterpret_cast<uint32_t*>(vals1 + ((nmax + 7) & ~7));  // [256][nw]
    __shared__ unsigned long long s_and, s_or;

    const uint64_t* src = kcode + bh * N + s0;
    unsigned long long my_and = ~0ull, my_or = 0ull;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        uint64_t k = src[r];
        keys0[r] = k;
        vals0[r] = (uint16_t)r;
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
    uint16_t* vs = vals0; uint16_t* vd = vals1;

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
            // block exclusive scan of per-thread sums
            __shared__ uint32_t wsum[SEG_MAX_WARPS];
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
        uint16_t* tv = vs; vs = vd; vd = tv;
    }
    uint64_t* outk = scode + bh * N + s0;
    int32_t* outp = perm + bh * N + s0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        outk[r] = ks[r];
        outp[r] = (int32_t)(s0 + vs[r]);
    }
}

static size_t seg_sort_smem(int64_t M, int nw) {
    return (size_t)M * 8 * 2 + (size_t)((M + 7) & ~7ll) * 2 * 2 + 256 * (size_t)nw * 4;
}

cudaError_t launch_seg_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm,
                            cudaStream_t st) {
    const int64_t N = p->N, BH = p->B * p->H;
    const int64_t M = run_len_max(p);
    const int64_t runs = num_runs(p);
    int nw = (int)((M + 32 * 8 - 1) / (32 * 8));   // ~8 keys per lane
    nw = nw < 1 ? 1 : (nw > SEG_MAX_WARPS ? SEG_MAX_WARPS : nw);
    const size_t smem = seg_sort_smem(M, nw);
    cudaError_t e = cudaFuncSetAttribute(seg_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    seg_sort_kernel<<<(unsigned)(BH * runs), nw * 32, smem, st>>>(kcode, scode, perm, N, M, runs);
    return cudaGetLastError();
}

// ============================================================================ K8
constexpr int TR_THREADS = 256;
constexpr int TR_IPT = 16;
constexpr int TR_TILE = TR_THREADS * TR_IPT;       // 4096 items per tile
constexpr int TR_WARPS = TR_THREADS / 32;
constexpr int TR_MAXB = 512;                       // up to 9-bit digits

struct TrPlan {
    int64_t L;        // items per (b,h) = N*k
    int64_t tiles;    // per (b,h)
    int nbits;        // key bits (keys in [0, N])
    int passes;
    int dbits;        // digit bits per pass
};

static TrPlan tr_plan(const onedf_problem* p) {
    TrPlan t;
    t.L = p->N * (int64_t)p->k;
    t.tiles = (t.L + TR_TILE - 1) / TR_TILE;
    int nb = 1;
    while ((1ll << nb) <= p->N) ++nb;     // sentinel N must fit
    t.nbits = nb;
    t.passes = (nb + 8) / 9;
    t.dbits = (nb + t.passes - 1) / t.passes;
    return t;
}

void transpose_carve(const onedf_problem* p, Carver* c, TransposeBufs* t) {
    const int64_t BH = p->B * p->H;
    TrPlan pl = tr_plan(p);
    for (int b = 0; b < 2; ++b) {
        t->keys[b] = c->take<uint32_t>((size_t)(BH * pl.L));
        t->vals[b] = c->take<uint32_t>((size_t)(BH * pl.L));
    }
    t->hist = c->take<uint32_t>((size_t)(BH * (1 << pl.dbits) * pl.tiles));
    t->offsets = c->take<int32_t>((size_t)(BH * (p->N + 1)));
    t->slots = nullptr;
}

__device__ __forceinline__ uint32_t tr_key_from_idx(int32_t j, uint32_t N) { return j < 0 ? N : (uint32_t)j; }

// Upsweep: digit counts of one tile -> hist[bh][digit][tile].
__global__ void __launch_bounds__(TR_THREADS) tr_upsweep_kernel(
    const int32_t* __restrict__ idx, const uint32_t* __restrict__ keys_in, uint32_t* __restrict__ hist,
    int64_t L, int64_t tiles, uint32_t N, int shift, int dbits) {
    __shared__ uint32_t h[TR_MAXB];
    const int nb = 1 << dbits;
    for (int t = threadIdx.x; t < nb; t += TR_THREADS) h[t] = 0;
    __syncthreads();
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    const int64_t base = bh * L + tile * TR_TILE;
    const int64_t lim = min64(TR_TILE, L - tile * TR_TILE);
    const uint32_t mask = (uint32_t)nb - 1;
    for (int t = threadIdx.x; t < lim; t += TR_THREADS) {
        uint32_t key = keys_in ? keys_in[base + t] : tr_key_from_idx(idx[base + t], N);
        atomicAdd(&h[(key >> shift) & mask], 1u);   // integer counts: order-independent
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += TR_THREADS) hist[(bh * nb + t) * tiles + tile] = h[t];
}

// Exclusive scan of hist[bh][*][*] in (digit, tile) order; one CTA per (b,h).
__global__ void __launch_bounds__(1024) tr_scan_kernel(uint32_t* __restrict__ hist, int64_t count) {
    uint32_t* h = hist + (int64_t)blockIdx.x * count;
    const int64_t per = (count + blockDim.x - 1) / blockDim.x;
    const int64_t a = threadIdx.x * per, b = min64(count, a + per);
    uint32_t sum = 0;
    for (int64_t t = a; t < b; ++t) sum += h[t];
    __shared__ uint32_t wsum[32];
    const int lane = lane_id(), w = threadIdx.x / 32;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < (int)(blockDim.x / 32) ? wsum[lane] : 0;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        wsum[lane] = inc - v;
    }
    __syncthreads();
    uint32_t run = wsum[w] + incl - sum;
    for (int64_t t = a; t < b; ++t) { uint32_t x = h[t]; h[t] = run; run += x; }
}

// Downsweep: stable scatter of one tile.  Warp w owns items [w*512, (w+1)*512)
// of the tile; lane l takes item w*512 + r*32 + l in round r, so (warp, round,
// lane) order == input order and ranks from __match_any_sync keep stability.
__global__ void __launch_bounds__(TR_THREADS) tr_downsweep_kernel(
    const int32_t* __restrict__ idx, const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, const uint32_t* __restrict__ hist,
    int64_t L, int64_t tiles, uint32_t N, int shift, int dbits) {
    __shared__ uint32_t wh[TR_MAXB * TR_WARPS];   // [digit][warp]
    const int nb = 1 << dbits;
    const uint32_t mask = (uint32_t)nb - 1;
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    const int64_t base = bh * L + tile * TR_TILE;
    const int64_t lim = min64(TR_TILE, L - tile * TR_TILE);
    const int w = threadIdx.x / 32, lane = lane_id();
    for (int t = threadIdx.x; t < nb * TR_WARPS; t += TR_THREADS) wh[t] = 0;
    __syncthreads();
    uint32_t key[TR_IPT], val[TR_IPT], rank[TR_IPT];
#pragma unroll
    for (int r = 0; r < TR_IPT; ++r) {
        const int64_t it = (int64_t)w * (32 * TR_IPT) + r * 32 + lane;
        const bool act = it < lim;
        if (act) {
            key[r] = keys_in ? keys_in[base + it] : tr_key_from_idx(idx[base + it], N);
            val[r] = vals_in ? vals_in[base + it] : (uint32_t)(tile * TR_TILE + it);
        } else {
            key[r] = 0xffffffffu; val[r] = 0;
        }
        const uint32_t d = act ? ((key[r] >> shift) & mask) : (uint32_t)TR_MAXB + lane;
        const unsigned peers = __match_any_sync(FULL, d);
        if (act) {
            rank[r] = wh[d * TR_WARPS + w] + __popc(peers & lanemask_lt());
        }
        __syncwarp();
        if (act && lane == __ffs(peers) - 1) wh[d * TR_WARPS + w] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix across warps + the global (digit, tile) offset
    for (int d = threadIdx.x; d < nb; d += TR_THREADS) {
        uint32_t run = hist[(bh * nb + d) * tiles + tile];
        for (int v = 0; v < TR_WARPS; ++v) { uint32_t c = wh[d * TR_WARPS + v]; wh[d * TR_WARPS + v] = run; run += c; }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < TR_IPT; ++r) {
        const int64_t it = (int64_t)w * (32 * TR_IPT) + r * 32 + lane;
        if (it < lim) {
            const uint32_t d = (key[r] >> shift) & mask;
            const uint32_t dst = wh[d * TR_WARPS + w] + rank[r];
            keys_out[bh * L + dst] = key[r];
            vals_out[bh * L + dst] = val[r];
        }
    }
}

// CSR offsets: off[j] = first sorted position with key >= j, off[N] = #valid.
__global__ void tr_offsets_kernel(const uint32_t* __restrict__ keys, int32_t* __restrict__ off, int64_t L,
                                  uint32_t N) {
    const int64_t bh = blockIdx.y;
    const uint32_t* kk = keys + bh * L;
    int32_t* o = off + bh * ((int64_t)N + 1);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= L; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t prev = p == 0 ? 0u : kk[p - 1] + 1u;     // first key not yet assigned
        const uint32_t cur = p == L ? N : kk[p];
        for (uint32_t j = prev; j <= cur && j <= N; ++j) o[j] = (int32_t)p;
        if (p == L) {
            // keys == N (invalid) never start a CSR row; nothing else to do
        }
    }
}

cudaError_t launch_transpose(const onedf_problem* p, const int32_t* idx, TransposeBufs* t, cudaStream_t st) {
    const int64_t BH = p->B * p->H;
    const TrPlan pl = tr_plan(p);
    const dim3 grid((unsigned)pl.tiles, (unsigned)BH);
    const uint32_t N = (uint32_t)p->N;
    int cur = -1;   // -1: read keys from idx, vals implicit
    for (int ps = 0; ps < pl.passes; ++ps) {
        const int shift = ps * pl.dbits;
        const int out = (cur + 1) & 1;
        const uint32_t* kin = cur < 0 ? nullptr : t->keys[cur];
        const uint32_t* vin = cur < 0 ? nullptr : t->vals[cur];
        tr_upsweep_kernel<<<grid, TR_THREADS, 0, st>>>(idx, kin, t->hist, pl.L, pl.tiles, N, shift, pl.dbits);
        tr_scan_kernel<<<(unsigned)BH, 1024, 0, st>>>(t->hist, (int64_t)(1 << pl.dbits) * pl.tiles);
        tr_downsweep_kernel<<<grid, TR_THREADS, 0, st>>>(idx, kin, vin, t->keys[out], t->vals[out], t->hist, pl.L,
                                                        pl.tiles, N, shift, pl.dbits);
        cur = out;
    }
    const unsigned ob = (unsigned)min64((pl.L + 1 + 255) / 256, 4096);
    tr_offsets_kernel<<<dim3(ob, (unsigned)BH), 256, 0, st>>>(t->keys[cur], t->offsets, pl.L, N);
    t->slots = t->vals[cur];
    return cudaGetLastError();
}

}  // namespace onedf
