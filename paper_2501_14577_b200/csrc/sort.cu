// sort.cu -- A3 segmented stable LSD radix sort of Morton codes (K3), also
// used for the Morton query schedule of the fwd/bwd kernels.
//
// A3 ("torch.sort", "radix sorted in O(N)", Alg. P:1786-1790,
// S:215-223): every run (chunk of M positions, or all N when non-causal) is
// sorted by (code, position).  Runs of <= SEG_SORT_MAX keys: one CTA owns one
// run (longer runs: the onesweep sort further down); keys and 16-bit local
// positions live in shared memory (ping-pong), 8-bit digits, and each pass
// is a stable counting sort built from warp-level __match_any_sync
// histograms: per warp a digit histogram (leader lane adds popc(peers)), a
// CTA-wide exclusive scan in (digit, warp) order, and a scatter whose rank
// is popc(peers & lanemask_lt).  Digits that are constant across the run
// (AND/OR reduction) are skipped, so only the varying bits of the codes
// cost a pass.  The backward transpose (A9) is in csr.cu.
#include "common.cuh"
#include "internal.h"

namespace onedf {

// ============================================================================ K3
constexpr int SEG_MAX_WARPS = 16;

// One CTA sorts one run of <= SEG_SORT_MAX keys: the run lives in shared
// memory with 16-bit local positions.  Longer runs go through the multi-CTA
// onesweep sort below.
__global__ void __launch_bounds__(SEG_MAX_WARPS * 32) seg_sort_kernel(
    const uint64_t* __restrict__ kcode, uint64_t* __restrict__ scode, int32_t* __restrict__ perm,
    int64_t N, int64_t M, int64_t runs_per_bh, Shard sh) {
    using Pos = uint16_t;
    extern __shared__ __align__(16) unsigned char smem[];
    const int64_t bh = blockIdx.x / runs_per_bh;
    const int64_t c = blockIdx.x % runs_per_bh;
    if (sh.on() && Shard::owner(c, sh.world) != sh.rank) return;   // sharded: other ranks' runs arrive by all-gather
    const int64_t s0 = c * M;
    const int n = (int)min64(M, N - s0);
    const int nw = blockDim.x / 32;
    const int nmax = (int)M;
    uint64_t* keys0 = reinterpret_cast<uint64_t*>(smem);
    uint64_t* keys1 = keys0 + nmax;
    const int npad = (nmax + 7) & ~7;       // keeps vals1 and hist 16-B aligned for odd run lengths
    Pos* vals0 = reinterpret_cast<Pos*>(keys1 + nmax);
    Pos* vals1 = vals0 + npad;
    uint32_t* hist = reinterpret_cast<uint32_t*>(vals1 + npad);   // [256][nw]
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

// ============================================================================ K3, long runs
// Onesweep LSD radix sort (decoupled look-back) for runs longer than SEG_SORT_MAX: every run is cut
// into tiles of OS_TILE keys and every CTA sorts one tile per 8-bit digit pass:
//   (0) one read of all keys: per-(run, pass) digit counts (integer atomics) -> exclusive digit
//       bases per run and pass;
//   per pass, one launch: the CTA takes the next tile ticket (tickets follow launch order, so a
//   tile's predecessors in its run have started -- the look-back cannot deadlock), ranks its keys
//   stably by digit in shared memory (per-warp __match_any_sync histograms, scan in (digit, warp)
//   order, as the on-chip sort), publishes its per-digit counts, looks back over the run's earlier
//   tiles for the exclusive prefix (aggregate / inclusive-prefix flags in one status word per
//   (run, tile, digit)), publishes its inclusive prefix and scatters to
//   base[digit] + prefix[digit] + rank within the tile.
// Stable (tile order = position order, then warp, then lane), all integer: bitwise the same
// permutation as the on-chip sort and std::sort on (code, position).
constexpr int OS_WARPS = 16;
constexpr int OS_THREADS = OS_WARPS * 32;
constexpr int OS_TILE = OS_THREADS * 8;       // 4096 keys per tile
constexpr uint32_t OS_FLAG_AGG = 1u << 30, OS_FLAG_INC = 2u << 30, OS_VAL = (1u << 30) - 1;

static int os_passes(const onedf_problem* p) { return (p->d_k * effective_bits(p) + 7) / 8; }
static int64_t os_tiles(const onedf_problem* p) { return (run_len_max(p) + OS_TILE - 1) / OS_TILE; }

void sort_carve(const onedf_problem* p, Carver* c, SortScratch* s) {
    const bool big = run_len_max(p) > SEG_SORT_MAX;
    const size_t n = big ? (size_t)(p->B * p->H * p->N) : 0;
    for (int b = 0; b < 2; ++b) {
        s->k[b] = big ? c->take<uint64_t>(n) : nullptr;
        s->v[b] = big ? c->take<uint32_t>(n) : nullptr;
    }
    const size_t runs = big ? (size_t)(p->B * p->H * num_runs(p)) : 0;
    s->base = big ? c->take<uint32_t>(runs * 8 * 256) : nullptr;
    s->status = big ? c->take<uint32_t>(runs * (size_t)os_tiles(p) * 256) : nullptr;
    s->ticket = big ? c->take<uint32_t>(8) : nullptr;
}

struct OsArgs {
    const uint64_t* kcode; uint64_t* scode; int32_t* perm;
    SortScratch scr;
    int64_t N, M, runs_per_bh, tiles;   // tiles per run (uniform; a short last run has empty tiles)
    Shard sh;                            // sharded: other ranks' runs arrive by all-gather (skipped)
};

// (0) digit counts of every pass, per run
__global__ void __launch_bounds__(OS_THREADS) os_hist_kernel(const OsArgs a, int passes) {
    __shared__ uint32_t h[8][256];
    for (int t = threadIdx.x; t < 8 * 256; t += OS_THREADS) (&h[0][0])[t] = 0;
    __syncthreads();
    const int64_t run = blockIdx.x / a.tiles, tile = blockIdx.x % a.tiles;
    const int64_t bh = run / a.runs_per_bh, c = run % a.runs_per_bh;
    if (a.sh.on() && Shard::owner(c, a.sh.world) != a.sh.rank) return;
    const int64_t s0 = c * a.M, n = min64(a.M, a.N - s0);
    const uint64_t* src = a.kcode + bh * a.N + s0;
    for (int64_t r = tile * OS_TILE + threadIdx.x; r < min64(n, (tile + 1) * OS_TILE); r += OS_THREADS) {
        const uint64_t k = src[r];
        for (int ps = 0; ps < passes; ++ps) atomicAdd(&h[ps][(k >> (8 * ps)) & 0xff], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < passes * 256; t += OS_THREADS) {
        const uint32_t v = (&h[0][0])[t];
        if (v) atomicAdd(a.scr.base + run * 8 * 256 + t, v);
    }
}

// counts -> exclusive digit bases, one warp per (run, pass): 8 digits per lane + a warp scan
__global__ void os_base_kernel(const OsArgs a, int64_t runs, int passes) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (t >= runs * passes) return;
    const int lane = lane_id();
    uint32_t* b = a.scr.base + (t / passes) * 8 * 256 + (t % passes) * 256 + lane * 8;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) { v[d] = b[d]; sum += v[d]; }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int d = 0; d < 8; ++d) { b[d] = run; run += v[d]; }
}

// one digit pass over one tile (the ticket decides which)
__global__ void __launch_bounds__(OS_THREADS) os_pass_kernel(const OsArgs a, int pass, int passes) {
    extern __shared__ __align__(16) unsigned char os_smem[];
    uint64_t* ks = reinterpret_cast<uint64_t*>(os_smem);          // [OS_TILE] the tile's keys
    uint32_t* vs = reinterpret_cast<uint32_t*>(ks + OS_TILE);     // [OS_TILE] their positions in the run
    __shared__ uint32_t hist[256 * OS_WARPS];
    __shared__ uint32_t adj[256];
    __shared__ uint32_t wsum[OS_WARPS];
    __shared__ uint32_t s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.scr.ticket + pass, 1u);
    __syncthreads();
    const int64_t tid = s_ticket;
    const int64_t run = tid / a.tiles, tile = tid % a.tiles;
    const int64_t bh = run / a.runs_per_bh, c = run % a.runs_per_bh;
    // sharded: the whole run is skipped (only later tiles of the same run look back at its tiles)
    if (a.sh.on() && Shard::owner(c, a.sh.world) != a.sh.rank) return;
    const int64_t s0 = c * a.M, n = min64(a.M, a.N - s0);
    const int64_t r0 = tile * OS_TILE;
    const int nt = (int)max((int64_t)0, min64(OS_TILE, n - r0));
    const int shift = 8 * pass;
    const int w = threadIdx.x / 32, lane = lane_id();
    const int64_t off = bh * a.N + s0 + r0;
    // load the tile: pass 0 from the codes (positions implicit), later passes from the ping-pong scratch
    const bool odd = pass & 1;                // ping-pong buffer of this pass (no dynamic indexing of the params)
    const uint64_t* ksrc = pass == 0 ? a.kcode + off : (odd ? a.scr.k[1] : a.scr.k[0]) + off;
    const uint32_t* vsrc = (odd ? a.scr.v[1] : a.scr.v[0]) + off;
    for (int r = threadIdx.x; r < nt; r += OS_THREADS) {
        ks[r] = ksrc[r];
        vs[r] = pass == 0 ? (uint32_t)(r0 + r) : vsrc[r];
    }
    for (int t = threadIdx.x; t < 256 * OS_WARPS; t += OS_THREADS) hist[t] = 0;
    __syncthreads();
    const int per_warp = OS_TILE / OS_WARPS;
    const int w0 = min(nt, w * per_warp), w1 = min(nt, w0 + per_warp);
    for (int b = w0; b < w1; b += 32) {                   // per-warp digit counts
        const int r = b + lane;
        const bool act = r < w1;
        const unsigned d = act ? (unsigned)((ks[r] >> shift) & 0xff) : 256u + lane;
        const unsigned peers = __match_any_sync(FULL, d);
        if (act && lane == __ffs(peers) - 1) hist[d * OS_WARPS + w] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // tile counts per digit: thread d (d < 256) publishes its aggregate, looks back, publishes inclusive
    uint32_t* st = a.scr.status + (run * a.tiles) * 256;
    if (threadIdx.x < 256) {
        const int d = threadIdx.x;
        uint32_t cnt = 0;
        for (int x = 0; x < OS_WARPS; ++x) cnt += hist[d * OS_WARPS + x];
        uint32_t excl = 0;
        if (tile == 0) {
            atomicExch(st + d, OS_FLAG_INC | cnt);
        } else {
            atomicExch(st + tile * 256 + d, OS_FLAG_AGG | cnt);
            for (int64_t t = tile - 1; t >= 0; --t) {
                uint32_t v;
                do { v = *(volatile uint32_t*)(st + t * 256 + d); } while ((v & ~OS_VAL) == 0);
                excl += v & OS_VAL;
                if ((v & ~OS_VAL) == OS_FLAG_INC) break;
            }
            atomicExch(st + tile * 256 + d, OS_FLAG_INC | (excl + cnt));
        }
        adj[d] = a.scr.base[run * 8 * 256 + pass * 256 + d] + excl;   // run base + earlier tiles
    }
    __syncthreads();
    // exclusive scan of hist in (digit, warp) order -> tile-local start of each (digit, warp)
    {
        const int total = 256 * OS_WARPS, per = total / OS_THREADS;
        const int a0 = threadIdx.x * per;
        uint32_t sum = 0;
        for (int t = a0; t < a0 + per; ++t) sum += hist[t];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        uint32_t woff = 0;
        for (int v = 0; v < w; ++v) woff += wsum[v];
        uint32_t runv = woff + incl - sum;
        for (int t = a0; t < a0 + per; ++t) { const uint32_t x = hist[t]; hist[t] = runv; runv += x; }
    }
    __syncthreads();
    // digit d's keys occupy tile-local slots from hist[d*W] (before the scatter advances it): the
    // global slot of tile-local slot x of digit d is adj[d] + x
    if (threadIdx.x < 256) adj[threadIdx.x] -= hist[threadIdx.x * OS_WARPS];
    __syncthreads();
    const bool last = pass == passes - 1;
    uint64_t* kdst = last ? (a.scode ? a.scode + bh * a.N + s0 : nullptr) : (odd ? a.scr.k[0] : a.scr.k[1]) + bh * a.N + s0;
    uint32_t* vdst = last ? nullptr : (odd ? a.scr.v[0] : a.scr.v[1]) + bh * a.N + s0;
    int32_t* pdst = a.perm + bh * a.N + s0;
    for (int b = w0; b < w1; b += 32) {
        const int r = b + lane;
        const bool act = r < w1;
        const uint64_t key = act ? ks[r] : 0;
        const unsigned d = act ? (unsigned)((key >> shift) & 0xff) : 256u + lane;
        const unsigned peers = __match_any_sync(FULL, d);
        if (act) {
            const uint32_t local = hist[d * OS_WARPS + w] + __popc(peers & lanemask_lt());
            const uint32_t dst = adj[d] + local;
            if (kdst) kdst[dst] = key;
            if (last) pdst[dst] = (int32_t)(s0 + (int64_t)vs[r]);
            else vdst[dst] = vs[r];
        }
        __syncwarp();
        if (act && lane == __ffs(peers) - 1) hist[d * OS_WARPS + w] += __popc(peers);
        __syncwarp();
    }
}

static cudaError_t launch_onesweep(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm,
                                   const SortScratch& scr, cudaStream_t st) {
    OsArgs a;
    a.kcode = kcode; a.scode = scode; a.perm = perm; a.scr = scr;
    a.N = p->N; a.M = run_len_max(p); a.runs_per_bh = num_runs(p); a.tiles = os_tiles(p);
    a.sh = make_shard(p);
    const int64_t runs = p->B * p->H * a.runs_per_bh;
    const int passes = os_passes(p);
    cudaError_t e = cudaMemsetAsync(scr.base, 0, (size_t)runs * 8 * 256 * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(scr.ticket, 0, 8 * 4, st);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)(runs * a.tiles);
    const size_t smem = (size_t)OS_TILE * 12;
    e = cudaFuncSetAttribute(os_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    os_hist_kernel<<<grid, OS_THREADS, 0, st>>>(a, passes);
    os_base_kernel<<<(unsigned)((runs * passes * 32 + 255) / 256), 256, 0, st>>>(a, runs, passes);
    for (int ps = 0; ps < passes; ++ps) {
        e = cudaMemsetAsync(scr.status, 0, (size_t)runs * a.tiles * 256 * 4, st);
        if (e != cudaSuccess) return e;
        os_pass_kernel<<<grid, OS_THREADS, smem, st>>>(a, ps, passes);
    }
    return cudaGetLastError();
}

cudaError_t launch_seg_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm,
                            const SortScratch& scr, cudaStream_t st) {
    const int64_t N = p->N, BH = p->B * p->H;
    const int64_t M = run_len_max(p);
    const int64_t runs = num_runs(p);
    if (M > SEG_SORT_MAX) return launch_onesweep(p, kcode, scode, perm, scr, st);
    int nw = (int)((M + 32 * 8 - 1) / (32 * 8));   // ~8 keys per lane
    nw = nw < 1 ? 1 : (nw > SEG_MAX_WARPS ? SEG_MAX_WARPS : nw);
    const size_t smem = seg_sort_smem(M, nw);
    cudaError_t e = cudaFuncSetAttribute(seg_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    seg_sort_kernel<<<(unsigned)(BH * runs), nw * 32, smem, st>>>(kcode, scode, perm, N, M, runs, make_shard(p));
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
