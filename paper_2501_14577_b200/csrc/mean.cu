// mean.cu -- A4 prefix means of the mean slot (K5) and A11 the mean-slot
// chain rule as a reverse scan (K10).
//
// A4 ("append the mean vector of the history tokens ... using cumsum",
// reading D8): Kbar_i = (1/(i+1)) sum_{t<=i} K_t and the same for
// V (causal), or the mean over all N (non-causal).  f64 accumulation, f32
// store.  A11 (S:323(a)): dK_t += sum_{i>=t} dKbar_i/(i+1), dV_t likewise,
// with dKbar_i = w_mu,i (q_i - Kbar_i) and dVbar_i = A_mu,i dO_i emitted by
// the backward query pass (non-causal: (1/N) sum over all i).
//
// One column-scan engine serves both, per matrix [B*H][N][C] (C = d_k or
// d_v): tiles of SCAN_TB rows x C columns; a 256-thread CTA maps thread
// (g, c) to column c of row-group g (CW = pow2 >= C columns, RG = 256/CW
// row-groups of SCAN_TB/RG consecutive rows), so each warp access to a row
// is one coalesced line.  Three launches with a FIXED combination order:
// (1) tile sums (rows of a row-group sequential, row-groups in order),
// (2) exclusive scan over tiles per column, (3) apply: each thread re-walks
// its rows from (tile prefix + earlier row-groups) and writes the running
// value.  Deterministic; the tile is L1-resident for the second walk.
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int SCAN_TB = 256;        // rows per tile
constexpr int SCAN_THREADS = 256;

static int64_t scan_tiles(const onedf_problem* p) { return (p->N + SCAN_TB - 1) / SCAN_TB; }

void mean_carve(const onedf_problem* p, Carver* c, MeanBufs* m) {
    const int64_t BH = p->B * p->H;
    const int64_t rows = p->causal ? p->N : 1;
    m->Kbar = c->take<float>((size_t)(BH * rows * p->d_k));
    m->Vbar = c->take<float>((size_t)(BH * rows * p->d_v));
    m->part = c->take<double>((size_t)(BH * (scan_tiles(p) + 1) * (p->d_k + p->d_v)));
}

static int pow2_at_least(int c) {
    int w = 1;
    while (w < c) w <<= 1;
    return w;
}

// Value of row i, column c of the scanned matrix.
//   MODE 0 (A4):  X[i][c]                                 (K or V itself)
//   MODE 1 (A11, K columns): w_mu,i (q_i[c] - Kbar_i[c]) * s_i
//   MODE 2 (A11, V columns): A_mu,i dO_i[c] * s_i        s_i = 1/(i+1) causal, 1 otherwise
struct ScanSrc {
    const void* X;        // MODE 0: K or V; MODE 1: Q; MODE 2: dO -- element type TX of the kernel
    const float* Kbar;    // MODE 1
    const float2* muco;   // MODE 1, 2
    int C, causal;
    double kt = 1.0;      // MODE 1: w (q - kt Kbar); 0 for the DOT score (dKbar = w q)
};

// X[e] widened to f64; TX = float, or bf16 for the value rows of a BF16 problem (reading D26)
template <typename TX>
__device__ __forceinline__ double xval(const ScanSrc& s, int64_t e) {
    return (double)ld1(static_cast<const TX*>(s.X), e);
}

// inv = 1/(i+1) for the causal scans (A11's weights), from the tile's table; 1 otherwise
template <int MODE, typename TX>
__device__ __forceinline__ double scan_value(const ScanSrc& s, int64_t bh, int64_t N, int64_t i, int c, double inv) {
    const int64_t row = bh * N + i;
    if (MODE == 0) return xval<TX>(s, row * s.C + c);
    const float2 mc = __ldg(s.muco + row);
    double y;
    if (MODE == 1) {
        if (mc.y == 0.f) return 0.0;      // no mean-slot weight (e.g. another rank's query: Kbar unwritten)
        const float kb = __ldg(s.Kbar + (bh * (s.causal ? N : 1) + (s.causal ? i : 0)) * s.C + c);
        y = (double)mc.y * (xval<TX>(s, row * s.C + c) - s.kt * (double)kb);
    } else {
        y = (double)mc.x * xval<TX>(s, row * s.C + c);
    }
    return s.causal ? y * inv : y;
}

constexpr int SCAN_UNROLL = 8;        // rows loaded ahead per thread (independent loads in flight)

// 1/(r+1) for the tile's rows, once per CTA (the divisor is shared by every column)
__device__ __forceinline__ void fill_inv(double* s_inv, int64_t tile) {
    for (int t = threadIdx.x; t < SCAN_TB; t += blockDim.x) s_inv[t] = 1.0 / (double)(tile * SCAN_TB + t + 1);
}

// sum of the thread's rows [r0, r1), loads batched SCAN_UNROLL at a time, fixed order
template <int MODE, typename TX>
__device__ __forceinline__ double rows_sum(const ScanSrc& s, int64_t bh, int64_t N, int64_t r0, int64_t r1, int c,
                                           const double* s_inv, int64_t tbase) {
    double acc = 0.0;
    int64_t r = r0;
    for (; r + SCAN_UNROLL <= r1; r += SCAN_UNROLL) {
        double v[SCAN_UNROLL];
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) v[u] = scan_value<MODE, TX>(s, bh, N, r + u, c, s_inv[r + u - tbase]);
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) acc += v[u];
    }
    for (; r < r1; ++r) acc += scan_value<MODE, TX>(s, bh, N, r, c, s_inv[r - tbase]);
    return acc;
}

// (1) tile sums -> part[bh][tile][c]
template <int MODE, typename TX>
__global__ void __launch_bounds__(SCAN_THREADS) scan_tile_sums_kernel(const ScanSrc s, int64_t N, int64_t ntile,
                                                                      int CW, double* __restrict__ part) {
    __shared__ double sh[SCAN_THREADS];
    __shared__ double s_inv[SCAN_TB];
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    const int c = threadIdx.x % CW, g = threadIdx.x / CW, RG = SCAN_THREADS / CW;
    const int per = SCAN_TB / RG;
    const int64_t r0 = tile * SCAN_TB + (int64_t)g * per, r1 = min64(N, r0 + per);
    if (MODE != 0) {
        fill_inv(s_inv, tile);
        __syncthreads();
    }
    double acc = 0.0;
    if (c < s.C) acc = rows_sum<MODE, TX>(s, bh, N, r0, r1, c, s_inv, tile * SCAN_TB);
    sh[threadIdx.x] = acc;
    __syncthreads();
    if (g == 0 && c < s.C) {
        double t = 0.0;
        for (int x = 0; x < RG; ++x) t += sh[x * CW + c];
        part[(bh * (ntile + 1) + tile) * s.C + c] = t;
    }
}

// (2) per (bh, column): exclusive scan over tiles (forward) or suffix scan
// (reverse); part[ntile] = total.  One CTA per (bh, column): every thread sums a
// contiguous stretch of tiles, a fixed warp/CTA scan combines the stretches, then
// every thread rewrites its stretch -- a fixed combination order (deterministic),
// and no serial walk over the ntile = N/256 tiles of a long sequence.
constexpr int TSCAN_THREADS = 256;
__global__ void __launch_bounds__(TSCAN_THREADS) scan_tiles_kernel(double* __restrict__ part, int64_t ntile, int C,
                                                                   int reverse) {
    __shared__ double s_w[TSCAN_THREADS / 32];
    const int64_t bh = blockIdx.x;
    const int c = blockIdx.y;
    const int64_t per = (ntile + TSCAN_THREADS - 1) / TSCAN_THREADS;
    const int64_t u0 = min64(ntile, (int64_t)threadIdx.x * per), u1 = min64(ntile, u0 + per);
    auto at = [&](int64_t u) -> double* {                 // u-th tile in scan order
        const int64_t b = reverse ? ntile - 1 - u : u;
        return part + (bh * (ntile + 1) + b) * C + c;
    };
    double sum = 0.0;
    for (int64_t u = u0; u < u1; ++u) sum += *at(u);
    const int lane = lane_id(), w = threadIdx.x / 32;
    double inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    double woff = 0.0;
    for (int x = 0; x < w; ++x) woff += s_w[x];
    double run = woff + (inc - sum);                       // exclusive prefix of this stretch
    if (threadIdx.x == TSCAN_THREADS - 1) part[(bh * (ntile + 1) + ntile) * C + c] = woff + inc;
    for (int64_t u = u0; u < u1; ++u) {
        double* x = at(u);
        const double t = *x;
        *x = run;
        run += t;
    }
}

// (3a) A4 apply: out[i] = (prefix through i) / (i + 1)  (causal only)
template <typename TX>
__global__ void __launch_bounds__(SCAN_THREADS) mean_apply_kernel(const ScanSrc s, int64_t N, int64_t ntile, int CW,
                                                                  const double* __restrict__ part,
                                                                  float* __restrict__ out, Shard shd) {
    __shared__ double sh[SCAN_THREADS];
    __shared__ double s_inv[SCAN_TB];
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    // sharded: the means are read only at this rank's query rows -- skip tiles with none of them
    if (shd.on()) {
        const int64_t r0 = tile * SCAN_TB, r1 = min64(N, r0 + SCAN_TB) - 1;
        bool any = false;
        for (int64_t c = r0 / shd.M; c <= r1 / shd.M && !any; ++c) any = Shard::owner(c, shd.world) == shd.rank;
        if (!any) return;
    }
    const int c = threadIdx.x % CW, g = threadIdx.x / CW, RG = SCAN_THREADS / CW;
    const int per = SCAN_TB / RG;
    const int64_t r0 = tile * SCAN_TB + (int64_t)g * per, r1 = min64(N, r0 + per);
    const int64_t tb = tile * SCAN_TB;
    fill_inv(s_inv, tile);
    const bool on = c < s.C;
    double own = 0.0;
    if (on) own = rows_sum<0, TX>(s, bh, N, r0, r1, c, s_inv, tb);
    sh[threadIdx.x] = own;
    __syncthreads();
    if (!on) return;
    double run = part[(bh * (ntile + 1) + tile) * s.C + c];
    for (int x = 0; x < g; ++x) run += sh[x * CW + c];
    int64_t r = r0;
    for (; r + SCAN_UNROLL <= r1; r += SCAN_UNROLL) {
        double v[SCAN_UNROLL];
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) v[u] = scan_value<0, TX>(s, bh, N, r + u, c, 1.0);
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) {
            run += v[u];
            out[(bh * N + r + u) * s.C + c] = (float)(run * s_inv[r + u - tb]);
        }
    }
    for (; r < r1; ++r) {
        run += scan_value<0, TX>(s, bh, N, r, c, 1.0);
        out[(bh * N + r) * s.C + c] = (float)(run * s_inv[r - tb]);
    }
}

__global__ void mean_global_kernel(const double* __restrict__ part, int64_t ntile, int C, int64_t N,
                                   float* __restrict__ out) {
    const int64_t bh = blockIdx.x;
    for (int c = threadIdx.x; c < C; c += blockDim.x)
        out[bh * C + c] = (float)(part[(bh * (ntile + 1) + ntile) * C + c] / (double)N);
}

// (3b) A11 apply: out[t] = D[t] + sum_{i >= t} y_i (causal, reverse walk) or
// out[t] = D[t] + (1/N) sum_i y_i (non-causal).  D is the key side's f32 result;
// out is D itself (float rows) or the bf16 dV of a BF16 problem (one rounding).
template <int MODE, typename TX, typename TO>
__global__ void __launch_bounds__(SCAN_THREADS) grad_apply_kernel(const ScanSrc s, int64_t N, int64_t ntile, int CW,
                                                                  const double* __restrict__ part,
                                                                  const float* D, TO* out) {
    __shared__ double sh[SCAN_THREADS];
    __shared__ double s_inv[SCAN_TB];
    const int64_t bh = blockIdx.y, tile = blockIdx.x;
    const int c = threadIdx.x % CW, g = threadIdx.x / CW, RG = SCAN_THREADS / CW;
    const int per = SCAN_TB / RG;
    const int64_t r0 = tile * SCAN_TB + (int64_t)g * per, r1 = min64(N, r0 + per);
    const int64_t tb = tile * SCAN_TB;
    const bool on = c < s.C;
    if (!s.causal) {
        if (!on) return;
        const double add = part[(bh * (ntile + 1) + ntile) * s.C + c] / (double)N;
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t e = (bh * N + r) * s.C + c;
            st1(out, e, (double)D[e] + add);
        }
        return;
    }
    fill_inv(s_inv, tile);
    __syncthreads();
    double own = 0.0;
    if (on) own = rows_sum<MODE, TX>(s, bh, N, r0, r1, c, s_inv, tb);
    sh[threadIdx.x] = own;
    __syncthreads();
    if (!on) return;
    double run = part[(bh * (ntile + 1) + tile) * s.C + c];    // sum over later tiles
    for (int x = RG - 1; x > g; --x) run += sh[x * CW + c];      // later row-groups of this tile
    int64_t r = r1 - 1;
    for (; r - SCAN_UNROLL + 1 >= r0; r -= SCAN_UNROLL) {
        double v[SCAN_UNROLL];
        float d[SCAN_UNROLL];
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) {
            v[u] = scan_value<MODE, TX>(s, bh, N, r - u, c, s_inv[r - u - tb]);
            d[u] = D[(bh * N + r - u) * s.C + c];
        }
#pragma unroll
        for (int u = 0; u < SCAN_UNROLL; ++u) {
            run += v[u];
            st1(out, (bh * N + r - u) * s.C + c, (double)d[u] + run);
        }
    }
    for (; r >= r0; --r) {
        run += scan_value<MODE, TX>(s, bh, N, r, c, s_inv[r - tb]);
        const int64_t e = (bh * N + r) * s.C + c;
        st1(out, e, (double)D[e] + run);
    }
}

cudaError_t launch_prefix_means(const onedf_problem* p, const float* K, const void* V, MeanBufs* m,
                                cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N, nt = scan_tiles(p);
    const dim3 grid((unsigned)nt, (unsigned)BH);
    double* partK = m->part;
    double* partV = m->part + BH * (nt + 1) * p->d_k;
    const ScanSrc sk{K, nullptr, nullptr, p->d_k, p->causal};
    const ScanSrc sv{V, nullptr, nullptr, p->d_v, p->causal};
    const int cwk = pow2_at_least(p->d_k), cwv = pow2_at_least(p->d_v);
    scan_tile_sums_kernel<0, float><<<grid, SCAN_THREADS, 0, st>>>(sk, N, nt, cwk, partK);
    ONEDF_DISPATCH_TV(p->vdtype, { scan_tile_sums_kernel<0, TV><<<grid, SCAN_THREADS, 0, st>>>(sv, N, nt, cwv, partV); });
    scan_tiles_kernel<<<dim3((unsigned)BH, (unsigned)p->d_k), TSCAN_THREADS, 0, st>>>(partK, nt, p->d_k, 0);
    scan_tiles_kernel<<<dim3((unsigned)BH, (unsigned)p->d_v), TSCAN_THREADS, 0, st>>>(partV, nt, p->d_v, 0);
    if (p->causal) {
        const Shard shd = make_shard(p);
        mean_apply_kernel<float><<<grid, SCAN_THREADS, 0, st>>>(sk, N, nt, cwk, partK, m->Kbar, shd);
        ONEDF_DISPATCH_TV(p->vdtype, {
            mean_apply_kernel<TV><<<grid, SCAN_THREADS, 0, st>>>(sv, N, nt, cwv, partV, m->Vbar, shd);
        });
    } else {
        mean_global_kernel<<<(unsigned)BH, 32, 0, st>>>(partK, nt, p->d_k, N, m->Kbar);
        mean_global_kernel<<<(unsigned)BH, 256, 0, st>>>(partV, nt, p->d_v, N, m->Vbar);
    }
    return cudaGetLastError();
}

cudaError_t launch_mean_grad_scan(const onedf_problem* p, const float* Q, const void* dO, const float* muco,
                                  MeanBufs* m, float* dK, const float* dV32, void* dV, cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N, nt = scan_tiles(p);
    const dim3 grid((unsigned)nt, (unsigned)BH);
    const float2* mc = reinterpret_cast<const float2*>(muco);
    double* partK = m->part;
    double* partV = m->part + BH * (nt + 1) * p->d_k;
    const ScanSrc sk{Q, m->Kbar, mc, p->d_k, p->causal, p->score == SC_DOT ? 0.0 : 1.0};
    const ScanSrc sv{dO, nullptr, mc, p->d_v, p->causal};
    const int cwk = pow2_at_least(p->d_k), cwv = pow2_at_least(p->d_v);
    scan_tile_sums_kernel<1, float><<<grid, SCAN_THREADS, 0, st>>>(sk, N, nt, cwk, partK);
    ONEDF_DISPATCH_TV(p->vdtype, { scan_tile_sums_kernel<2, TV><<<grid, SCAN_THREADS, 0, st>>>(sv, N, nt, cwv, partV); });
    scan_tiles_kernel<<<dim3((unsigned)BH, (unsigned)p->d_k), TSCAN_THREADS, 0, st>>>(partK, nt, p->d_k, 1);
    scan_tiles_kernel<<<dim3((unsigned)BH, (unsigned)p->d_v), TSCAN_THREADS, 0, st>>>(partV, nt, p->d_v, 1);
    grad_apply_kernel<1, float, float><<<grid, SCAN_THREADS, 0, st>>>(sk, N, nt, cwk, partK, dK, dK);
    ONEDF_DISPATCH_TV(p->vdtype, {
        grad_apply_kernel<2, TV, TV><<<grid, SCAN_THREADS, 0, st>>>(sv, N, nt, cwv, partV, dV32, static_cast<TV*>(dV));
    });
    return cudaGetLastError();
}

// bf16 dV without the mean slot: one rounding of the key side's f32 rows
__global__ void round_rows_kernel(const float* __restrict__ src, bf16* __restrict__ dst, int64_t n4) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n4) return;
    const float4 x = __ldg(reinterpret_cast<const float4*>(src) + t);
    st4(dst, t, x.x, x.y, x.z, x.w);
}

cudaError_t launch_round_rows(const float* src, bf16* dst, int64_t n, cudaStream_t st) {
    const int64_t n4 = n / 4;
    if (n4 > 0) round_rows_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(src, dst, n4);
    return cudaGetLastError();
}

}  // namespace onedf
