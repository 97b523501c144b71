// encode.cu -- A1 bounds fit + A2 Morton encode (K1, K2).
//
// A1: per (b,h), per dim, lo = min over Q u K, hi = max; hi == lo widens by
//     +-0.5 ("min ... max ... in the dataset", D10).
// A2: g = clamp(floor(((x - lo)/(hi - lo)) * (2^b - 1)), 0, 2^b - 1) in f64
//     (op order of D9), code = Eq. 4 interleave: bit
//     plane MSB first, coordinate 0 first within a plane.
//
// Memory: both kernels stream Q and K once with 128-bit loads (4 rows of
// d_k floats = d_k float4 per thread); the fit is a 2-level min/max
// (partials per (bh, split) then a per-CTA re-reduction in the encoder), so
// the grid covers all 148 SMs even at B*H = 96.
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int ENC_THREADS = 256;
constexpr int ENC_ROWS = 4;   // rows per thread (one float4 per coordinate)

template <int DK>
__device__ __forceinline__ void load_rows4(const float* __restrict__ X, int64_t row0, int64_t nrows,
                                           bool vec_ok, float (&out)[ENC_ROWS][DK]) {
    if (vec_ok && nrows == ENC_ROWS) {
        const float4* src = reinterpret_cast<const float4*>(X + row0 * DK);
        float flat[ENC_ROWS * DK];
#pragma unroll
        for (int v = 0; v < DK; ++v) {
            float4 t = __ldg(src + v);
            flat[4 * v + 0] = t.x; flat[4 * v + 1] = t.y; flat[4 * v + 2] = t.z; flat[4 * v + 3] = t.w;
        }
#pragma unroll
        for (int r = 0; r < ENC_ROWS; ++r)
#pragma unroll
            for (int d = 0; d < DK; ++d) out[r][d] = flat[r * DK + d];
    } else {
#pragma unroll
        for (int r = 0; r < ENC_ROWS; ++r)
#pragma unroll
            for (int d = 0; d < DK; ++d) out[r][d] = r < nrows ? __ldg(X + (row0 + r) * DK + d) : 0.f;
    }
}

// ---------------------------------------------------------------- K1 partial bounds
template <int DK>
__global__ void __launch_bounds__(ENC_THREADS) bounds_partial_kernel(
    const float* __restrict__ Q, const float* __restrict__ K, int64_t N, int splits, bool vec_ok,
    float* __restrict__ part /* [BH][splits][2][DK] */, void* ws, Shard sh) {
    const int s = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int64_t groups = (N + ENC_ROWS - 1) / ENC_ROWS;
    const int64_t gper = (groups + splits - 1) / splits;
    const int64_t g0 = (int64_t)s * gper, g1 = min(groups, g0 + gper);
    float lo[DK], hi[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) { lo[d] = INFINITY; hi[d] = -INFINITY; }
    bool bad = false;
    for (int64_t g = g0 + threadIdx.x; g < g1; g += ENC_THREADS) {
        const int64_t row0 = bh * N + g * ENC_ROWS;
        const int64_t nrows = min64(ENC_ROWS, N - g * ENC_ROWS);
        float x[ENC_ROWS][DK];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            load_rows4<DK>(t == 0 ? Q : K, row0, nrows, vec_ok, x);
#pragma unroll
            for (int r = 0; r < ENC_ROWS; ++r) {
                if (r >= nrows) break;
                if (sh.on() && !sh.owns_row(g * ENC_ROWS + r)) continue;   // sharded: owned rows only
#pragma unroll
                for (int d = 0; d < DK; ++d) {
                    float v = x[r][d];
                    bad |= !isfinite(v);
                    lo[d] = fminf(lo[d], v);
                    hi[d] = fmaxf(hi[d], v);
                }
            }
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) set_flag(ws, ONEDF_OP_ENCODE, FLAG_NONFINITE_INPUT);
    __shared__ float red[2][DK][ENC_THREADS / 32];
#pragma unroll
    for (int d = 0; d < DK; ++d) {
        float a = lo[d], b = hi[d];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = fminf(a, __shfl_xor_sync(FULL, a, o));
            b = fmaxf(b, __shfl_xor_sync(FULL, b, o));
        }
        if (lane_id() == 0) { red[0][d][threadIdx.x / 32] = a; red[1][d][threadIdx.x / 32] = b; }
    }
    __syncthreads();
    if (threadIdx.x < DK) {
        const int d = threadIdx.x;
        float a = INFINITY, b = -INFINITY;
        for (int w = 0; w < ENC_THREADS / 32; ++w) { a = fminf(a, red[0][d][w]); b = fmaxf(b, red[1][d][w]); }
        float* out = part + ((bh * splits + s) * 2) * DK;
        out[d] = a;
        out[DK + d] = b;
    }
}

// ---------------------------------------------------------------- Morton spreads
__device__ __forceinline__ uint64_t spread1(uint64_t x) { return x; }
__device__ __forceinline__ uint64_t spread2(uint64_t x) {
    x &= 0xffffffffull;
    x = (x | (x << 16)) & 0x0000ffff0000ffffull;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}
__device__ __forceinline__ uint64_t spread3(uint64_t x) {
    x &= 0x1fffffull;
    x = (x | (x << 32)) & 0x001f00000000ffffull;
    x = (x | (x << 16)) & 0x001f0000ff0000ffull;
    x = (x | (x << 8)) & 0x100f00f00f00f00full;
    x = (x | (x << 4)) & 0x10c30c30c30c30c3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}
template <int DK>
__device__ __forceinline__ uint64_t spread(uint64_t x, int b) {
    if constexpr (DK == 1) return spread1(x);
    else if constexpr (DK == 2) return spread2(x);
    else if constexpr (DK == 3) return spread3(x);
    else {
        uint64_t out = 0;
        for (int t = 0; t < b; ++t) out |= ((x >> t) & 1ull) << (t * DK);
        return out;
    }
}

// Eq. 4: bit t of g_d lands at code bit t*DK + (DK-1-d).
template <int DK>
__device__ __forceinline__ uint64_t morton(const float* x, const double* lo, const double* hi, double top, int b) {
    uint64_t code = 0;
#pragma unroll
    for (int d = 0; d < DK; ++d) {
        double t = __ddiv_rn((double)x[d] - lo[d], hi[d] - lo[d]);
        double g = floor(__dmul_rn(t, top));
        g = g >= 0.0 ? g : 0.0;           // NaN -> 0 (no undefined cast; the input is flagged by K1)
        g = g > top ? top : g;
        code |= spread<DK>((uint64_t)g, b) << (DK - 1 - d);
    }
    return code;
}

// ---------------------------------------------------------------- K2 encode
template <int DK>
__global__ void __launch_bounds__(ENC_THREADS) encode_kernel(
    const float* __restrict__ Q, const float* __restrict__ K, int64_t N, int b, bool vec_ok,
    const float* __restrict__ part, int splits, const double* __restrict__ lohi_in,
    uint64_t* __restrict__ qcode, uint64_t* __restrict__ kcode, double* __restrict__ lohi_out,
    void* ws, Shard sh) {
    const int64_t bh = blockIdx.y;
    __shared__ double s_lo[DK], s_hi[DK];
    if (threadIdx.x < DK) {
        const int d = threadIdx.x;
        double lo, hi;
        if (lohi_in) {
            lo = lohi_in[bh * 2 * DK + d];
            hi = lohi_in[bh * 2 * DK + DK + d];
        } else {
            float a = INFINITY, c = -INFINITY;
            for (int s = 0; s < splits; ++s) {
                const float* pp = part + ((bh * splits + s) * 2) * DK;
                a = fminf(a, pp[d]);
                c = fmaxf(c, pp[DK + d]);
            }
            lo = a; hi = c;
            if (hi == lo) { lo -= 0.5; hi += 0.5; }
        }
        if (!isfinite(lo) || !isfinite(hi) || !(hi > lo)) set_flag(ws, ONEDF_OP_ENCODE, FLAG_NONFINITE_INPUT);
        s_lo[d] = lo; s_hi[d] = hi;
        if (lohi_out && blockIdx.x == 0) {
            lohi_out[bh * 2 * DK + d] = lo;
            lohi_out[bh * 2 * DK + DK + d] = hi;
        }
    }
    __syncthreads();
    double lo[DK], hi[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) { lo[d] = s_lo[d]; hi[d] = s_hi[d]; }
    const double top = (double)((1ull << b) - 1ull);
    const int64_t g = (int64_t)blockIdx.x * ENC_THREADS + threadIdx.x;
    if (g * ENC_ROWS >= N) return;
    // sharded: codes of other ranks' rows are never read (their runs arrive by all-gather)
    if (sh.on()) {
        bool any = false;
#pragma unroll
        for (int r = 0; r < ENC_ROWS; ++r) any |= g * ENC_ROWS + r < N && sh.owns_row(g * ENC_ROWS + r);
        if (!any) return;
    }
    const int64_t row0 = bh * N + g * ENC_ROWS;
    const int64_t nrows = min64(ENC_ROWS, N - g * ENC_ROWS);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        float x[ENC_ROWS][DK];
        load_rows4<DK>(t == 0 ? Q : K, row0, nrows, vec_ok, x);
        uint64_t c[ENC_ROWS];
#pragma unroll
        for (int r = 0; r < ENC_ROWS; ++r) c[r] = morton<DK>(x[r], lo, hi, top, b);
        uint64_t* out = (t == 0 ? qcode : kcode) + row0;
        if (nrows == ENC_ROWS && (((uintptr_t)out) & 15) == 0) {
            reinterpret_cast<ulonglong2*>(out)[0] = make_ulonglong2(c[0], c[1]);
            reinterpret_cast<ulonglong2*>(out)[1] = make_ulonglong2(c[2], c[3]);
        } else {
            for (int r = 0; r < nrows; ++r) out[r] = c[r];
        }
    }
}

static int bounds_splits(int64_t N, int64_t BH) {
    // enough CTAs to cover the chip a few times, each streaming >= 8K rows
    int64_t want = (4 * 148 + BH - 1) / BH;
    int64_t maxs = (N + 8191) / 8192;
    int64_t s = want < maxs ? want : maxs;
    return (int)(s < 1 ? 1 : (s > 64 ? 64 : s));
}

size_t encode_ws_bytes(const onedf_problem* p, Carver* c) {
    const int64_t BH = p->B * p->H;
    c->take<float>((size_t)BH * bounds_splits(p->N, BH) * 2 * p->d_k);
    return c->bytes();
}

cudaError_t launch_encode(const onedf_problem* p, int b, const float* Q, const float* K, const double* lohi_in,
                          uint64_t* qcode, uint64_t* kcode, double* lohi_out, void* ws, Carver* c,
                          cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int splits = bounds_splits(N, BH);
    float* part = c->take<float>((size_t)BH * splits * 2 * p->d_k);
    const bool vec_ok = ((N * p->d_k) % 4 == 0) && ((((uintptr_t)Q) | ((uintptr_t)K)) & 15) == 0;
    const int64_t groups = (N + ENC_ROWS - 1) / ENC_ROWS;
    dim3 egrid((unsigned)((groups + ENC_THREADS - 1) / ENC_THREADS), (unsigned)BH);
    ONEDF_DISPATCH_DK(p->d_k, {
        // always run: with caller-fixed bounds it is the finiteness check
        bounds_partial_kernel<DK><<<dim3(splits, (unsigned)BH), ENC_THREADS, 0, st>>>(Q, K, N, splits, vec_ok, part,
                                                                                      ws, make_shard(p));
        encode_kernel<DK><<<egrid, ENC_THREADS, 0, st>>>(Q, K, N, b, vec_ok, part, splits, lohi_in, qcode, kcode,
                                                         lohi_out, ws, make_shard(p));
    });
    return cudaGetLastError();
}

// ---------------------------------------------------------------- bounds-only entry points
// raw per-(b,h) per-dim min/max from the split partials (no widening)
__global__ void bounds_reduce_kernel(const float* __restrict__ part, int splits, int dk, double* __restrict__ lohi) {
    const int64_t bh = blockIdx.x;
    const int d = threadIdx.x;
    if (d >= dk) return;
    float a = INFINITY, c = -INFINITY;
    for (int s = 0; s < splits; ++s) {
        const float* pp = part + ((bh * splits + s) * 2) * dk;
        a = fminf(a, pp[d]);
        c = fmaxf(c, pp[dk + d]);
    }
    lohi[bh * 2 * dk + d] = a;
    lohi[bh * 2 * dk + dk + d] = c;
}

// D10: hi == lo widens by +-0.5 (the same rule encode_kernel applies when fitting)
__global__ void bounds_finish_kernel(double* __restrict__ lohi, int64_t BH, int dk, void* ws) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= BH * dk) return;
    const int64_t bh = t / dk;
    const int d = (int)(t % dk);
    double lo = lohi[bh * 2 * dk + d], hi = lohi[bh * 2 * dk + dk + d];
    if (hi == lo) { lo -= 0.5; hi += 0.5; }
    if (!isfinite(lo) || !isfinite(hi) || !(hi > lo)) set_flag(ws, ONEDF_OP_ENCODE, FLAG_NONFINITE_INPUT);
    lohi[bh * 2 * dk + d] = lo;
    lohi[bh * 2 * dk + dk + d] = hi;
}

cudaError_t launch_bounds_partial(const onedf_problem* p, const float* Q, const float* K, double* lohi, void* ws,
                                  Carver* c, cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int splits = bounds_splits(N, BH);
    float* part = c->take<float>((size_t)BH * splits * 2 * p->d_k);
    const bool vec_ok = ((N * p->d_k) % 4 == 0) && ((((uintptr_t)Q) | ((uintptr_t)K)) & 15) == 0;
    ONEDF_DISPATCH_DK(p->d_k, {
        bounds_partial_kernel<DK><<<dim3(splits, (unsigned)BH), ENC_THREADS, 0, st>>>(Q, K, N, splits, vec_ok, part,
                                                                                      ws, make_shard(p));
    });
    bounds_reduce_kernel<<<(unsigned)BH, 32, 0, st>>>(part, splits, p->d_k, lohi);
    return cudaGetLastError();
}

cudaError_t launch_bounds_finish(const onedf_problem* p, double* lohi, void* ws, cudaStream_t st) {
    const int64_t n = p->B * p->H * p->d_k;
    bounds_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(lohi, p->B * p->H, p->d_k, ws);
    return cudaGetLastError();
}

// Fixed-order combine of per-rank partials: f64 sum in rank order, one f32 rounding.
__global__ void rank_sum_kernel(const float* __restrict__ parts, int64_t n, int32_t world, float* __restrict__ out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int32_t r = 0; r < world; ++r) acc += (double)__ldg(parts + (int64_t)r * n + x);
        out[x] = (float)acc;
    }
}

cudaError_t launch_rank_sum(const float* parts, int64_t n, int32_t world, float* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = min64((n + 255) / 256, 148 * 16);
    rank_sum_kernel<<<(unsigned)blocks, 256, 0, st>>>(parts, n, world, out);
    return cudaGetLastError();
}

}  // namespace onedf
