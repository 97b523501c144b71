// proj.cu -- NEXT-4: the upstream projections f_q, f_k and the
// Cauchy scale gamma^2 = sigma(theta) in front of the encoder (K2), and their
// backward.
//
// P:1549 "trainable projection networks f_k and f_q" map the d_model token
// features to the low d_K per head; read as one linear layer per head
// (reading D27): q_{b,h,n} = W_q[h] x_{b,n} + b_q[h], k likewise.
// "gamma^2 as the output of a sigmoid function applied to a trainable
// parameter": eps = sigma(theta).  Backward (chain rule):
//   dx_{b,n} = sum_h W_q[h]^T dq_{b,h,n} + W_k[h]^T dk_{b,h,n}
//   dW_q[h]  = sum_{b,n} dq_{b,h,n} x_{b,n}^T,   db_q[h] = sum_{b,n} dq_{b,h,n}
//   dtheta   = d_eps sigma(theta) (1 - sigma(theta)).
//
// All three contractions are tiny-output GEMMs (O = 2 H d_k = 72 columns at the
// bench shape) kept on the SIMT pipes in f64: exact f32 products, f64 sums in a
// fixed order, one rounding to f32 -- the projected coordinates feed the
// quantiser and the f32 ranking, so they are reproduced to the last bit by
// construction (tensor-core TF32/BF16 would round the inputs; DESIGN R6).
// Layouts: X, dX [B, N, d_model]; W, dW [H, d_k, d_model]; b, db [H, d_k];
// Q, K, dQ, dK [B, H, N, d_k].  Output column o < H d_k is q (h = o / d_k,
// d = o % d_k), o >= H d_k is k.
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int PJ_THREADS = 256;
constexpr int PJ_RT = 4;              // rows per thread
constexpr int PJ_CT = 9;              // output columns per thread
constexpr int PJ_ROWS = 32 * PJ_RT;   // rows per CTA (32 row groups)
constexpr int PJ_COLS = 8 * PJ_CT;    // output columns per CTA (8 column groups) = 72
constexpr int PJ_MC = 32;             // d_model slice staged per step

struct ProjArgs {
    const float* X; const float* Wq; const float* Wk; const float* bq; const float* bk; const float* theta;
    float* Q; float* K; float* eps;
    int64_t B, H, N; int dk, dm;
    void* ws;
};

__device__ __forceinline__ const float* w_row(const ProjArgs& a, int o) {
    const int hd = (int)a.H * a.dk;
    return (o < hd ? a.Wq : a.Wk) + (int64_t)(o < hd ? o : o - hd) * a.dm;
}

// Q, K (and eps = sigma(theta)).  CTA: PJ_ROWS rows (b, n) x PJ_COLS output columns; thread (ty, tx)
// owns rows ty + 32 i and columns tx + 8 c; the d_model axis is walked in slices of PJ_MC with
// x (f32) and w (widened to f64 once per CTA) staged in shared memory.
__global__ void __launch_bounds__(PJ_THREADS, 2) project_kernel(const ProjArgs a) {
    __shared__ float xs[PJ_ROWS][PJ_MC + 1];
    __shared__ double wsm[PJ_COLS][PJ_MC + 1];       // +1: the 8 column groups hit distinct banks
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;
    const int64_t rows = a.B * a.N;
    const int64_t r0 = (int64_t)blockIdx.x * PJ_ROWS;
    const int o0 = blockIdx.y * PJ_COLS;
    const int O = 2 * (int)a.H * a.dk;
    if (a.eps && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        const float th = __ldg(a.theta);
        if (!isfinite(th)) set_flag(a.ws, ONEDF_OP_ENCODE, FLAG_NONFINITE_INPUT);
        *a.eps = (float)(1.0 / (1.0 + exp(-(double)th)));
    }
    double acc[PJ_RT][PJ_CT];
#pragma unroll
    for (int i = 0; i < PJ_RT; ++i)
#pragma unroll
        for (int c = 0; c < PJ_CT; ++c) acc[i][c] = 0.0;
    for (int m0 = 0; m0 < a.dm; m0 += PJ_MC) {
        __syncthreads();
        for (int t = threadIdx.x; t < PJ_ROWS * PJ_MC; t += PJ_THREADS) {
            const int r = t / PJ_MC, m = t % PJ_MC;
            xs[r][m] = (r0 + r < rows && m0 + m < a.dm) ? __ldg(a.X + (r0 + r) * a.dm + m0 + m) : 0.f;
        }
        for (int t = threadIdx.x; t < PJ_COLS * PJ_MC; t += PJ_THREADS) {
            const int o = t / PJ_MC, m = t % PJ_MC;
            wsm[o][m] = (o0 + o < O && m0 + m < a.dm) ? (double)__ldg(w_row(a, o0 + o) + m0 + m) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int m = 0; m < PJ_MC; ++m) {
            double x[PJ_RT], w[PJ_CT];
#pragma unroll
            for (int i = 0; i < PJ_RT; ++i) x[i] = (double)xs[ty + 32 * i][m];
#pragma unroll
            for (int c = 0; c < PJ_CT; ++c) w[c] = wsm[tx + 8 * c][m];
#pragma unroll
            for (int i = 0; i < PJ_RT; ++i)
#pragma unroll
                for (int c = 0; c < PJ_CT; ++c) acc[i][c] = fma(x[i], w[c], acc[i][c]);
        }
    }
    const int hd = (int)a.H * a.dk;
#pragma unroll
    for (int i = 0; i < PJ_RT; ++i) {
        const int64_t r = r0 + ty + 32 * i;
        if (r >= rows) continue;
        const int64_t b = r / a.N, n = r % a.N;
#pragma unroll
        for (int c = 0; c < PJ_CT; ++c) {
            const int o = o0 + tx + 8 * c;
            if (o >= O) continue;
            const bool isq = o < hd;
            const int oo = isq ? o : o - hd;
            const int h = oo / a.dk, d = oo % a.dk;
            const float* bias = isq ? a.bq : a.bk;
            const double v = acc[i][c] + (bias ? (double)__ldg(bias + oo) : 0.0);
            (isq ? a.Q : a.K)[((b * a.H + h) * a.N + n) * a.dk + d] = (float)v;
        }
    }
}

// dX = sum_o dY[., o] W[o, .] with dY[(b,n), o] = dq_{b,h,n,d} / dk_{b,h,n,d}.  CTA: PJ_ROWS rows x
// 64 d_model columns; thread (ty, tx) owns rows ty + 32 i and columns tx + 8 c (c < 8); the O
// axis is walked in slices of PJB_OC with dY and W staged in shared memory as f64.
constexpr int PJB_OC = 24;
constexpr int PJB_MT = 64;

struct ProjBwdArgs {
    const float* X; const float* Wq; const float* Wk; const float* theta;
    const float* dQ; const float* dK; const double* d_eps;
    float* dX; double* part;          // part [G][O][d_model + 1]: per row-group dW | db partials
    float* dWq; float* dWk; float* dbq; float* dbk; float* dtheta;
    int64_t B, H, N; int dk, dm, G;
};

__device__ __forceinline__ float dy_value(const ProjBwdArgs& a, int64_t r, int o) {
    const int hd = (int)a.H * a.dk;
    const bool isq = o < hd;
    const int oo = isq ? o : o - hd;
    const int h = oo / a.dk, d = oo % a.dk;
    const int64_t b = r / a.N, n = r % a.N;
    return __ldg((isq ? a.dQ : a.dK) + ((b * a.H + h) * a.N + n) * a.dk + d);
}

__device__ __forceinline__ const float* w_row_b(const ProjBwdArgs& a, int o) {
    const int hd = (int)a.H * a.dk;
    return (o < hd ? a.Wq : a.Wk) + (int64_t)(o < hd ? o : o - hd) * a.dm;
}

__global__ void __launch_bounds__(PJ_THREADS, 2) project_dx_kernel(const ProjBwdArgs a) {
    __shared__ double ys[PJ_ROWS][PJB_OC + 1];
    __shared__ double wsm[PJB_OC][PJB_MT + 1];
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;
    const int64_t rows = a.B * a.N;
    const int64_t r0 = (int64_t)blockIdx.x * PJ_ROWS;
    const int m0 = blockIdx.y * PJB_MT;
    const int O = 2 * (int)a.H * a.dk;
    double acc[PJ_RT][8];
#pragma unroll
    for (int i = 0; i < PJ_RT; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[i][c] = 0.0;
    for (int oc = 0; oc < O; oc += PJB_OC) {
        __syncthreads();
        for (int t = threadIdx.x; t < PJ_ROWS * PJB_OC; t += PJ_THREADS) {
            const int r = t / PJB_OC, o = t % PJB_OC;
            ys[r][o] = (r0 + r < rows && oc + o < O) ? (double)dy_value(a, r0 + r, oc + o) : 0.0;
        }
        for (int t = threadIdx.x; t < PJB_OC * PJB_MT; t += PJ_THREADS) {
            const int o = t / PJB_MT, m = t % PJB_MT;
            wsm[o][m] = (oc + o < O && m0 + m < a.dm) ? (double)__ldg(w_row_b(a, oc + o) + m0 + m) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int o = 0; o < PJB_OC; ++o) {
            double y[PJ_RT], w[8];
#pragma unroll
            for (int i = 0; i < PJ_RT; ++i) y[i] = ys[ty + 32 * i][o];
#pragma unroll
            for (int c = 0; c < 8; ++c) w[c] = wsm[o][tx + 8 * c];
#pragma unroll
            for (int i = 0; i < PJ_RT; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[i][c] = fma(y[i], w[c], acc[i][c]);
        }
    }
#pragma unroll
    for (int i = 0; i < PJ_RT; ++i) {
        const int64_t r = r0 + ty + 32 * i;
        if (r >= rows) continue;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int m = m0 + tx + 8 * c;
            if (m < a.dm) a.dX[r * a.dm + m] = (float)acc[i][c];
        }
    }
}

// dW / db partials: row group g (a fixed contiguous range of the B*N rows, G groups whatever the
// device) x PJ_COLS output columns x 64 d_model columns; thread (to, tm) owns outputs to + 8 c and
// columns tm + 32 u (u < 2); rows are walked in slices of 32 in ascending order (fixed order).
// Column d_model of the partial holds db (the tm == 0 threads of the m-tile 0 CTAs).
__global__ void __launch_bounds__(PJ_THREADS) project_dw_partial_kernel(const ProjBwdArgs a) {
    __shared__ double ys[32][PJ_COLS + 1];
    __shared__ float xs[32][PJB_MT + 1];
    const int tm = threadIdx.x % 32, to = threadIdx.x / 32;    // 32 x 8
    const int64_t rows = a.B * a.N;
    const int g = blockIdx.x;
    const int64_t per = (rows + a.G - 1) / a.G;
    const int64_t ra = (int64_t)g * per, rb = min64(rows, ra + per);
    const int m0 = blockIdx.y * PJB_MT, o0 = blockIdx.z * PJ_COLS;
    const int O = 2 * (int)a.H * a.dk;
    const bool with_db = blockIdx.y == 0;
    double acc[PJ_CT][2], accb[PJ_CT];
#pragma unroll
    for (int c = 0; c < PJ_CT; ++c) { acc[c][0] = acc[c][1] = 0.0; accb[c] = 0.0; }
    for (int64_t s = ra; s < rb; s += 32) {
        __syncthreads();
        for (int t = threadIdx.x; t < 32 * PJ_COLS; t += PJ_THREADS) {
            const int r = t / PJ_COLS, o = t % PJ_COLS;
            ys[r][o] = (s + r < rb && o0 + o < O) ? (double)dy_value(a, s + r, o0 + o) : 0.0;
        }
        for (int t = threadIdx.x; t < 32 * PJB_MT; t += PJ_THREADS) {
            const int r = t / PJB_MT, m = t % PJB_MT;
            xs[r][m] = (s + r < rb && m0 + m < a.dm) ? __ldg(a.X + (s + r) * a.dm + m0 + m) : 0.f;
        }
        __syncthreads();
        for (int r = 0; r < 32; ++r) {
            const double x0 = (double)xs[r][tm], x1 = (double)xs[r][tm + 32];
#pragma unroll
            for (int c = 0; c < PJ_CT; ++c) {
                const double y = ys[r][to + 8 * c];
                acc[c][0] = fma(y, x0, acc[c][0]);
                acc[c][1] = fma(y, x1, acc[c][1]);
                accb[c] += y;
            }
        }
    }
    const int64_t stride = (int64_t)a.dm + 1;
#pragma unroll
    for (int c = 0; c < PJ_CT; ++c) {
        const int o = o0 + to + 8 * c;
        if (o >= O) continue;
        double* prow = a.part + ((int64_t)g * O + o) * stride;
        if (m0 + tm < a.dm) prow[m0 + tm] = acc[c][0];
        if (m0 + tm + 32 < a.dm) prow[m0 + tm + 32] = acc[c][1];
        if (with_db && tm == 0) prow[a.dm] = accb[c];
    }
}

// dW, db = the G row-group partials summed in group order; dtheta = d_eps sigma (1 - sigma).
__global__ void project_dw_reduce_kernel(const ProjBwdArgs a) {
    const int O = 2 * (int)a.H * a.dk;
    const int64_t stride = (int64_t)a.dm + 1;
    const int64_t total = (int64_t)O * stride;
    const int hd = (int)a.H * a.dk;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int o = (int)(t / stride), m = (int)(t % stride);
        double s = 0.0;
        for (int g = 0; g < a.G; ++g) s += a.part[((int64_t)g * O + o) * stride + m];
        const bool isq = o < hd;
        const int oo = isq ? o : o - hd;
        if (m < a.dm) (isq ? a.dWq : a.dWk)[(int64_t)oo * a.dm + m] = (float)s;
        else if (isq ? a.dbq : a.dbk) (isq ? a.dbq : a.dbk)[oo] = (float)s;
    }
    if (a.dtheta && blockIdx.x == 0 && threadIdx.x == 0) {
        const double sg = 1.0 / (1.0 + exp(-(double)__ldg(a.theta)));
        *a.dtheta = (float)(*a.d_eps * sg * (1.0 - sg));
    }
}

constexpr int PJ_GROUPS = 64;          // row groups of the dW reduction (fixed: deterministic everywhere)

size_t project_ws_bytes(const onedf_problem* p, int d_model, Carver* c) {
    const int64_t O = 2 * p->H * (int64_t)p->d_k;
    c->take<double>((size_t)(PJ_GROUPS * O * ((int64_t)d_model + 1)));
    return c->bytes();
}

cudaError_t launch_project(const onedf_problem* p, int d_model, const float* X, const float* Wq, const float* Wk,
                           const float* bq, const float* bk, const float* theta, float* Q, float* K, float* eps,
                           void* ws, cudaStream_t st) {
    ProjArgs a;
    a.X = X; a.Wq = Wq; a.Wk = Wk; a.bq = bq; a.bk = bk; a.theta = theta;
    a.Q = Q; a.K = K; a.eps = theta ? eps : nullptr;
    a.B = p->B; a.H = p->H; a.N = p->N; a.dk = p->d_k; a.dm = d_model; a.ws = ws;
    const int O = 2 * (int)p->H * p->d_k;
    const dim3 grid((unsigned)((p->B * p->N + PJ_ROWS - 1) / PJ_ROWS), (unsigned)((O + PJ_COLS - 1) / PJ_COLS));
    project_kernel<<<grid, PJ_THREADS, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_project_bwd(const onedf_problem* p, int d_model, const float* X, const float* Wq, const float* Wk,
                               const float* theta, const float* dQ, const float* dK, const double* d_eps, float* dX,
                               float* dWq, float* dWk, float* dbq, float* dbk, float* dtheta, void* ws,
                               cudaStream_t st) {
    ProjBwdArgs a;
    a.X = X; a.Wq = Wq; a.Wk = Wk; a.theta = theta; a.dQ = dQ; a.dK = dK; a.d_eps = d_eps;
    a.dX = dX; a.dWq = dWq; a.dWk = dWk; a.dbq = dbq; a.dbk = dbk; a.dtheta = (theta && d_eps) ? dtheta : nullptr;
    a.B = p->B; a.H = p->H; a.N = p->N; a.dk = p->d_k; a.dm = d_model; a.G = PJ_GROUPS;
    Carver c(ws);
    a.part = c.take<double>((size_t)(PJ_GROUPS * 2 * p->H * (int64_t)p->d_k * ((int64_t)d_model + 1)));
    const int O = 2 * (int)p->H * p->d_k;
    const int64_t rows = p->B * p->N;
    if (dX) {
        const dim3 gx((unsigned)((rows + PJ_ROWS - 1) / PJ_ROWS), (unsigned)((d_model + PJB_MT - 1) / PJB_MT));
        project_dx_kernel<<<gx, PJ_THREADS, 0, st>>>(a);
    }
    const dim3 gw((unsigned)PJ_GROUPS, (unsigned)((d_model + PJB_MT - 1) / PJB_MT), (unsigned)((O + PJ_COLS - 1) / PJ_COLS));
    project_dw_partial_kernel<<<gw, PJ_THREADS, 0, st>>>(a);
    project_dw_reduce_kernel<<<148, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace onedf
