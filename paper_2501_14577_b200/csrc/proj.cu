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

// dX = sum_o dY[., o] W[o, .] with dY[(b,n), o] = dq_{b,h,n,d} / dk_{b,h,n,d}.  CTA: PJ_ROWS rows;
// thread (ty, tx) owns rows ty + 32 i and, per d_model tile of PJB_MT, columns tx + 8 c (c < 8).
constexpr int PJB_MT = 64;

struct ProjBwdArgs {
    const float* X; const float* Wq; const float* Wk; const float* theta;
    const float* dQ; const float* dK; const double* d_eps;
    float* dX; double* part;          // part [G][O][d_model + 1]: per row-group dW | db partials
    float* dWq; float* dWk; float* dbq; float* dbk; float* dtheta;
    int64_t B, H, N; int dk, dm, G;
};

// dY column o (a q or k coordinate (h, d)) as a base pointer: dY[r][o] = col[o][rowoff(r)], with
// rowoff(b, n) = (b H N + n) d_k -- the 64-bit index split once per column and once per row, so the
// staging loops do no division.
__device__ __forceinline__ const float* dy_col(const ProjBwdArgs& a, int o) {
    const int hd = (int)a.H * a.dk;
    const bool isq = o < hd;
    const int oo = isq ? o : o - hd;
    return (isq ? a.dQ : a.dK) + ((int64_t)(oo / a.dk) * a.N) * a.dk + oo % a.dk;
}
__device__ __forceinline__ int64_t dy_rowoff(const ProjBwdArgs& a, int64_t r) {
    return ((r / a.N) * a.H * a.N + r % a.N) * a.dk;
}

__device__ __forceinline__ const float* w_row_b(const ProjBwdArgs& a, int o) {
    const int hd = (int)a.H * a.dk;
    return (o < hd ? a.Wq : a.Wk) + (int64_t)(o < hd ? o : o - hd) * a.dm;
}

// dX: the CTA stages its rows' whole dY tile [PJ_ROWS x O] once (f64, dynamic shared memory) and
// walks d_model in tiles of PJB_MT columns, staging W[:, tile] for each.
__global__ void __launch_bounds__(PJ_THREADS, 2) project_dx_kernel(const ProjBwdArgs a) {
    extern __shared__ double dsm[];
    const int O = 2 * (int)a.H * a.dk;
    const int OS = O + 1;                                   // row stride of ys (odd: no bank conflicts)
    double* ys = dsm;                                       // [PJ_ROWS][OS]
    double* wsm = dsm + PJ_ROWS * OS;                       // [O][PJB_MT + 1]
    __shared__ int64_t s_row[PJ_ROWS];
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;
    const int64_t rows = a.B * a.N;
    const int64_t r0 = (int64_t)blockIdx.x * PJ_ROWS;
    for (int r = threadIdx.x; r < PJ_ROWS; r += PJ_THREADS) s_row[r] = r0 + r < rows ? dy_rowoff(a, r0 + r) : -1;
    __syncthreads();
    for (int o = threadIdx.x / 32; o < O; o += PJ_THREADS / 32) {           // a warp per column
        const float* col = dy_col(a, o);
        for (int r = threadIdx.x % 32; r < PJ_ROWS; r += 32)
            ys[r * OS + o] = s_row[r] >= 0 ? (double)__ldg(col + s_row[r]) : 0.0;
    }
    for (int m0 = 0; m0 < a.dm; m0 += PJB_MT) {
        __syncthreads();
        for (int t = threadIdx.x; t < O * PJB_MT; t += PJ_THREADS) {
            const int o = t / PJB_MT, m = t % PJB_MT;
            wsm[o * (PJB_MT + 1) + m] = m0 + m < a.dm ? (double)__ldg(w_row_b(a, o) + m0 + m) : 0.0;
        }
        __syncthreads();
        double acc[PJ_RT][8];
#pragma unroll
        for (int i = 0; i < PJ_RT; ++i)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[i][c] = 0.0;
#pragma unroll 4
        for (int o = 0; o < O; ++o) {
            double y[PJ_RT], w[8];
#pragma unroll
            for (int i = 0; i < PJ_RT; ++i) y[i] = ys[(ty + 32 * i) * OS + o];
#pragma unroll
            for (int c = 0; c < 8; ++c) w[c] = wsm[o * (PJB_MT + 1) + tx + 8 * c];
#pragma unroll
            for (int i = 0; i < PJ_RT; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[i][c] = fma(y[i], w[c], acc[i][c]);
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
}

static size_t dx_smem(int O) { return sizeof(double) * ((size_t)PJ_ROWS * (O + 1) + (size_t)O * (PJB_MT + 1)); }

// dW partials: row group g (a fixed contiguous range of the B*N rows, G groups whatever the device)
// x PJ_COLS output columns x PJW_MT d_model columns; thread (to, tm) owns outputs to + 8 c (c < 9)
// and columns tm + 32 u (u < 4); rows are walked in slices of 32 in ascending order (fixed order).
// The m-tile 0 CTAs also sum db (column d_model of the partial rows).
constexpr int PJW_MT = 128;
__global__ void __launch_bounds__(PJ_THREADS, 2) project_dw_partial_kernel(const ProjBwdArgs a) {
    __shared__ double ys[32][PJ_COLS + 1];
    __shared__ float xs[32][PJW_MT + 4];
    __shared__ int64_t s_row[32];
    __shared__ const float* s_col[PJ_COLS];
    const int tm = threadIdx.x % 32, to = threadIdx.x / 32;    // 32 x 8
    const int64_t rows = a.B * a.N;
    const int g = blockIdx.x;
    const int64_t per = (rows + a.G - 1) / a.G;
    const int64_t ra = (int64_t)g * per, rb = min64(rows, ra + per);
    const int m0 = blockIdx.y * PJW_MT, o0 = blockIdx.z * PJ_COLS;
    const int O = 2 * (int)a.H * a.dk;
    for (int o = threadIdx.x; o < PJ_COLS; o += PJ_THREADS) s_col[o] = o0 + o < O ? dy_col(a, o0 + o) : nullptr;
    const bool with_db = blockIdx.y == 0 && threadIdx.x < PJ_COLS;
    double dbacc = 0.0;                             // thread t < PJ_COLS: db of column o0 + t
    double acc[PJ_CT][4];
#pragma unroll
    for (int c = 0; c < PJ_CT; ++c)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[c][u] = 0.0;
    for (int64_t s = ra; s < rb; s += 32) {
        __syncthreads();
        if (threadIdx.x < 32) s_row[threadIdx.x] = s + threadIdx.x < rb ? dy_rowoff(a, s + threadIdx.x) : -1;
        for (int t = threadIdx.x; t < 32 * PJW_MT; t += PJ_THREADS) {
            const int r = t / PJW_MT, m = t % PJW_MT;
            xs[r][m] = (s + r < rb && m0 + m < a.dm) ? __ldg(a.X + (s + r) * a.dm + m0 + m) : 0.f;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < 32 * PJ_COLS; t += PJ_THREADS) {
            const int r = t / PJ_COLS, o = t % PJ_COLS;
            const float* col = s_col[o];
            ys[r][o] = (s_row[r] >= 0 && col) ? (double)__ldg(col + s_row[r]) : 0.0;
        }
        __syncthreads();
        if (with_db)
            for (int r = 0; r < 32; ++r) dbacc += ys[r][threadIdx.x];
#pragma unroll 2
        for (int r = 0; r < 32; ++r) {
            double x[4], y[PJ_CT];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = (double)xs[r][tm + 32 * u];
#pragma unroll
            for (int c = 0; c < PJ_CT; ++c) y[c] = ys[r][to + 8 * c];
#pragma unroll
            for (int c = 0; c < PJ_CT; ++c)
#pragma unroll
                for (int u = 0; u < 4; ++u) acc[c][u] = fma(y[c], x[u], acc[c][u]);
        }
    }
    const int64_t stride = (int64_t)a.dm + 1;
#pragma unroll
    for (int c = 0; c < PJ_CT; ++c) {
        const int o = o0 + to + 8 * c;
        if (o >= O) continue;
        double* prow = a.part + ((int64_t)g * O + o) * stride;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (m0 + tm + 32 * u < a.dm) prow[m0 + tm + 32 * u] = acc[c][u];
    }
    if (with_db && o0 + (int)threadIdx.x < O) a.part[((int64_t)g * O + o0 + threadIdx.x) * stride + a.dm] = dbacc;
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

constexpr int PJ_GROUPS = 148;         // row groups of the dW reduction (fixed: deterministic on any device)

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
        const size_t smem = dx_smem(O);
        if (smem > 200 * 1024) return cudaErrorNotSupported;                  // O <= ~130 (validated)
        cudaError_t e = cudaFuncSetAttribute(project_dx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        project_dx_kernel<<<(unsigned)((rows + PJ_ROWS - 1) / PJ_ROWS), PJ_THREADS, smem, st>>>(a);
    }
    const dim3 gw((unsigned)PJ_GROUPS, (unsigned)((d_model + PJW_MT - 1) / PJW_MT), (unsigned)((O + PJ_COLS - 1) / PJ_COLS));
    project_dw_partial_kernel<<<gw, PJ_THREADS, 0, st>>>(a);
    project_dw_reduce_kernel<<<148, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace onedf
