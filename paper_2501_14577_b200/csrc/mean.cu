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
// Both are 3-phase blocked scans with a FIXED combination order (block sums
// -> sequential scan over blocks -> in-block sequential scan), so results are
// deterministic.  Threads map to columns, rows run sequentially, so every
// warp access to a d_v-wide row is one coalesced 128-B line.
#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int MEAN_TB = 128;   // rows per scan block

static int64_t mean_blocks(const onedf_problem* p) { return (p->N + MEAN_TB - 1) / MEAN_TB; }

void mean_carve(const onedf_problem* p, Carver* c, MeanBufs* m) {
    const int64_t BH = p->B * p->H;
    const int64_t rows = p->causal ? p->N : 1;
    m->Kbar = c->take<float>((size_t)(BH * rows * p->d_k));
    m->Vbar = c->take<float>((size_t)(BH * rows * p->d_v));
    m->part = c->take<double>((size_t)(BH * (mean_blocks(p) + 1) * (p->d_k + p->d_v)));
}

// ------------------------------------------------------------------ forward prefix means
__global__ void mean_block_sums_kernel(const float* __restrict__ K, const float* __restrict__ V, int64_t N, int dk,
                                       int dv, int64_t nblk, double* __restrict__ part) {
    const int64_t bh = blockIdx.y, blk = blockIdx.x;
    const int W = dk + dv;
    const int64_t r0 = blk * MEAN_TB, r1 = min64(N, r0 + MEAN_TB);
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
        double acc = 0.0;
        if (c < dk) {
            for (int64_t r = r0; r < r1; ++r) acc += (double)K[(bh * N + r) * dk + c];
        } else {
            const int cv = c - dk;
            for (int64_t r = r0; r < r1; ++r) acc += (double)V[(bh * N + r) * dv + cv];
        }
        part[(bh * (nblk + 1) + blk) * W + c] = acc;
    }
}

// exclusive scan over blocks (forward direction); part[nblk] = total
__global__ void mean_scan_blocks_kernel(double* __restrict__ part, int64_t nblk, int W, int64_t N, int causal,
                                        float* __restrict__ Kbar, float* __restrict__ Vbar, int dk, int dv) {
    const int64_t bh = blockIdx.x;
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
        double run = 0.0;
        for (int64_t b = 0; b < nblk; ++b) {
            double* x = part + (bh * (nblk + 1) + b) * W + c;
            double t = *x;
            *x = run;
            run += t;
        }
        part[(bh * (nblk + 1) + nblk) * W + c] = run;
        if (!causal) {
            const float mean = (float)(run / (double)N);
            if (c < dk) Kbar[bh * dk + c] = mean;
            else Vbar[bh * dv + (c - dk)] = mean;
        }
    }
}

__global__ void mean_write_kernel(const float* __restrict__ K, const float* __restrict__ V, int64_t N, int dk, int dv,
                                  int64_t nblk, const double* __restrict__ part, float* __restrict__ Kbar,
                                  float* __restrict__ Vbar) {
    const int64_t bh = blockIdx.y, blk = blockIdx.x;
    const int W = dk + dv;
    const int64_t r0 = blk * MEAN_TB, r1 = min64(N, r0 + MEAN_TB);
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
        double acc = part[(bh * (nblk + 1) + blk) * W + c];
        if (c < dk) {
            for (int64_t r = r0; r < r1; ++r) {
                acc += (double)K[(bh * N + r) * dk + c];
                Kbar[(bh * N + r) * dk + c] = (float)(acc / (double)(r + 1));
            }
        } else {
            const int cv = c - dk;
            for (int64_t r = r0; r < r1; ++r) {
                acc += (double)V[(bh * N + r) * dv + cv];
                Vbar[(bh * N + r) * dv + cv] = (float)(acc / (double)(r + 1));
            }
        }
    }
}

static int mean_threads(int W) { return W <= 64 ? 64 : (W <= 128 ? 128 : 256); }

cudaError_t launch_prefix_means(const onedf_problem* p, const float* K, const float* V, MeanBufs* m,
                                cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N, nblk = mean_blocks(p);
    const int dk = p->d_k, dv = p->d_v, W = dk + dv;
    const int th = mean_threads(W);
    mean_block_sums_kernel<<<dim3((unsigned)nblk, (unsigned)BH), th, 0, st>>>(K, V, N, dk, dv, nblk, m->part);
    mean_scan_blocks_kernel<<<(unsigned)BH, th, 0, st>>>(m->part, nblk, W, N, p->causal, m->Kbar, m->Vbar, dk, dv);
    if (p->causal)
        mean_write_kernel<<<dim3((unsigned)nblk, (unsigned)BH), th, 0, st>>>(K, V, N, dk, dv, nblk, m->part, m->Kbar,
                                                                            m->Vbar);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ backward chain rule (A11)
// y_i[c] = dKbar_i[c] (c < dk) or dVbar_i[c - dk]; scaled by 1/(i+1) when causal.
__device__ __forceinline__ double mean_grad_y(int c, int64_t bh, int64_t i, int64_t N, int dk, int dv, int causal,
                                              const float* __restrict__ Q, const float* __restrict__ Kbar,
                                              const float* __restrict__ dO, const float2* __restrict__ muco) {
    const float2 mc = muco[bh * N + i];
    double y;
    if (c < dk) {
        const float kb = Kbar[(bh * (causal ? N : 1) + (causal ? i : 0)) * dk + c];
        y = (double)mc.y * ((double)Q[(bh * N + i) * dk + c] - (double)kb);
    } else {
        y = (double)mc.x * (double)dO[(bh * N + i) * dv + (c - dk)];
    }
    return causal ? y / (double)(i + 1) : y;
}

__global__ void grad_block_sums_kernel(const float* __restrict__ Q, const float* __restrict__ Kbar,
                                       const float* __restrict__ dO, const float2* __restrict__ muco, int64_t N,
                                       int dk, int dv, int causal, int64_t nblk, double* __restrict__ part) {
    const int64_t bh = blockIdx.y, blk = blockIdx.x;
    const int W = dk + dv;
    const int64_t r0 = blk * MEAN_TB, r1 = min64(N, r0 + MEAN_TB);
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t r = r1 - 1; r >= r0; --r) acc += mean_grad_y(c, bh, r, N, dk, dv, causal, Q, Kbar, dO, muco);
        part[(bh * (nblk + 1) + blk) * W + c] = acc;
    }
}

// exclusive SUFFIX scan over blocks: part[b] = sum of blocks > b; part[nblk] = total
__global__ void grad_scan_blocks_kernel(double* __restrict__ part, int64_t nblk, int W) {
    const int64_t bh = blockIdx.x;
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
        double run = 0.0;
        for (int64_t b = nblk - 1; b >= 0; --b) {
            double* x = part + (bh * (nblk + 1) + b) * W + c;
            double t = *x;
            *x = run;
            run += t;
        }
        part[(bh * (nblk + 1) + nblk) * W + c] = run;
    }
}

__global__ void grad_apply_kernel(const float* __restrict__ Q, const float* __restrict__ Kbar,
                                  const float* __restrict__ dO, const float2* __restrict__ muco, int64_t N, int dk,
                                  int dv, int causal, int64_t nblk, const double* __restrict__ part,
                                  float* __restrict__ dK, float* __restrict__ dV) {
    const int64_t bh = blockIdx.y, blk = blockIdx.x;
    const int W = dk + dv;
    const int64_t r0 = blk * MEAN_TB, r1 = min64(N, r0 + MEAN_TB);
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
        float* out = c < dk ? dK + bh * N * dk + c : dV + bh * N * dv + (c - dk);
        const int stride = c < dk ? dk : dv;
        if (causal) {
            double acc = part[(bh * (nblk + 1) + blk) * W + c];
            for (int64_t r = r1 - 1; r >= r0; --r) {
                acc += mean_grad_y(c, bh, r, N, dk, dv, causal, Q, Kbar, dO, muco);
                out[r * stride] = (float)((double)out[r * stride] + acc);
            }
        } else {
            const double add = part[(bh * (nblk + 1) + nblk) * W + c] / (double)N;
            for (int64_t r = r0; r < r1; ++r) out[r * stride] = (float)((double)out[r * stride] + add);
        }
    }
}

cudaError_t launch_mean_grad_scan(const onedf_problem* p, const float* Q, const float* dO, const float* muco,
                                  MeanBufs* m, float* dK, float* dV, cudaStream_t st) {
    const int64_t BH = p->B * p->H, N = p->N, nblk = mean_blocks(p);
    const int dk = p->d_k, dv = p->d_v, W = dk + dv;
    const int th = mean_threads(W);
    const float2* mc = reinterpret_cast<const float2*>(muco);
    grad_block_sums_kernel<<<dim3((unsigned)nblk, (unsigned)BH), th, 0, st>>>(Q, m->Kbar, dO, mc, N, dk, dv,
                                                                              p->causal, nblk, m->part);
    grad_scan_blocks_kernel<<<(unsigned)BH, th, 0, st>>>(m->part, nblk, W);
    grad_apply_kernel<<<dim3((unsigned)nblk, (unsigned)BH), th, 0, st>>>(Q, m->Kbar, dO, mc, N, dk, dv, p->causal,
                                                                         nblk, m->part, dK, dV);
    return cudaGetLastError();
}

}  // namespace onedf
