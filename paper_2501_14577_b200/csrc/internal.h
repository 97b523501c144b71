// internal.h -- launchers shared between the kernel translation units and abi.cu.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "onedf.h"

namespace onedf {

// Optional stage events (onedf_*_traced): record events[s] after stage s.
struct Trace {
    void* const* ev = nullptr;
    int n = 0;
    void mark(int s, cudaStream_t st) const {
        if (ev && s < n && ev[s]) cudaEventRecord((cudaEvent_t)ev[s], st);
    }
};

// Longest run the shared-memory segmented sort keeps on chip (keys + ping-pong
// in smem); longer runs sort through global scratch (SortScratch).
constexpr int64_t SEG_SORT_MAX = 8192;

int effective_bits(const onedf_problem* p);
int effective_window(const onedf_problem* p);
int64_t run_len_max(const onedf_problem* p);   // M (causal, capped at N) or N
int64_t num_runs(const onedf_problem* p);
Shard make_shard(const onedf_problem* p);      // world <= 1 -> unsharded

// encode.cu
size_t encode_ws_bytes(const onedf_problem* p, Carver* c);
cudaError_t launch_encode(const onedf_problem* p, int b, const float* Q, const float* K, const double* lohi_in,
                          uint64_t* qcode, uint64_t* kcode, double* lohi_out, void* ws, Carver* c,
                          cudaStream_t st);

// bounds-only launches (onedf_bounds_partial / _finish)
cudaError_t launch_bounds_partial(const onedf_problem* p, const float* Q, const float* K, double* lohi, void* ws,
                                  Carver* c, cudaStream_t st);
cudaError_t launch_bounds_finish(const onedf_problem* p, double* lohi, void* ws, cudaStream_t st);
cudaError_t launch_rank_sum(const float* parts, int64_t n, int32_t world, float* out, cudaStream_t st);

// sort.cu
// Global scratch of the onesweep sort of runs longer than SEG_SORT_MAX (else null): ping-pong
// keys/positions, per-(run, pass) digit bases, per-(run, tile, digit) look-back status words and the
// per-pass tile tickets.
struct SortScratch {
    uint64_t* k[2];
    uint32_t* v[2];
    uint32_t* base;     // [runs][8][256]  digit counts -> exclusive digit offsets per pass
    uint32_t* status;   // [runs][tiles][256] decoupled look-back words (flag << 30 | count)
    uint32_t* ticket;   // [8]             dynamic tile order per pass
};
void sort_carve(const onedf_problem* p, Carver* c, SortScratch* s);
cudaError_t launch_seg_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode /* nullable */,
                            int32_t* perm, const SortScratch& scr, cudaStream_t st);
cudaError_t launch_query_order(const onedf_problem* p, const uint64_t* qcode, int32_t* qorder,
                               const SortScratch& scr, cudaStream_t st);


// csr.cu -- A9 key-major CSR of the selected (query, slot) records
// Segments longer than this are ordered by csr_long_order_kernel (a bitmap over query positions;
// none at long64k, where the longest is ~450);
// shorter ones by the key side itself (register bitonic sort of (i << KEY_POS_BITS | position) keys).
#ifndef ONEDF_KEY_REG_SEG
#define ONEDF_KEY_REG_SEG 512
#endif
constexpr int KEY_REG_SEG = ONEDF_KEY_REG_SEG;     // 256 or 512 (register rows of the key side's sort)
constexpr int KEY_POS_BITS = KEY_REG_SEG > 256 ? 9 : 8;   // u32 sort key (i << bits | position): N < 2^(32-bits)
__host__ __device__ inline bool csr_long_segment(int64_t len, int64_t N) {
    return len > KEY_REG_SEG || N >= (1ll << (32 - KEY_POS_BITS));
}

struct CsrBufs {
    int32_t* cursor;    // [BH][N]    in-degree counts -> insertion cursors
    int32_t* offsets;   // [BH][N+1]  segment of key j = records [off[j], off[j+1])
    int32_t* rec_i;     // [BH][N*k]  query position i of each selected (query, slot) record   (SoA:
    float2* rec_aw;     // [BH][N*k]  its (A_ij, w_ij)                                          12 B/record)
    int32_t* order;     // [BH][N*k]  ascending-i order of the long segments (csr_long_segment)
    int32_t* nlong;     // [1]        number of long segments
    int2* longseg;      // [BH*N]     their (bh, j), in no particular order (each is ordered independently)
    int32_t* bsum;      // [BH][N/4096 + 1] block sums of the multi-CTA offset scan
};
void csr_carve(const onedf_problem* p, Carver* c, CsrBufs* t);
// qorder: the query schedule (nullable -> natural order); only its grouping of similar queries matters.
// indeg: nullable, the forward's in-degree counts of this idx (then copied instead of counted)
cudaError_t launch_csr_count(const onedf_problem* p, const int32_t* idx, const int32_t* qorder,
                             const int32_t* indeg, CsrBufs* t, cudaStream_t st);
// after the query side has appended every record: ascending-i order of each long segment
cudaError_t launch_csr_long_order(const onedf_problem* p, CsrBufs* t, cudaStream_t st);

// mean.cu
struct MeanBufs {
    float* Kbar;        // [BH][rows][d_k], rows = N (causal) or 1
    float* Vbar;        // [BH][rows][d_v]
    double* part;       // scan partials
};
void mean_carve(const onedf_problem* p, Carver* c, MeanBufs* m);
cudaError_t launch_prefix_means(const onedf_problem* p, const float* K, const void* V, MeanBufs* m,
                                cudaStream_t st);
// A11: dK_t += sum_{i>=t} wmu_i (q_i - Kbar_i)/(i+1), dV_t = dV32_t + sum_{i>=t} Amu_i dO_i/(i+1) (causal; 1/N
// all i otherwise); dV32 is the key side's f32 result (== dV for float storage, in place)
cudaError_t launch_mean_grad_scan(const onedf_problem* p, const float* Q, const void* dO, const float* muco,
                                  MeanBufs* m, float* dK, const float* dV32, void* dV, cudaStream_t st);
// dst = bf16(src), n values (n % 4 == 0)
cudaError_t launch_round_rows(const float* src, bf16* dst, int64_t n, cudaStream_t st);

// fwd.cu
struct FwdBufs {
    float* recs;        // [BH][N][RecW] sorted key records
    int32_t* qorder;    // [BH][N] query schedule (per chunk, by qcode)
    SortScratch scr;    // for the query-order sort of long runs
};
void fwd_carve(const onedf_problem* p, Carver* c, FwdBufs* f);
// qorder: the caller's query schedule (nullable -> sorted here from qcode)
cudaError_t launch_fwd(const onedf_problem* p, const float* Q, const float* K, const void* V, const float* eps,
                       const uint64_t* qcode, const uint64_t* scode, const int32_t* perm, const int32_t* qorder,
                       void* O, int32_t* idx, float* Z, int32_t* indeg, const MeanBufs* m, FwdBufs* f, void* ws,
                       cudaStream_t st, const Trace& tr);

// bwd.cu
constexpr int EPS_PARTS = 1024;   // fixed first-level split of the d_eps reduction
struct BwdBufs {
    float2* muco;       // [BH][N]    (A_mu, w_mu)
    double* eps_q;      // [BH][N]    per-query d_eps contribution
    double* eps_part;   // [EPS_PARTS]
    int32_t* qorder;    // [BH][N]    query schedule (when only qcode is given)
    float* dV32;        // [BH][N][d_v] key-side f32 dV of a BF16 problem (rounded once at the end), else null
    SortScratch scr;    // for the query-order sort of long runs
};
void bwd_carve(const onedf_problem* p, Carver* c, BwdBufs* b);
cudaError_t launch_bwd(const onedf_problem* p, const float* Q, const float* K, const void* V, const float* eps,
                       const void* dO, const int32_t* idx, const uint64_t* qcode, const int32_t* qorder,
                       const int32_t* perm, const int32_t* indeg, float* dQ, float* dK, void* dV, double* d_eps,
                       const MeanBufs* m, BwdBufs* b, CsrBufs* t, void* ws, cudaStream_t st, const Trace& tr);

// proj.cu (NEXT-4 projections f_q, f_k and eps = sigma(theta))
size_t project_ws_bytes(const onedf_problem* p, int d_model, Carver* c);
cudaError_t launch_project(const onedf_problem* p, int d_model, const float* X, const float* Wq, const float* Wk,
                           const float* bq, const float* bk, const float* theta, float* Q, float* K, float* eps,
                           void* ws, cudaStream_t st);
cudaError_t launch_project_bwd(const onedf_problem* p, int d_model, const float* X, const float* Wq, const float* Wk,
                               const float* theta, const float* dQ, const float* dK, const double* d_eps, float* dX,
                               float* dWq, float* dWk, float* dbq, float* dbk, float* dtheta, void* ws,
                               cudaStream_t st);

// workload.cu (NEXT-3 locality workload)
cudaError_t launch_code_knn(const onedf_problem* p, const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                            int exclude_self, int32_t* idx, cudaStream_t st);
cudaError_t launch_overlap(const int32_t* a, int ka, const int32_t* b, int kb, int64_t rows, int64_t self_period,
                           int32_t* counts, cudaStream_t st);

}  // namespace onedf
