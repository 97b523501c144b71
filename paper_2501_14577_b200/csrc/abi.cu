// abi.cu -- the extern "C" boundary declared in include/onedf.h: synchronous
// argument validation, workspace layout, and the launch sequence of each call.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace onedf {

int effective_bits(const onedf_problem* p) {
    if (p->bits) return p->bits;
    const int b = 63 / p->d_k;
    return b > 32 ? 32 : b;
}
int effective_window(const onedf_problem* p) { return p->window ? p->window : 2 * p->k; }
int64_t run_len_max(const onedf_problem* p) {
    if (!p->causal) return p->N;
    return p->chunk < p->N ? p->chunk : p->N;
}
int64_t num_runs(const onedf_problem* p) { return p->causal ? (p->N + p->chunk - 1) / p->chunk : 1; }
Shard make_shard(const onedf_problem* p) {
    Shard s;
    if (p->shard_world > 1) {
        s.rank = p->shard_rank;
        s.world = p->shard_world;
        s.M = run_len_max(p);
        s.C = num_runs(p);
    }
    return s;
}

static onedf_status check_device() {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return ONEDF_ERR_CUDA; }
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
        cudaGetLastError();
        return ONEDF_ERR_CUDA;
    }
    return (major == 10 && minor == 0) ? ONEDF_OK : ONEDF_ERR_UNSUPPORTED;
}

static onedf_status validate(const onedf_problem* p) {
    if (!p) return ONEDF_ERR_INVALID_ARG;
    if (p->B < 1 || p->H < 1 || p->N < 1 || p->N >= (1ll << 31)) return ONEDF_ERR_INVALID_ARG;
    if (p->B * p->H > 65535) return ONEDF_ERR_INVALID_ARG;
    if (p->d_k < 1 || p->d_k > 8) return ONEDF_ERR_INVALID_ARG;
    if (p->d_v < 4 || p->d_v > 256 || p->d_v % 4) return ONEDF_ERR_INVALID_ARG;
    if (p->k < 1 || p->k > 256) return ONEDF_ERR_INVALID_ARG;
    if (p->window < 0 || p->bits < 0) return ONEDF_ERR_INVALID_ARG;
    const int W = effective_window(p);
    if (W < p->k || W > (1 << 20)) return ONEDF_ERR_INVALID_ARG;
    if (p->causal != 0 && p->causal != 1) return ONEDF_ERR_INVALID_ARG;
    if (p->mean_slot != 0 && p->mean_slot != 1) return ONEDF_ERR_INVALID_ARG;
    if (p->causal && p->chunk < 1) return ONEDF_ERR_INVALID_ARG;
    const int b = effective_bits(p);
    if (b < 1 || b > 32 || p->d_k * b > 63) return ONEDF_ERR_INVALID_ARG;
    if (p->N * (int64_t)p->k >= (1ll << 31)) return ONEDF_ERR_INVALID_ARG;
    if (p->shard_world < 0 || p->shard_world > 4096) return ONEDF_ERR_INVALID_ARG;
    if (p->score < ONEDF_SCORE_CAUCHY || p->score > ONEDF_SCORE_DOT) return ONEDF_ERR_INVALID_ARG;
    if (p->select != ONEDF_SELECT_EUCLID && p->select != ONEDF_SELECT_CODE) return ONEDF_ERR_INVALID_ARG;
    if (p->vdtype != ONEDF_DTYPE_F32 && p->vdtype != ONEDF_DTYPE_BF16) return ONEDF_ERR_INVALID_ARG;
    if (p->shard_world > 1) {
        if (p->shard_rank < 0 || p->shard_rank >= p->shard_world) return ONEDF_ERR_INVALID_ARG;
        if (!p->causal) return ONEDF_ERR_UNSUPPORTED;   // sequence sharding is defined over causal chunks
        if (p->vdtype != ONEDF_DTYPE_F32) return ONEDF_ERR_UNSUPPORTED;   // partial dV rows are exchanged in f32
    } else if (p->shard_rank != 0) {
        return ONEDF_ERR_INVALID_ARG;
    }
    return ONEDF_OK;
}

// ---------------------------------------------------------------- workspace layouts
struct FwdLayout { MeanBufs m; FwdBufs f; size_t bytes; };
struct BwdLayout { MeanBufs m; BwdBufs b; CsrBufs t; size_t bytes; };

static FwdLayout fwd_layout(const onedf_problem* p, void* ws) {
    FwdLayout L;
    Carver c(ws);
    mean_carve(p, &c, &L.m);
    fwd_carve(p, &c, &L.f);
    L.bytes = c.bytes();
    return L;
}
static BwdLayout bwd_layout(const onedf_problem* p, void* ws) {
    BwdLayout L;
    Carver c(ws);
    mean_carve(p, &c, &L.m);
    bwd_carve(p, &c, &L.b);
    csr_carve(p, &c, &L.t);
    L.bytes = c.bytes();
    return L;
}
static size_t encode_bytes(const onedf_problem* p) {
    Carver c(nullptr);
    return encode_ws_bytes(p, &c);
}
static size_t sort_bytes(const onedf_problem* p) {
    Carver c(nullptr);
    SortScratch s;
    sort_carve(p, &c, &s);
    return c.bytes();
}

// The host-buffer step pipelines groups of (b,h) slices: H2D of group g+1 and
// D2H of group g-1 overlap the compute of group g (three streams, events).
constexpr int STEP_GROUPS_MAX = 8;

struct StepLayout {
    float *Q, *K, *dQ, *dK, *Z, *eps;
    char *V, *dO, *O, *dV;          // value rows of the storage type p->vdtype
    double* d_eps;
    uint64_t *qcode, *kcode, *scode;
    int32_t *perm, *qorder, *idx, *indeg;
    float* means;                   // the forward's prefix means, read by the backward
    size_t sub_off, sub_bytes, bytes;
};
static size_t value_bytes(const onedf_problem* p) { return p->vdtype == ONEDF_DTYPE_BF16 ? 2 : 4; }
static StepLayout step_layout(const onedf_problem* p, void* ws) {
    StepLayout L;
    const size_t e = encode_bytes(p), s = sort_bytes(p);
    const size_t f = fwd_layout(p, nullptr).bytes, b = bwd_layout(p, nullptr).bytes;
    size_t sub = e > s ? e : s;
    sub = sub > f ? sub : f;
    sub = sub > b ? sub : b;
    Carver c(ws);
    const int64_t BH = p->B * p->H, N = p->N, nk = BH * N * p->d_k;
    const size_t nvb = (size_t)(BH * N * p->d_v) * value_bytes(p);
    L.Q = c.take<float>(nk); L.K = c.take<float>(nk); L.V = c.take<char>(nvb); L.dO = c.take<char>(nvb);
    L.O = c.take<char>(nvb); L.dQ = c.take<float>(nk); L.dK = c.take<float>(nk); L.dV = c.take<char>(nvb);
    L.Z = c.take<float>(BH * N); L.eps = c.take<float>(1); L.d_eps = c.take<double>(STEP_GROUPS_MAX + 1);
    L.qcode = c.take<uint64_t>(BH * N); L.kcode = c.take<uint64_t>(BH * N); L.scode = c.take<uint64_t>(BH * N);
    L.perm = c.take<int32_t>(BH * N); L.qorder = c.take<int32_t>(BH * N); L.idx = c.take<int32_t>(BH * N * p->k);
    L.indeg = c.take<int32_t>(BH * N);
    // room for every group's means region (each 256-B aligned; groups of fewer slices need no more)
    L.means = p->mean_slot ? c.take<float>((size_t)(onedf_means_floats(p) + 2 * 64 * STEP_GROUPS_MAX)) : nullptr;
    c.take<char>(0);
    L.sub_off = c.off;
    L.sub_bytes = sub;
    c.take<char>(sub);
    L.bytes = c.bytes();
    return L;
}

__global__ void set_scalar_kernel(float* dst, float v) { *dst = v; }

// d_eps of the whole batch: the groups' partial sums added in group order (fixed, deterministic)
__global__ void sum_groups_kernel(double* parts, int n) {
    double s = 0.0;
    for (int g = 0; g < n; ++g) s += parts[1 + g];
    parts[0] = s;
}

static onedf_status finish(cudaError_t e) {
    if (e != cudaSuccess) { cudaGetLastError(); return ONEDF_ERR_CUDA; }
    return ONEDF_OK;
}

static onedf_status pre(const onedf_problem* p, void* ws, size_t ws_bytes, int op) {
    onedf_status s = validate(p);
    if (s != ONEDF_OK) return s;
    if (!ws || (((uintptr_t)ws) & 255) != 0 || ws_bytes < onedf_workspace_size(p, op)) return ONEDF_ERR_WORKSPACE;
    return check_device();
}

// Zero the flag word of `op` in the workspace header (common.cuh FLAG_WORDS).
static cudaError_t zero_flags(void* ws, int op, cudaStream_t st) {
    return cudaMemsetAsync((char*)ws + 4 * op, 0, 4, st);
}

// Internal entry points (flag zeroing optional so the host step can chain them).
static onedf_status do_encode(const onedf_problem* p, const float* Q, const float* K, const double* lohi_in,
                              uint64_t* qcode, uint64_t* kcode, double* lohi_out, void* ws, cudaStream_t st,
                              bool zero) {
    if (zero && zero_flags(ws, ONEDF_OP_ENCODE, st) != cudaSuccess) return finish(cudaGetLastError());
    Carver c(ws);
    return finish(launch_encode(p, effective_bits(p), Q, K, lohi_in, qcode, kcode, lohi_out, ws, &c, st));
}
static onedf_status do_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode /* nullable */,
                            int32_t* perm, void* ws, cudaStream_t st) {
    Carver c(ws);
    SortScratch scr;
    sort_carve(p, &c, &scr);
    return finish(launch_seg_sort(p, kcode, scode, perm, scr, st));
}
// A caller-owned prefix-means buffer (onedf.h: Kbar [B,H,rows,d_k] then Vbar [B,H,rows,d_v], f32).
// Both blocks start 256-B aligned (the kernels read the rows as float4).
static int64_t align64(int64_t x) { return (x + 63) / 64 * 64; }
static void means_view(const onedf_problem* p, float* means, MeanBufs* m) {
    const int64_t rows = p->causal ? p->N : 1;
    m->Kbar = means;
    m->Vbar = means + align64(p->B * p->H * rows * p->d_k);
}
static onedf_status do_fwd(const onedf_problem* p, const float* Q, const float* K, const void* V, const float* eps,
                           const uint64_t* qcode, const uint64_t* scode, const int32_t* perm, const int32_t* qorder,
                           void* O, int32_t* idx, float* Z, int32_t* indeg, float* means, void* ws, cudaStream_t st,
                           bool zero, const Trace& tr = Trace()) {
    if (zero && zero_flags(ws, ONEDF_OP_FWD, st) != cudaSuccess) return finish(cudaGetLastError());
    FwdLayout L = fwd_layout(p, ws);
    if (means) means_view(p, means, &L.m);          // the prefix means land in the caller's buffer
    cudaError_t e = cudaSuccess;
    if (p->mean_slot) e = launch_prefix_means(p, K, V, &L.m, st);
    tr.mark(0, st);
    if (e == cudaSuccess) e = launch_fwd(p, Q, K, V, eps, qcode, scode, perm, qorder, O, idx, Z, indeg, &L.m, &L.f, ws, st,
                                              tr);
    return finish(e);
}
static onedf_status do_bwd(const onedf_problem* p, const float* Q, const float* K, const void* V, const float* eps,
                           const void* dO, const int32_t* idx, const uint64_t* qcode, const int32_t* qorder,
                           const int32_t* perm, const int32_t* indeg, const float* means, float* dQ, float* dK,
                           void* dV, double* d_eps, void* ws, cudaStream_t st, bool zero,
                           const Trace& tr = Trace()) {
    if (zero && zero_flags(ws, ONEDF_OP_BWD, st) != cudaSuccess) return finish(cudaGetLastError());
    BwdLayout L = bwd_layout(p, ws);
    cudaError_t e = cudaSuccess;
    if (means) means_view(p, const_cast<float*>(means), &L.m);   // the forward's prefix means: read only
    else if (p->mean_slot) e = launch_prefix_means(p, K, V, &L.m, st);
    tr.mark(0, st);
    if (e == cudaSuccess)
        e = launch_bwd(p, Q, K, V, eps, dO, idx, qcode, qorder, perm, indeg, dQ, dK, dV, d_eps, &L.m, &L.b, &L.t, ws, st,
                       tr);
    return finish(e);
}

}  // namespace onedf

using namespace onedf;

extern "C" {

onedf_status onedf_validate(const onedf_problem* p) { return validate(p); }

int64_t onedf_max_run_length(void) { return SEG_SORT_MAX; }

size_t onedf_workspace_size(const onedf_problem* p, int op) {
    if (validate(p) != ONEDF_OK) return 0;
    switch (op) {
        case ONEDF_OP_ENCODE: return encode_bytes(p);
        case ONEDF_OP_SORT: return sort_bytes(p);
        case ONEDF_OP_FWD: return fwd_layout(p, nullptr).bytes;
        case ONEDF_OP_BWD: return bwd_layout(p, nullptr).bytes;
        case ONEDF_OP_STEP_HOST: return step_layout(p, nullptr).bytes;
        default: return 0;
    }
}

onedf_status onedf_encode(const onedf_problem* p, const float* Q, const float* K, const double* lohi_in,
                          uint64_t* qcode, uint64_t* kcode, double* lohi_out, void* ws, size_t ws_bytes,
                          onedf_stream_t stream) {
    if (validate(p) == ONEDF_OK && p->shard_world > 1 && !lohi_in)
        return ONEDF_ERR_INVALID_ARG;   // sharded FIT: bounds_partial + all-reduce + bounds_finish
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_ENCODE);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !qcode || !kcode) return ONEDF_ERR_INVALID_ARG;
    return do_encode(p, Q, K, lohi_in, qcode, kcode, lohi_out, ws, (cudaStream_t)stream, true);
}

onedf_status onedf_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm, void* ws,
                        size_t ws_bytes, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_SORT);
    if (s != ONEDF_OK) return s;
    if (!kcode || !perm) return ONEDF_ERR_INVALID_ARG;
    if (zero_flags(ws, ONEDF_OP_SORT, (cudaStream_t)stream) != cudaSuccess) return finish(cudaGetLastError());
    return do_sort(p, kcode, scode, perm, ws, (cudaStream_t)stream);
}

// value-row pointers: 16-B aligned (float4 chunks) for float rows, 8-B (4 x bf16) for bf16 rows
static bool rows_misaligned(const onedf_problem* p, const void* a, const void* b, const void* c = nullptr) {
    const uintptr_t m = p->vdtype == ONEDF_DTYPE_BF16 ? 7 : 15;
    return ((((uintptr_t)a) | ((uintptr_t)b) | ((uintptr_t)c)) & m) != 0;
}

int64_t onedf_means_floats(const onedf_problem* p) {
    if (!p || !p->mean_slot) return 0;
    const int64_t rows = p->B * p->H * (p->causal ? p->N : 1);
    return align64(rows * p->d_k) + align64(rows * p->d_v);
}

onedf_status onedf_topk_attn_fwd(const onedf_problem* p, const float* Q, const float* K, const void* V,
                                 const float* eps, const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                                 const int32_t* qorder, void* O, int32_t* idx, float* Z, int32_t* indeg, float* means,
                                 void* ws, size_t ws_bytes, onedf_stream_t stream) {
    return onedf_topk_attn_fwd_traced(p, Q, K, V, eps, qcode, scode, perm, qorder, O, idx, Z, indeg, means, ws,
                                      ws_bytes, nullptr, 0, stream);
}

onedf_status onedf_topk_attn_bwd(const onedf_problem* p, const float* Q, const float* K, const void* V,
                                 const float* eps, const void* O, const void* dO, const int32_t* idx, const float* Z,
                                 const uint64_t* qcode, const int32_t* qorder, const int32_t* perm,
                                 const int32_t* indeg, const float* means, float* dQ, float* dK, void* dV,
                                 double* d_eps, void* ws, size_t ws_bytes, onedf_stream_t stream) {
    return onedf_topk_attn_bwd_traced(p, Q, K, V, eps, O, dO, idx, Z, qcode, qorder, perm, indeg, means, dQ, dK, dV,
                                      d_eps, ws, ws_bytes, nullptr, 0, stream);
}

onedf_status onedf_topk_attn_fwd_traced(const onedf_problem* p, const float* Q, const float* K, const void* V,
                                        const float* eps, const uint64_t* qcode, const uint64_t* scode,
                                        const int32_t* perm, const int32_t* qorder, void* O, int32_t* idx, float* Z,
                                        int32_t* indeg, float* means, void* ws, size_t ws_bytes, void* const* events,
                                        int n_events, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_FWD);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !V || !eps || !qcode || !scode || !perm || !O || !idx || !Z) return ONEDF_ERR_INVALID_ARG;
    if (rows_misaligned(p, V, O)) return ONEDF_ERR_INVALID_ARG;
    Trace tr;
    tr.ev = events;
    tr.n = n_events;
    return do_fwd(p, Q, K, V, eps, qcode, scode, perm, qorder, O, idx, Z, indeg, means, ws, (cudaStream_t)stream, true,
                  tr);
}

onedf_status onedf_topk_attn_bwd_traced(const onedf_problem* p, const float* Q, const float* K, const void* V,
                                        const float* eps, const void* O, const void* dO, const int32_t* idx,
                                        const float* Z, const uint64_t* qcode, const int32_t* qorder,
                                        const int32_t* perm, const int32_t* indeg, const float* means, float* dQ,
                                        float* dK, void* dV, double* d_eps, void* ws, size_t ws_bytes,
                                        void* const* events, int n_events, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_BWD);
    if (s != ONEDF_OK) return s;
    // O and Z are part of the interface but not read (reading R3: recomputed in f64)
    if (!Q || !K || !V || !eps || !O || !dO || !idx || !Z || !dQ || !dK || !dV || !d_eps)
        return ONEDF_ERR_INVALID_ARG;
    if (rows_misaligned(p, V, dO, dV)) return ONEDF_ERR_INVALID_ARG;
    Trace tr;
    tr.ev = events;
    tr.n = n_events;
    return do_bwd(p, Q, K, V, eps, dO, idx, qcode, qorder, perm, indeg, means, dQ, dK, dV, d_eps, ws,
                  (cudaStream_t)stream, true, tr);
}

onedf_status onedf_topk_attn_step_host(const onedf_problem* p, const float* Q_h, const float* K_h, const void* V_h,
                                       float eps, const void* dO_h, void* O_h, float* dQ_h, float* dK_h,
                                       void* dV_h, double* d_eps_h, void* ws, size_t ws_bytes,
                                       onedf_stream_t stream) {
    if (validate(p) == ONEDF_OK && p->shard_world > 1) return ONEDF_ERR_UNSUPPORTED;   // needs the caller's collectives
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_STEP_HOST);
    if (s != ONEDF_OK) return s;
    if (!Q_h || !K_h || !V_h || !dO_h || !O_h || !dQ_h || !dK_h || !dV_h || !d_eps_h) return ONEDF_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    StepLayout L = step_layout(p, ws);
    void* sub = (char*)ws + L.sub_off;
    const int64_t BH = p->B * p->H, N = p->N;
    const int G = (int)min64(BH, STEP_GROUPS_MAX);
    // side streams for the copies; events order them against the compute on `st`
    cudaStream_t sin = nullptr, sout = nullptr;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_in[STEP_GROUPS_MAX] = {}, ev_c[STEP_GROUPS_MAX] = {};
    cudaError_t e = cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_end, cudaEventDisableTiming);
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
        e = cudaEventCreateWithFlags(&ev_in[g], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_c[g], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(ws, 0, 4 * FLAG_WORDS, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(sub, 0, 4 * FLAG_WORDS, st);
    // eps by value: written by a one-thread kernel so the call needs no host staging buffer
    if (e == cudaSuccess) {
        set_scalar_kernel<<<1, 1, 0, st>>>(L.eps, eps);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev_start, st);       // prior work on `st` precedes the copies
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sin, ev_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, ev_start, 0);
    int64_t h0 = 0, moff = 0;
    for (int g = 0; g < G && e == cudaSuccess; ++g) {
        const int64_t nh = BH / G + (g < BH % G ? 1 : 0);           // slices of group g: [h0, h0 + nh)
        onedf_problem pg = *p;
        pg.B = 1;
        pg.H = nh;
        const size_t es = value_bytes(p);
        const size_t ok = (size_t)(h0 * N * p->d_k), ov = (size_t)(h0 * N * p->d_v) * es, o1 = (size_t)(h0 * N);
        const size_t bk = (size_t)(nh * N * p->d_k) * 4, bv = (size_t)(nh * N * p->d_v) * es;
        // group g's prefix means: its own region (onedf_means_floats of the group's problem)
        float* gmeans = L.means ? L.means + moff : nullptr;
        const char* Vh = static_cast<const char*>(V_h);
        const char* dOh = static_cast<const char*>(dO_h);
        e = cudaMemcpyAsync(L.Q + ok, Q_h + ok, bk, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) e = cudaMemcpyAsync(L.K + ok, K_h + ok, bk, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) e = cudaMemcpyAsync(L.V + ov, Vh + ov, bv, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) e = cudaMemcpyAsync(L.dO + ov, dOh + ov, bv, cudaMemcpyHostToDevice, sin);
        if (e == cudaSuccess) e = cudaEventRecord(ev_in[g], sin);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_in[g], 0);
        if (e != cudaSuccess) break;
        if ((s = do_encode(&pg, L.Q + ok, L.K + ok, nullptr, L.qcode + o1, L.kcode + o1, nullptr, sub, st, false)) !=
            ONEDF_OK)
            break;
        if ((s = do_sort(&pg, L.kcode + o1, L.scode + o1, L.perm + o1, sub, st)) != ONEDF_OK) break;
        // the Morton query schedule, sorted once for both passes
        if ((s = do_sort(&pg, L.qcode + o1, nullptr, L.qorder + o1, sub, st)) != ONEDF_OK) break;
        if ((s = do_fwd(&pg, L.Q + ok, L.K + ok, L.V + ov, L.eps, L.qcode + o1, L.scode + o1, L.perm + o1,
                        L.qorder + o1, L.O + ov, L.idx + o1 * p->k, L.Z + o1, L.indeg + o1, gmeans, sub, st,
                        false)) != ONEDF_OK)
            break;
        if ((s = do_bwd(&pg, L.Q + ok, L.K + ok, L.V + ov, L.eps, L.dO + ov, L.idx + o1 * p->k, L.qcode + o1,
                        L.qorder + o1, L.perm + o1, L.indeg + o1, gmeans, L.dQ + ok, L.dK + ok, L.dV + ov,
                        L.d_eps + 1 + g,
                        sub, st, false)) != ONEDF_OK)
            break;
        e = cudaEventRecord(ev_c[g], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(sout, ev_c[g], 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(static_cast<char*>(O_h) + ov, L.O + ov, bv, cudaMemcpyDeviceToHost, sout);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dQ_h + ok, L.dQ + ok, bk, cudaMemcpyDeviceToHost, sout);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dK_h + ok, L.dK + ok, bk, cudaMemcpyDeviceToHost, sout);
        if (e == cudaSuccess) e = cudaMemcpyAsync(static_cast<char*>(dV_h) + ov, L.dV + ov, bv, cudaMemcpyDeviceToHost, sout);
        h0 += nh;
        moff += onedf_means_floats(&pg);
    }
    if (s == ONEDF_OK && e == cudaSuccess) {
        sum_groups_kernel<<<1, 1, 0, st>>>(L.d_eps, G);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(ws, sub, 4 * FLAG_WORDS, cudaMemcpyDeviceToDevice, st);   // surface device flags
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_eps_h, L.d_eps, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev_end, sout);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_end, 0);      // the caller's stream covers all copies
    }
    // streams/events are released once their pending work completes (no synchronisation here)
    for (int g = 0; g < G; ++g) {
        if (ev_in[g]) cudaEventDestroy(ev_in[g]);
        if (ev_c[g]) cudaEventDestroy(ev_c[g]);
    }
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_end) cudaEventDestroy(ev_end);
    if (sin) cudaStreamDestroy(sin);
    if (sout) cudaStreamDestroy(sout);
    if (s != ONEDF_OK) return s;
    return finish(e);
}

onedf_status onedf_project_encode(const onedf_problem* p, int32_t d_model, const float* X, const float* Wq,
                                  const float* Wk, const float* bq, const float* bk, const float* theta,
                                  const double* lohi_in, float* Q, float* K, float* eps, uint64_t* qcode,
                                  uint64_t* kcode, double* lohi_out, void* ws, size_t ws_bytes,
                                  onedf_stream_t stream) {
    if (validate(p) == ONEDF_OK && p->shard_world > 1 && !lohi_in) return ONEDF_ERR_INVALID_ARG;
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_ENCODE);
    if (s != ONEDF_OK) return s;
    if (d_model < 1 || !X || !Wq || !Wk || !Q || !K || !qcode || !kcode || (theta && !eps)) return ONEDF_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (zero_flags(ws, ONEDF_OP_ENCODE, st) != cudaSuccess) return finish(cudaGetLastError());
    cudaError_t e = launch_project(p, d_model, X, Wq, Wk, bq, bk, theta, Q, K, eps, ws, st);
    if (e != cudaSuccess) return finish(e);
    return do_encode(p, Q, K, lohi_in, qcode, kcode, lohi_out, ws, st, false);
}

size_t onedf_project_workspace_size(const onedf_problem* p, int32_t d_model) {
    if (validate(p) != ONEDF_OK || d_model < 1) return 0;
    Carver c(nullptr);
    return project_ws_bytes(p, d_model, &c);
}

onedf_status onedf_project_bwd(const onedf_problem* p, int32_t d_model, const float* X, const float* Wq,
                               const float* Wk, const float* theta, const float* dQ, const float* dK,
                               const double* d_eps, float* dX, float* dWq, float* dWk, float* dbq, float* dbk,
                               float* dtheta, void* ws, size_t ws_bytes, onedf_stream_t stream) {
    onedf_status s = validate(p);
    if (s != ONEDF_OK) return s;
    if (d_model < 1) return ONEDF_ERR_INVALID_ARG;
    if (!ws || (((uintptr_t)ws) & 255) != 0 || ws_bytes < onedf_project_workspace_size(p, d_model))
        return ONEDF_ERR_WORKSPACE;
    if ((s = check_device()) != ONEDF_OK) return s;
    if (!X || !Wq || !Wk || !dQ || !dK || !dWq || !dWk || (dtheta && (!theta || !d_eps))) return ONEDF_ERR_INVALID_ARG;
    if (dX && 2 * p->H * p->d_k > 128) return ONEDF_ERR_UNSUPPORTED;    // dX stages all 2 H d_k columns on chip
    return finish(launch_project_bwd(p, d_model, X, Wq, Wk, theta, dQ, dK, d_eps, dX, dWq, dWk, dbq, dbk, dtheta, ws,
                                     (cudaStream_t)stream));
}

int32_t onedf_shard_owner(int64_t chunk, int32_t world) {
    if (world <= 1 || chunk < 0) return 0;
    return Shard::owner(chunk, world);
}

onedf_status onedf_bounds_partial(const onedf_problem* p, const float* Q, const float* K, double* lohi, void* ws,
                                  size_t ws_bytes, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_ENCODE);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !lohi) return ONEDF_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (zero_flags(ws, ONEDF_OP_ENCODE, st) != cudaSuccess) return finish(cudaGetLastError());
    Carver c(ws);
    return finish(launch_bounds_partial(p, Q, K, lohi, ws, &c, st));
}

onedf_status onedf_bounds_finish(const onedf_problem* p, double* lohi, void* ws, size_t ws_bytes,
                                 onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_ENCODE);
    if (s != ONEDF_OK) return s;
    if (!lohi) return ONEDF_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (zero_flags(ws, ONEDF_OP_ENCODE, st) != cudaSuccess) return finish(cudaGetLastError());
    return finish(launch_bounds_finish(p, lohi, ws, st));
}

onedf_status onedf_rank_sum(const float* parts, int64_t n, int32_t world, float* out, onedf_stream_t stream) {
    if (!parts || !out || n < 0 || world < 1) return ONEDF_ERR_INVALID_ARG;
    onedf_status s = check_device();
    if (s != ONEDF_OK) return s;
    return finish(launch_rank_sum(parts, n, world, out, (cudaStream_t)stream));
}

onedf_status onedf_code_knn(const onedf_problem* p, const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                            int32_t exclude_self, int32_t* idx, onedf_stream_t stream) {
    onedf_status s = validate(p);
    if (s != ONEDF_OK) return s;
    if (p->causal) return ONEDF_ERR_UNSUPPORTED;
    if (!qcode || !scode || !perm || !idx) return ONEDF_ERR_INVALID_ARG;
    if ((s = check_device()) != ONEDF_OK) return s;
    return finish(launch_code_knn(p, qcode, scode, perm, exclude_self ? 1 : 0, idx, (cudaStream_t)stream));
}

onedf_status onedf_overlap(const int32_t* a, int32_t ka, const int32_t* b, int32_t kb, int64_t rows,
                           int64_t self_period, int32_t* counts, onedf_stream_t stream) {
    if (!a || !b || !counts || ka < 1 || kb < 1 || rows < 0) return ONEDF_ERR_INVALID_ARG;
    onedf_status s = check_device();
    if (s != ONEDF_OK) return s;
    return finish(launch_overlap(a, ka, b, kb, rows, self_period, counts, (cudaStream_t)stream));
}

onedf_status onedf_check_device_status(const void* ws, onedf_stream_t stream) {
    if (!ws) return ONEDF_ERR_INVALID_ARG;
    unsigned flags[FLAG_WORDS] = {0, 0, 0, 0};
    if (cudaMemcpyAsync(flags, ws, sizeof(flags), cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
        cudaGetLastError();
        return ONEDF_ERR_CUDA;
    }
    unsigned any = 0;
    for (int w = 0; w < FLAG_WORDS; ++w) any |= flags[w];
    return any ? ONEDF_ERR_NONFINITE : ONEDF_OK;
}

const char* onedf_status_string(onedf_status s) {
    switch (s) {
        case ONEDF_OK: return "ok";
        case ONEDF_ERR_INVALID_ARG: return "invalid argument";
        case ONEDF_ERR_UNSUPPORTED: return "unsupported (device is not sm_100, or size beyond this build)";
        case ONEDF_ERR_CUDA: return "CUDA error";
        case ONEDF_ERR_NONFINITE: return "non-finite input or eps <= 0 detected on device";
        case ONEDF_ERR_WORKSPACE: return "workspace missing, misaligned or too small";
        default: return "unknown status";
    }
}

int onedf_version(void) { return ONEDF_VERSION; }

}  // extern "C"
