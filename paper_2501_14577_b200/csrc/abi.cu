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
    if (p->shard_world > 1) {
        if (p->shard_rank < 0 || p->shard_rank >= p->shard_world) return ONEDF_ERR_INVALID_ARG;
        if (!p->causal) return ONEDF_ERR_UNSUPPORTED;   // sequence sharding is defined over causal chunks
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

struct StepLayout {
    float *Q, *K, *V, *dO, *O, *dQ, *dK, *dV, *Z, *eps;
    double* d_eps;
    uint64_t *qcode, *kcode, *scode;
    int32_t *perm, *idx;
    size_t sub_off, sub_bytes, bytes;
};
static StepLayout step_layout(const onedf_problem* p, void* ws) {
    StepLayout L;
    const size_t e = encode_bytes(p), s = sort_bytes(p);
    const size_t f = fwd_layout(p, nullptr).bytes, b = bwd_layout(p, nullptr).bytes;
    size_t sub = e > s ? e : s;
    sub = sub > f ? sub : f;
    sub = sub > b ? sub : b;
    Carver c(ws);
    const int64_t BH = p->B * p->H, N = p->N, nk = BH * N * p->d_k, nv = BH * N * p->d_v;
    L.Q = c.take<float>(nk); L.K = c.take<float>(nk); L.V = c.take<float>(nv); L.dO = c.take<float>(nv);
    L.O = c.take<float>(nv); L.dQ = c.take<float>(nk); L.dK = c.take<float>(nk); L.dV = c.take<float>(nv);
    L.Z = c.take<float>(BH * N); L.eps = c.take<float>(1); L.d_eps = c.take<double>(1);
    L.qcode = c.take<uint64_t>(BH * N); L.kcode = c.take<uint64_t>(BH * N); L.scode = c.take<uint64_t>(BH * N);
    L.perm = c.take<int32_t>(BH * N); L.idx = c.take<int32_t>(BH * N * p->k);
    c.take<char>(0);
    L.sub_off = c.off;
    L.sub_bytes = sub;
    c.take<char>(sub);
    L.bytes = c.bytes();
    return L;
}

__global__ void set_scalar_kernel(float* dst, float v) { *dst = v; }

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

// Internal entry points (flag zeroing optional so the host step can chain them).
static onedf_status do_encode(const onedf_problem* p, const float* Q, const float* K, const double* lohi_in,
                              uint64_t* qcode, uint64_t* kcode, double* lohi_out, void* ws, cudaStream_t st,
                              bool zero) {
    if (zero && cudaMemsetAsync(ws, 0, 4, st) != cudaSuccess) return finish(cudaGetLastError());
    Carver c(ws);
    return finish(launch_encode(p, effective_bits(p), Q, K, lohi_in, qcode, kcode, lohi_out, ws, &c, st));
}
static onedf_status do_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm,
                            void* ws, cudaStream_t st) {
    Carver c(ws);
    SortScratch scr;
    sort_carve(p, &c, &scr);
    return finish(launch_seg_sort(p, kcode, scode, perm, scr, st));
}
static onedf_status do_fwd(const onedf_problem* p, const float* Q, const float* K, const float* V, const float* eps,
                           const uint64_t* qcode, const uint64_t* scode, const int32_t* perm, float* O, int32_t* idx,
                           float* Z, void* ws, cudaStream_t st, bool zero, const Trace& tr = Trace()) {
    if (zero && cudaMemsetAsync(ws, 0, 4, st) != cudaSuccess) return finish(cudaGetLastError());
    FwdLayout L = fwd_layout(p, ws);
    cudaError_t e = cudaSuccess;
    if (p->mean_slot) e = launch_prefix_means(p, K, V, &L.m, st);
    tr.mark(0, st);
    if (e == cudaSuccess) e = launch_fwd(p, Q, K, V, eps, qcode, scode, perm, O, idx, Z, &L.m, &L.f, ws, st, tr);
    return finish(e);
}
static onedf_status do_bwd(const onedf_problem* p, const float* Q, const float* K, const float* V, const float* eps,
                           const float* O, const float* dO, const int32_t* idx, const float* Z, const uint64_t* qcode,
                           const int32_t* perm, float* dQ, float* dK, float* dV, double* d_eps, void* ws,
                           cudaStream_t st, bool zero, const Trace& tr = Trace()) {
    if (zero && cudaMemsetAsync(ws, 0, 4, st) != cudaSuccess) return finish(cudaGetLastError());
    BwdLayout L = bwd_layout(p, ws);
    cudaError_t e = cudaSuccess;
    if (p->mean_slot) e = launch_prefix_means(p, K, V, &L.m, st);
    tr.mark(0, st);
    if (e == cudaSuccess)
        e = launch_bwd(p, Q, K, V, eps, O, dO, idx, Z, qcode, perm, dQ, dK, dV, d_eps, &L.m, &L.b, &L.t, ws, st, tr);
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
    if (!kcode || !scode || !perm) return ONEDF_ERR_INVALID_ARG;
    if (cudaMemsetAsync(ws, 0, 4, (cudaStream_t)stream) != cudaSuccess) return finish(cudaGetLastError());
    return do_sort(p, kcode, scode, perm, ws, (cudaStream_t)stream);
}

onedf_status onedf_topk_attn_fwd(const onedf_problem* p, const float* Q, const float* K, const float* V,
                                 const float* eps, const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                                 float* O, int32_t* idx, float* Z, void* ws, size_t ws_bytes, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_FWD);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !V || !eps || !qcode || !scode || !perm || !O || !idx || !Z) return ONEDF_ERR_INVALID_ARG;
    if ((((uintptr_t)V) | ((uintptr_t)O)) & 15) return ONEDF_ERR_INVALID_ARG;
    return do_fwd(p, Q, K, V, eps, qcode, scode, perm, O, idx, Z, ws, (cudaStream_t)stream, true);
}

onedf_status onedf_topk_attn_bwd(const onedf_problem* p, const float* Q, const float* K, const float* V,
                                 const float* eps, const float* O, const float* dO, const int32_t* idx,
                                 const float* Z, const uint64_t* qcode, const int32_t* perm, float* dQ, float* dK,
                                 float* dV, double* d_eps, void* ws, size_t ws_bytes, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_BWD);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !V || !eps || !O || !dO || !idx || !Z || !dQ || !dK || !dV || !d_eps)
        return ONEDF_ERR_INVALID_ARG;
    if ((((uintptr_t)V) | ((uintptr_t)dO) | ((uintptr_t)dV)) & 15) return ONEDF_ERR_INVALID_ARG;
    return do_bwd(p, Q, K, V, eps, O, dO, idx, Z, qcode, perm, dQ, dK, dV, d_eps, ws, (cudaStream_t)stream, true);
}

onedf_status onedf_topk_attn_fwd_traced(const onedf_problem* p, const float* Q, const float* K, const float* V,
                                        const float* eps, const uint64_t* qcode, const uint64_t* scode,
                                        const int32_t* perm, float* O, int32_t* idx, float* Z, void* ws,
                                        size_t ws_bytes, void* const* events, int n_events, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_FWD);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !V || !eps || !qcode || !scode || !perm || !O || !idx || !Z) return ONEDF_ERR_INVALID_ARG;
    if ((((uintptr_t)V) | ((uintptr_t)O)) & 15) return ONEDF_ERR_INVALID_ARG;
    Trace tr;
    tr.ev = events;
    tr.n = n_events;
    return do_fwd(p, Q, K, V, eps, qcode, scode, perm, O, idx, Z, ws, (cudaStream_t)stream, true, tr);
}

onedf_status onedf_topk_attn_bwd_traced(const onedf_problem* p, const float* Q, const float* K, const float* V,
                                        const float* eps, const float* O, const float* dO, const int32_t* idx,
                                        const float* Z, const uint64_t* qcode, const int32_t* perm, float* dQ,
                                        float* dK, float* dV, double* d_eps, void* ws, size_t ws_bytes,
                                        void* const* events, int n_events, onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_BWD);
    if (s != ONEDF_OK) return s;
    if (!Q || !K || !V || !eps || !O || !dO || !idx || !Z || !dQ || !dK || !dV || !d_eps)
        return ONEDF_ERR_INVALID_ARG;
    if ((((uintptr_t)V) | ((uintptr_t)dO) | ((uintptr_t)dV)) & 15) return ONEDF_ERR_INVALID_ARG;
    Trace tr;
    tr.ev = events;
    tr.n = n_events;
    return do_bwd(p, Q, K, V, eps, O, dO, idx, Z, qcode, perm, dQ, dK, dV, d_eps, ws, (cudaStream_t)stream, true,
                  tr);
}

onedf_status onedf_topk_attn_step_host(const onedf_problem* p, const float* Q_h, const float* K_h, const float* V_h,
                                       float eps, const float* dO_h, float* O_h, float* dQ_h, float* dK_h,
                                       float* dV_h, double* d_eps_h, void* ws, size_t ws_bytes,
                                       onedf_stream_t stream) {
    if (validate(p) == ONEDF_OK && p->shard_world > 1) return ONEDF_ERR_UNSUPPORTED;   // needs the caller's collectives
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_STEP_HOST);
    if (s != ONEDF_OK) return s;
    if (!Q_h || !K_h || !V_h || !dO_h || !O_h || !dQ_h || !dK_h || !dV_h || !d_eps_h) return ONEDF_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    StepLayout L = step_layout(p, ws);
    void* sub = (char*)ws + L.sub_off;
    const int64_t BH = p->B * p->H, N = p->N;
    const size_t bk = (size_t)(BH * N * p->d_k) * 4, bv = (size_t)(BH * N * p->d_v) * 4;
    cudaError_t e = cudaMemsetAsync(ws, 0, 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(sub, 0, 4, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(L.Q, Q_h, bk, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(L.K, K_h, bk, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(L.V, V_h, bv, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(L.dO, dO_h, bv, cudaMemcpyHostToDevice, st);
    // eps by value: written by a one-thread kernel so the call needs no host staging buffer
    if (e == cudaSuccess) {
        set_scalar_kernel<<<1, 1, 0, st>>>(L.eps, eps);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return finish(e);
    if ((s = do_encode(p, L.Q, L.K, nullptr, L.qcode, L.kcode, nullptr, sub, st, false)) != ONEDF_OK) return s;
    if ((s = do_sort(p, L.kcode, L.scode, L.perm, sub, st)) != ONEDF_OK) return s;
    if ((s = do_fwd(p, L.Q, L.K, L.V, L.eps, L.qcode, L.scode, L.perm, L.O, L.idx, L.Z, sub, st, false)) != ONEDF_OK)
        return s;
    if ((s = do_bwd(p, L.Q, L.K, L.V, L.eps, L.O, L.dO, L.idx, L.Z, L.qcode, L.perm, L.dQ, L.dK, L.dV, L.d_eps, sub,
                    st, false)) !=
        ONEDF_OK)
        return s;
    e = cudaMemcpyAsync(ws, sub, 4, cudaMemcpyDeviceToDevice, st);   // surface device flags in the caller's header
    if (e == cudaSuccess) e = cudaMemcpyAsync(O_h, L.O, bv, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dQ_h, L.dQ, bk, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dK_h, L.dK, bk, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dV_h, L.dV, bv, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_eps_h, L.d_eps, 8, cudaMemcpyDeviceToHost, st);
    return finish(e);
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
    if (cudaMemsetAsync(ws, 0, 4, st) != cudaSuccess) return finish(cudaGetLastError());
    Carver c(ws);
    return finish(launch_bounds_partial(p, Q, K, lohi, ws, &c, st));
}

onedf_status onedf_bounds_finish(const onedf_problem* p, double* lohi, void* ws, size_t ws_bytes,
                                 onedf_stream_t stream) {
    onedf_status s = pre(p, ws, ws_bytes, ONEDF_OP_ENCODE);
    if (s != ONEDF_OK) return s;
    if (!lohi) return ONEDF_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(ws, 0, 4, st) != cudaSuccess) return finish(cudaGetLastError());
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
    unsigned flags = 0;
    if (cudaMemcpyAsync(&flags, ws, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
        cudaGetLastError();
        return ONEDF_ERR_CUDA;
    }
    return flags ? ONEDF_ERR_NONFINITE : ONEDF_OK;
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
