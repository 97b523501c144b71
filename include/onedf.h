/*
 * onedf.h -- C ABI of the B200-native (sm_100a) ZETA top-k attention hot path.
 *
 * ZETA / "1DFormer" (arXiv 2501.14577).  Citations: "P:n" = PAPER.md line n
 * (final draft D unless noted), "S:n" = SPEC.md line n, "Dk" = reading k in
 * DESIGN.md ("Readings").  The operation each entry point performs is defined
 * in DESIGN.md section "Path" and, bit for bit / within the stated tolerance,
 * by the CPU oracle under oracle/ (test infrastructure, never linked here).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * Ownership.  Every pointer except the onedf_problem* is CALLER-OWNED DEVICE
 *   memory (allocated e.g. by PyTorch's caching allocator), except the
 *   host-buffer entry point onedf_topk_attn_step_host which says otherwise.
 *   The library never allocates, frees or synchronises.
 * Layout.  Contiguous row-major, fastest in the last dimension:
 *   Q, K            float  [B, H, N, d_k]
 *   V, O, dO, dV    [B, H, N, d_v] of the VALUE STORAGE TYPE p->vdtype:
 *                   float (ONEDF_DTYPE_F32) or bfloat16 (ONEDF_DTYPE_BF16,
 *                   SURVEY 8(f) NEXT-4); every sum over them is accumulated in
 *                   f64 whatever the storage type (reading D26)
 *   qcode, kcode    uint64 [B, H, N]        Morton codes (d_k*b bits used)
 *   scode, perm     uint64 / int32 [B, H, N]  chunk-major sorted runs: run c
 *                   occupies positions [c*M, min((c+1)*M, N)) of each (b,h)
 *                   row, sorted by (code, original position); perm holds the
 *                   original positions.  Non-causal: one run of N.
 *   lohi            double [B, H, 2, d_k]   per-dim (lo[d_k], hi[d_k])
 *   idx             int32  [B, H, N, k]     ascending by (D, j), -1 padded
 *   Z               float  [B, H, N]        Cauchy normaliser incl. mean slot
 * Streams.  Every launch goes on `stream` (a cudaStream_t; NULL = legacy
 *   default stream).  No global mutable state: calls on different streams
 *   with disjoint workspaces are thread-safe.
 * Errors.  Argument checks are synchronous and happen before any launch:
 *   ONEDF_ERR_INVALID_ARG   a field out of range (see onedf_validate) or a
 *                           NULL required pointer;
 *   ONEDF_ERR_WORKSPACE     ws_bytes < onedf_workspace_size(p, op) or ws NULL;
 *   ONEDF_ERR_UNSUPPORTED   current device is not sm_100 (B200), or a size
 *                           beyond what this build implements (see validate);
 *   ONEDF_ERR_CUDA          a launch failed (cudaGetLastError).
 *   Data errors detected on the device (non-finite Q/K in encode; eps <= 0 or
 *   non-finite in fwd/bwd) set flag bits in the workspace header: one 32-bit
 *   word per op (bytes [4*op, 4*op+4), op = ONEDF_OP_ENCODE .. ONEDF_OP_BWD),
 *   each zeroed only when that op starts, so one workspace shared by the whole
 *   pipeline keeps every op's flags until that op runs again.  Zero these 16
 *   bytes once when a workspace is allocated (the rest of a workspace needs
 *   no initialisation); onedf_topk_attn_step_host zeroes them itself.
 *   onedf_check_device_status(ws) synchronises the stream and reports any set
 *   flag as ONEDF_ERR_NONFINITE.  No exceptions cross the ABI.
 * Determinism.  Every output is bitwise reproducible run to run: no float
 *   atomics anywhere; every reduction has a fixed order.
 */
#ifndef ONEDF_H
#define ONEDF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ONEDF_VERSION 600

typedef struct CUstream_st* onedf_stream_t;   /* == cudaStream_t */

typedef enum {
    ONEDF_OK = 0,
    ONEDF_ERR_INVALID_ARG = 1,
    ONEDF_ERR_UNSUPPORTED = 2,
    ONEDF_ERR_CUDA = 3,
    ONEDF_ERR_NONFINITE = 4,
    ONEDF_ERR_WORKSPACE = 5
} onedf_status;

/* The paper's problem statement (Alg. "KwData" P:1778: keys, sequence length
 * N, chunk size M, top-k value k; Q, K in R^{B x N x d_K}, V in R^{B x N x d_V}
 * P:1329; causal masks P:1335; trainable Cauchy scale P:1361). */
typedef struct {
    int64_t B, H, N;     /* batch, heads, positions; 1 <= N, N*k < 2^31            */
    int32_t d_k, d_v;    /* 1 <= d_k <= 8 ; 4 <= d_v <= 256, d_v % 4 == 0             */
    int32_t k;           /* 1 <= k <= 256 : neighbours kept (|I_q|)            */
    int32_t window;      /* W >= k : candidates per sorted run; 0 -> 2k (D1)   */
    int32_t chunk;       /* M >= 1 : causal chunk size; ignored if !causal    */
    int32_t bits;        /* b : bits per dim, d_k*b <= 63, b <= 32; 0 -> min(63/d_k,32) */
    int32_t causal;      /* 1: key j visible to query i iff j < floor(i/M)*M (D6); 0: all */
    int32_t mean_slot;   /* 1: append the prefix-mean token (D8); 0: off      */
    int32_t shard_rank;  /* sequence sharding (NEXT-1, see "Sequence sharding" below): */
    int32_t shard_world; /*   this rank of shard_world; shard_world 0 or 1 = unsharded  */
    int32_t score;       /* attention weight S(q, k) of a selected slot (reading D24):  */
                         /*   ONEDF_SCORE_CAUCHY 1/(D + eps) (Eq. 5, the method)        */
                         /*   ONEDF_SCORE_NEG_EUCLID exp(-D), ONEDF_SCORE_INV_EUCLID    */
                         /*   1/(sqrt(D) + 1e-6), ONEDF_SCORE_DOT exp(q.k / sqrt(d_k))  */
    int32_t select;      /* index set of a query (reading D25): ONEDF_SELECT_EUCLID the */
                         /*   exact Euclidean top-k of the candidate windows (D5, the   */
                         /*   method); ONEDF_SELECT_CODE SPEC's code-distance merge      */
    int32_t vdtype;      /* storage type of V, O, dO, dV (NEXT-4, reading D26):          */
                         /*   ONEDF_DTYPE_F32 (the method's fp32 contract) or            */
                         /*   ONEDF_DTYPE_BF16 (halves the gathered row bytes; sums f64) */
} onedf_problem;

/* Value storage types (onedf_problem.vdtype).  BF16: V and dO are read as
 * bfloat16 and widened exactly; O and dV are rounded once to bfloat16 (round
 * to nearest even) from the f64 result.  Q, K, dQ, dK, Z stay float.
 * Sequence sharding (shard_world > 1) supports F32 only (the partial dV rows
 * it exchanges would otherwise be rounded per rank). */
enum { ONEDF_DTYPE_F32 = 0, ONEDF_DTYPE_BF16 = 1 };

/* Score variants: the paper's comparison operators
 * ("Negative Euclidean, Cauchy Softmax ..., and Inverse Euclidean";
 * P:2092-2105 "Normalized Dot Prod"), formulas per SPEC S:380/S:401.  The
 * index set is the same Euclidean top-k for every score; only the
 * weights change.  Z holds sum S for CAUCHY and INV_EUCLID and log(sum S)
 * (the log-sum-exp) for NEG_EUCLID and DOT; eps is read only by CAUCHY and
 * d_eps is 0 for the others. */
enum { ONEDF_SCORE_CAUCHY = 0, ONEDF_SCORE_NEG_EUCLID = 1, ONEDF_SCORE_INV_EUCLID = 2, ONEDF_SCORE_DOT = 3 };

/* Selection variant (SPEC S:224-228 query_topk): the same
 * per-run windows (D1-D3), candidates ordered by (|scode - qcode| as u64, j)
 * instead of (D32, j); idx is emitted in that order.  Everything downstream
 * (weights, gather, backward) is unchanged. */
enum { ONEDF_SELECT_EUCLID = 0, ONEDF_SELECT_CODE = 1 };

enum {
    ONEDF_OP_ENCODE = 0,
    ONEDF_OP_SORT = 1,
    ONEDF_OP_FWD = 2,
    ONEDF_OP_BWD = 3,
    ONEDF_OP_STEP_HOST = 4
};

/* Synchronous range checks of every field (no device work). */
onedf_status onedf_validate(const onedf_problem* p);

/* Longest sorted run (M causal, N non-causal) the segmented sort keeps in
 * shared memory; longer runs sort through global scratch in the workspace
 * (onedf_workspace_size(p, ONEDF_OP_SORT) grows by 24 bytes per position). */
int64_t onedf_max_run_length(void);

/* Bytes of device workspace `op` needs (0 if the problem is invalid).  The
 * workspace must be 256-byte aligned; apart from the 16-byte flag header (see
 * "Errors") its contents need not be initialised. */
size_t onedf_workspace_size(const onedf_problem* p, int op);

/* A1 + A2: bounds and Morton encode (P:952-954 draft C quantiser, Eq. 4
 * P:1276-1280 interleave, "Q_z, K_z = Z-order(Q), Z-order(K)").
 *   lohi_in   NULL -> fit per (b,h) per dim jointly over Q and K, constant dims
 *             widened by +-0.5 (D10); else caller-fixed bounds [B,H,2,d_k].
 *   g = clamp(floor(((x - lo)/(hi - lo)) * (2^b - 1)), 0, 2^b - 1) in f64 (D9);
 *   code = bit planes MSB first, coordinate 0 first within a plane (Eq. 4).
 *   lohi_out  nullable; receives the bounds used.
 * Non-finite Q/K -> NONFINITE flag (codes of such rows are unspecified). */
onedf_status onedf_encode(const onedf_problem* p, const float* Q, const float* K,
                          const double* lohi_in, uint64_t* qcode, uint64_t* kcode,
                          double* lohi_out, void* ws, size_t ws_bytes, onedf_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-4: the upstream projections and the Cauchy scale fused
 * in front of the encoder.  P:1549 "trainable projection networks f_k and f_q"
 * map the d_model token features to d_K per head, read as one linear layer
 * per head (reading D27); "gamma^2 as the output of a sigmoid function
 * applied to a trainable parameter":
 *   q_{b,h,n} = Wq[h] x_{b,n} + bq[h],  k_{b,h,n} = Wk[h] x_{b,n} + bk[h],
 *   eps = sigma(theta) = 1 / (1 + exp(-theta)).
 * Layouts: X [B, N, d_model] float; Wq, Wk [H, d_k, d_model] float; bq, bk
 * [H, d_k] float (nullable: no bias); theta device float scalar (nullable: eps
 * not written); Q, K [B, H, N, d_k] float (outputs, then encoded exactly as by
 * onedf_encode(Q, K, lohi_in, ...)); eps device float scalar.  Sums are f64
 * over exact f32 products in a fixed order, one rounding to f32 (bitwise
 * reproducible).  Non-finite theta sets the ENCODE flag word.
 * Workspace: onedf_workspace_size(p, ONEDF_OP_ENCODE). */
onedf_status onedf_project_encode(const onedf_problem* p, int32_t d_model, const float* X,
                                  const float* Wq, const float* Wk, const float* bq, const float* bk,
                                  const float* theta, const double* lohi_in, float* Q, float* K,
                                  float* eps, uint64_t* qcode, uint64_t* kcode, double* lohi_out,
                                  void* ws, size_t ws_bytes, onedf_stream_t stream);

/* Backward of onedf_project_encode's projections (the codes are constants,
 * D16): given dQ, dK (onedf_topk_attn_bwd) and d_eps (device double),
 *   dX = sum_h Wq[h]^T dq + Wk[h]^T dk        [B, N, d_model] (nullable: skipped)
 *   dWq[h] = sum_{b,n} dq x^T, dWk likewise   [H, d_k, d_model]
 *   dbq[h] = sum_{b,n} dq, dbk likewise       [H, d_k] (nullable)
 *   dtheta = d_eps sigma(theta) (1 - sigma(theta))   device float (nullable)
 * dW/db sum fixed row groups in a fixed order (bitwise reproducible).  dX needs
 * 2 H d_k <= 128 (its kernel stages every output column on chip), else UNSUPPORTED.
 * Workspace: onedf_project_workspace_size(p, d_model). */
size_t onedf_project_workspace_size(const onedf_problem* p, int32_t d_model);
onedf_status onedf_project_bwd(const onedf_problem* p, int32_t d_model, const float* X,
                               const float* Wq, const float* Wk, const float* theta,
                               const float* dQ, const float* dK, const double* d_eps, float* dX,
                               float* dWq, float* dWk, float* dbq, float* dbk, float* dtheta,
                               void* ws, size_t ws_bytes, onedf_stream_t stream);

/* A3: segmented stable sort of key codes ("torch.sort", "radix
 * sorted", Alg. P:1786-1790 "divide the sorted keys into multiple chunks",
 * S:215-223).  Each run sorted by (code, position); scode/perm chunk-major.
 * scode may be NULL (only the permutation is written).  Applied to the QUERY
 * codes, perm is the Morton query schedule `qorder` that onedf_topk_attn_fwd
 * and _bwd accept as a scheduling hint (one sort serves both passes). */
onedf_status onedf_sort(const onedf_problem* p, const uint64_t* kcode, uint64_t* scode,
                        int32_t* perm, void* ws, size_t ws_bytes, onedf_stream_t stream);

/* A4-A7: prefix means, causal candidate search, exact top-k, Cauchy weights
 * and value gather (Eq. 5, Eq. 6).
 *   For query i: for every admissible run c (c < floor(i/M), or the single
 *   non-causal run): p_c = lower_bound(run_c, qcode_i) (D3), w = min(W, len),
 *   s = min(max(p_c - floor(W/2), 0), len - w) (D2); candidates = union of
 *   run_c[s, s+w).  I_i = first min(k, #candidates) by (D32, j) where D32 is
 *   the f32 squared distance summed left to right without FMA (D23).
 *   S_ij = 1/(||q_i - k_j||^2 + eps) (f64), mean slot S_imu with the inclusive
 *   prefix means (D8), Z_i = sum S, o_i = sum (S/Z) v.  Chunk-0 queries with
 *   mean_slot == 0: o = 0, Z = 0, idx = -1 (D7).
 *   eps       device float scalar, eps > 0 and finite (else NONFINITE flag).
 *   qorder    nullable scheduling hint [B,H,N] int32: onedf_sort's perm of the
 *             QUERY codes (per chunk, positions by (qcode, i)).  Queries are
 *             visited in that order (Morton-adjacent queries share candidate
 *             records and V rows in L1); NULL -> the forward sorts qcode
 *             itself.  Any per-chunk permutation gives bitwise the same outputs.
 *   O, idx, Z outputs (idx/Z are what onedf_topk_attn_bwd consumes).
 *   indeg     nullable output [B,H,N] int32 (caller-owned device memory): the in-degree
 *             of every key, #{(i, slot): idx[i][slot] == j} over this call's queries
 *             (A9's counts, exact integers: one atomic add per selected slot in the
 *             top-k kernel).  Pass it to onedf_topk_attn_bwd with the same idx to skip
 *             the backward's counting pass over idx.
 *   means     nullable output, caller-owned device memory of onedf_means_floats(p) f32:
 *             the inclusive prefix means of A4 (D8) -- Kbar [B,H,rows,d_k] followed by
 *             Vbar [B,H,rows,d_v], rows = N (causal) or 1 -- written there instead of the
 *             workspace.  Pass it to onedf_topk_attn_bwd (same K, V) to skip recomputing
 *             them.  Ignored when mean_slot == 0. */
onedf_status onedf_topk_attn_fwd(const onedf_problem* p, const float* Q, const float* K,
                                 const void* V, const float* eps, const uint64_t* qcode,
                                 const uint64_t* scode, const int32_t* perm, const int32_t* qorder,
                                 void* O, int32_t* idx, float* Z, int32_t* indeg, float* means,
                                 void* ws, size_t ws_bytes, onedf_stream_t stream);
/* Floats of the `means` buffer: B*H*rows*(d_k + d_v) (0 when mean_slot == 0). */
int64_t onedf_means_floats(const onedf_problem* p);

/* A8-A12: backward with I held fixed (D16), appendix P:2006-2045 with the
 * dot-product reading D15, the mean-slot chain rule (S:323(a)) and one shared
 * eps (D20).  dK/dV accumulate through a key-major CSR of the selected
 * (query, slot) records (integer in-degree counts and cursors) and f64 segment
 * sums in ascending query order -- no float atomics, bitwise reproducible.
 *   O, Z, idx  the forward's outputs for the same inputs.  Only idx is read:
 *              the backward recomputes the normaliser Z and c_i = dO_i . o_i
 *              in f64 from the per-slot dots dO_i . v_j (reading R3), so no
 *              f32-rounded forward value enters g_ij = (dO_i.v_j - c_i)/Z_i;
 *              O and Z stay in the signature for interface stability.
 *   qcode      nullable scheduling hint: the forward's query codes.  When
 *              given, queries are visited in Morton order per chunk (better
 *              L1 reuse of the gathered V rows); outputs are bitwise the same.
 *   qorder     nullable scheduling hint: the query schedule itself (onedf_sort
 *              of qcode, as passed to the forward); wins over qcode and saves
 *              re-sorting it.  Outputs are bitwise the same.
 *   perm       nullable scheduling hint: onedf_sort's perm.  When given, keys
 *              are visited in sorted-run order; outputs are bitwise the same.
 *   indeg      nullable: the in-degree counts onedf_topk_attn_fwd wrote for THIS idx
 *              (same problem, same shard); they size the CSR segments instead of a
 *              counting pass over idx.  Counts that do not match idx are a caller
 *              error (records would land in the wrong segments); outputs are bitwise
 *              the same as with NULL.
 *   means      nullable: the prefix means onedf_topk_attn_fwd wrote for the same K, V
 *              (read only); NULL recomputes them.  Outputs are bitwise the same.
 *   dQ, dK     overwritten (f32); dV overwritten (p->vdtype); d_eps device DOUBLE scalar, overwritten with
 *   the sum over all (b,h,i). */
onedf_status onedf_topk_attn_bwd(const onedf_problem* p, const float* Q, const float* K,
                                 const void* V, const float* eps, const void* O,
                                 const void* dO, const int32_t* idx, const float* Z,
                                 const uint64_t* qcode, const int32_t* qorder, const int32_t* perm,
                                 const int32_t* indeg, const float* means, float* dQ, float* dK,
                                 void* dV, double* d_eps, void* ws, size_t ws_bytes,
                                 onedf_stream_t stream);

/* Instrumented twins of the fwd/bwd calls: identical launches and results,
 * plus cudaEventRecord(events[s], stream) right after internal stage s
 * (entries at s >= n_events, or NULL entries, are skipped).  `events` holds
 * caller-created cudaEvent_t handles.  Stages:
 *   fwd: 0 prefix means (A4)  1 sorted key records (K4)  2 top-k attention (A5-A7)
 *   bwd: 0 prefix means (A4)  1 transpose: in-degree CSR (A9)  2 query side (A8)
 *        3 key side (A10, incl. the ordering of long CSR segments)  4 mean-slot scan (A11)
 *        5 eps reduce (A12)    */
onedf_status onedf_topk_attn_fwd_traced(const onedf_problem* p, const float* Q, const float* K,
                                        const void* V, const float* eps, const uint64_t* qcode,
                                        const uint64_t* scode, const int32_t* perm,
                                        const int32_t* qorder, void* O,
                                        int32_t* idx, float* Z, int32_t* indeg, float* means, void* ws,
                                        size_t ws_bytes, void* const* events, int n_events,
                                        onedf_stream_t stream);
onedf_status onedf_topk_attn_bwd_traced(const onedf_problem* p, const float* Q, const float* K,
                                        const void* V, const float* eps, const void* O,
                                        const void* dO, const int32_t* idx, const float* Z,
                                        const uint64_t* qcode, const int32_t* qorder,
                                        const int32_t* perm, const int32_t* indeg, const float* means,
                                        float* dQ, float* dK, void* dV, double* d_eps,
                                        void* ws, size_t ws_bytes, void* const* events, int n_events,
                                        onedf_stream_t stream);

/* End-to-end training step from HOST buffers (the user-facing call the e2e
 * metric times): async H2D copies of Q, K, V, dO (host pointers; pinned for
 * full speed), then encode -> sort -> fwd -> bwd on the device, then async
 * D2H copies of O, dQ, dK, dV (host pointers) and d_eps (host double*).
 * The (b,h) slices are processed in up to 8 groups: the H2D copy of the next
 * group and the D2H copy of the previous one run on two internal streams
 * (created and released by the call, ordered by events) while `stream`
 * computes the current group, so PCIe traffic overlaps the kernels.  Every
 * slice's outputs equal the device path's bit for bit; d_eps is the groups'
 * partial sums added in group order.
 * V_h, dO_h, O_h, dV_h are of the storage type p->vdtype (bf16 halves their
 * PCIe bytes).  The query codes are sorted once per group and the schedule
 * serves both passes.
 * eps is passed by value.  All device buffers live in `ws` (device,
 * onedf_workspace_size(p, ONEDF_OP_STEP_HOST) bytes).  Returns after
 * enqueueing; synchronise `stream` before reading the host outputs. */
onedf_status onedf_topk_attn_step_host(const onedf_problem* p, const float* Q_h, const float* K_h,
                                       const void* V_h, float eps, const void* dO_h,
                                       void* O_h, float* dQ_h, float* dK_h, void* dV_h,
                                       double* d_eps_h, void* ws, size_t ws_bytes,
                                       onedf_stream_t stream);

/* ---------------------------------------------------------------------------
 * Sequence sharding (north_star "sequence sharding, with
 * an NCCL all-gather over NVLink of the earlier ranks' sorted Morton runs").
 * Causal problems only (shard_world > 1 with causal == 0 -> UNSUPPORTED).
 * The C = ceil(N/M) chunks of every (b,h) are dealt zig-zag over the
 * shard_world ranks: chunk c belongs to rank onedf_shard_owner(c, world)
 * (g = c mod 2*world; owner = g < world ? g : 2*world-1-g), so the causal work
 * (proportional to c) balances.  Every rank keeps FULL-LENGTH
 * [B,H,N,.] buffers; a rank "owns" the rows of its chunks:
 *   onedf_bounds_partial   raw per-dim min/max over the owned rows of Q and K;
 *                          the caller all-reduces them (MIN over lo, MAX over
 *                          hi), then onedf_bounds_finish applies D10 and the
 *                          result is onedf_encode's lohi_in (required).
 *   onedf_encode/_sort     as unsharded; only owned rows/runs are meaningful.
 *                          The caller then all-gathers the owned runs of
 *                          scode/perm and the owned rows of K and V, so that
 *                          scode, perm, K, V are complete on every rank.
 *   onedf_topk_attn_fwd    computes O, idx, Z of the OWNED queries only
 *                          (other rows are not written).
 *   onedf_topk_attn_bwd    dQ of the owned queries; dK, dV and d_eps are this
 *                          rank's PARTIAL sums over its owned queries (all N
 *                          rows written); the caller exchanges the partial rows
 *                          to their owners and sums them in rank order with
 *                          onedf_rank_sum (deterministic), and sums d_eps in
 *                          rank order.
 * Non-owned rows of Q and dO must hold finite values (e.g. zeros); they are
 * never read into a result but pass through the mean-slot scans with a zero
 * coefficient. */
int32_t onedf_shard_owner(int64_t chunk, int32_t world);

/* Raw min (lohi[...,0,:]) and max (lohi[...,1,:]) per (b,h) per dim over the
 * owned rows of Q and K (all rows if unsharded); no widening.  lohi: device
 * double [B,H,2,d_k], overwritten.  Non-finite input -> NONFINITE flag.
 * Workspace: onedf_workspace_size(p, ONEDF_OP_ENCODE). */
onedf_status onedf_bounds_partial(const onedf_problem* p, const float* Q, const float* K,
                                  double* lohi, void* ws, size_t ws_bytes, onedf_stream_t stream);

/* D10 in place: a dim with hi == lo becomes [lo - 0.5, hi + 0.5]; non-finite
 * or hi < lo -> NONFINITE flag.  onedf_encode(lohi_in = NULL) is exactly
 * bounds_partial -> bounds_finish -> encode(lohi_in). */
onedf_status onedf_bounds_finish(const onedf_problem* p, double* lohi, void* ws, size_t ws_bytes,
                                 onedf_stream_t stream);

/* out[x] = (float) sum_{r = 0 .. world-1} (double) parts[r*n + x], summed in
 * rank order r = 0, 1, ... (the fixed-order combine of the sharded dK/dV
 * partials).  parts: device float [world][n]; out: device float [n]. */
onedf_status onedf_rank_sum(const float* parts, int64_t n, int32_t world, float* out,
                            onedf_stream_t stream);

/* ---------------------------------------------------------------------------
 * Locality / recall workload (Fig. 4 P:1561-1581 "overlap
 * between the top-64 nearest neighbors before and after projection"; the k
 * ablation P:1583-1587).
 *
 * onedf_code_knn: for every query i, the k keys nearest in Morton code,
 *   ordered by (|kcode_j - qcode_i| as u64, j) ascending (ties by position,
 *   D19), -1 padded; exclude_self != 0 drops j == i.  Reads qcode and the
 *   sorted run (scode, perm) of onedf_encode/onedf_sort.  Non-causal problems
 *   only (causal -> UNSUPPORTED).  idx: device int32 [B,H,N,k].  No workspace.
 * onedf_overlap: counts[r] = |{a[r][x] : a[r][x] >= 0, a[r][x] != r mod
 *   self_period (if self_period > 0)} ∩ {b[r][y]}| for r < rows, each index
 *   counted once; a [rows, ka], b [rows, kb] device int32, counts device
 *   int32 [rows].  The Fig. 4 metric is counts / k. */
onedf_status onedf_code_knn(const onedf_problem* p, const uint64_t* qcode, const uint64_t* scode,
                            const int32_t* perm, int32_t exclude_self, int32_t* idx, onedf_stream_t stream);
onedf_status onedf_overlap(const int32_t* a, int32_t ka, const int32_t* b, int32_t kb, int64_t rows,
                           int64_t self_period, int32_t* counts, onedf_stream_t stream);

/* Synchronises `stream`, then reads the flag words of `ws` (a workspace
 * previously passed to encode/sort/fwd/bwd; see "Errors"): ONEDF_OK, or
 * ONEDF_ERR_NONFINITE if any op's flag is set. */
onedf_status onedf_check_device_status(const void* ws, onedf_stream_t stream);

const char* onedf_status_string(onedf_status s);
int onedf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ONEDF_H */
