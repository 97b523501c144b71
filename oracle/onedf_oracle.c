/*
 * onedf_oracle.c -- plain, slow, obviously-correct CPU oracle for the ZETA
 * (arXiv 2501.14577, early-draft name "1DFormer") causal top-k attention path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2501_14577_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Citation convention: "P:n" = /root/reference/PAPER.md line n (draft D, the
 * final paper, unless noted), "S:n" = SPEC.md line n, "Dk" = reading k listed
 * in DESIGN.md section "Readings".  Every function follows the algorithm step
 * by step in the paper's order; there is no blocking, fusion or reordering.
 *
 * Precision: all arithmetic is IEEE f64 (compiled with -ffp-contract=off, no
 * fast-math), EXCEPT the one place where floating point decides an integer
 * result inside the method: the ranking distance used to pick the top-k set
 * (step "Select").  There both the oracle and the CUDA path take the decision
 * in the kernel's precision, f32, with the pinned operation order
 *   D32 = ((0 + t_0*t_0) + t_1*t_1) + ... ,  t_d = q_d - k_d   (f32, no FMA)
 * so that the selected index sets are comparable bit-exactly (reading D23).
 * Quantisation (another float->integer decision) is f64 on both sides (D9).
 *
 * Parity pins: see tests/test_oracle_pins.py; nothing here is "parity
 * unpinned" except what DESIGN.md lists.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* Mirrors the *meaning* of the ABI's problem struct;
 * declared independently here on purpose (no shared headers). */
typedef struct {
    int64_t B, H, N;
    int32_t d_k, d_v;
    int32_t k;
    int32_t window;     /* W; 0 -> 2k (D1) */
    int32_t chunk;      /* M (causal only) */
    int32_t bits;       /* b; 0 -> min(floor(63/d_k), 32) (D11) */
    int32_t causal;
    int32_t mean_slot;
    int32_t score;      /* 0 Cauchy (Eq. 5); 1..3 the comparison operators (reading D24) */
    int32_t select;     /* 0 Euclidean top-k of the windows (D5); 1 SPEC's code-distance merge (D25) */
} oref_problem;

enum { OREF_OK = 0, OREF_ERR_INVALID_ARG = 1, OREF_ERR_NONFINITE = 4 };

int oref_default_bits(int d_k) {
    int b = 63 / d_k;                       /* D11 */
    return b > 32 ? 32 : b;
}

static int eff_bits(const oref_problem* p) { return p->bits ? p->bits : oref_default_bits(p->d_k); }
static int eff_window(const oref_problem* p) { return p->window ? p->window : 2 * p->k; }

/* ------------------------------------------------------------------------ */
/* Step 1: bounds.  "min(x), max(x) ... in the dataset" (draft C);
 * per (b,h), per dim, jointly over Q and K (D10); a constant
 * column is widened by +-0.5.                                        */
int oref_fit_bounds(const oref_problem* p, const float* Q, const float* K, double* lohi) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k;
    for (int64_t bh = 0; bh < BH; ++bh) {
        for (int d = 0; d < dk; ++d) {
            double lo = INFINITY, hi = -INFINITY;
            for (int64_t i = 0; i < N; ++i) {
                double q = Q[(bh * N + i) * dk + d];
                double k = K[(bh * N + i) * dk + d];
                if (!isfinite(q) || !isfinite(k)) return OREF_ERR_NONFINITE;
                if (q < lo) lo = q;
                if (q > hi) hi = q;
                if (k < lo) lo = k;
                if (k > hi) hi = k;
            }
            if (hi == lo) { lo -= 0.5; hi += 0.5; }
            lohi[bh * 2 * dk + d] = lo;
            lohi[bh * 2 * dk + dk + d] = hi;
        }
    }
    return OREF_OK;
}

/* Step 2: quantise, "floor((x - min)(2^b - 1)/(max - min))", evaluated
 * in the pinned order of reading D9: t = (x-lo)/(hi-lo); g = floor(t*(2^b-1));
 * clamp to [0, 2^b-1].                                                       */
uint64_t oref_quantize(double x, double lo, double hi, int b) {
    double t = (x - lo) / (hi - lo);
    double top = (double)((((uint64_t)1) << b) - 1);
    double g = floor(t * top);
    if (g < 0.0) g = 0.0;
    if (g > top) g = top;
    return (uint64_t)g;
}

/* Step 3: interleave, Eq. 4: Z = b_11 b_21 ... b_d1 b_12 ... b_dn,
 * i.e. most-significant bit plane first, coordinate 1 first within a plane. */
uint64_t oref_interleave(const uint64_t* g, int d, int b) {
    uint64_t code = 0;
    for (int t = b - 1; t >= 0; --t)
        for (int j = 0; j < d; ++j)
            code = (code << 1) | ((g[j] >> t) & 1u);
    return code;
}

/* Inverse of Eq. 4 (used by tests only). */
void oref_deinterleave(uint64_t code, int d, int b, uint64_t* g) {
    for (int j = 0; j < d; ++j) g[j] = 0;
    int pos = d * b - 1;
    for (int t = b - 1; t >= 0; --t)
        for (int j = 0; j < d; ++j) {
            g[j] |= ((code >> pos) & 1u) << t;
            --pos;
        }
}

static int finite_rows(const float* X, int64_t n) {
    for (int64_t i = 0; i < n; ++i) if (!isfinite(X[i])) return 0;
    return 1;
}

/* onedf_encode analogue: bounds (fit, or caller-fixed) + quantise + interleave
 * for every query and key row ("Q_z, K_z = Z-order(Q), Z-order(K)"). */
int oref_encode(const oref_problem* p, const float* Q, const float* K, const double* lohi_in,
                uint64_t* qcode, uint64_t* kcode, double* lohi_out) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k, b = eff_bits(p);
    if (dk < 1 || dk > 8 || b < 1 || b > 32 || dk * b > 63) return OREF_ERR_INVALID_ARG;
    if (!finite_rows(Q, BH * N * dk) || !finite_rows(K, BH * N * dk)) return OREF_ERR_NONFINITE;
    double* lohi = (double*)malloc(sizeof(double) * BH * 2 * dk);
    if (lohi_in) {
        memcpy(lohi, lohi_in, sizeof(double) * BH * 2 * dk);
    } else {
        int st = oref_fit_bounds(p, Q, K, lohi);
        if (st) { free(lohi); return st; }
    }
    #pragma omp parallel for schedule(static)
    for (int64_t bh = 0; bh < BH; ++bh) {
        const double* lo = lohi + bh * 2 * dk;
        const double* hi = lo + dk;
        uint64_t g[8];
        for (int64_t i = 0; i < N; ++i) {
            for (int d = 0; d < dk; ++d) g[d] = oref_quantize((double)Q[(bh * N + i) * dk + d], lo[d], hi[d], b);
            qcode[bh * N + i] = oref_interleave(g, dk, b);
            for (int d = 0; d < dk; ++d) g[d] = oref_quantize((double)K[(bh * N + i) * dk + d], lo[d], hi[d], b);
            kcode[bh * N + i] = oref_interleave(g, dk, b);
        }
    }
    if (lohi_out) memcpy(lohi_out, lohi, sizeof(double) * BH * 2 * dk);
    free(lohi);
    return OREF_OK;
}

/* ------------------------------------------------------------------------ */
/* Runs (D4, D18): causal -> run c holds positions [cM, min((c+1)M, N));
 * non-causal -> one run of all N.                                            */
static int64_t run_count(const oref_problem* p) {
    return p->causal ? (p->N + p->chunk - 1) / p->chunk : 1;
}
static void run_span(const oref_problem* p, int64_t c, int64_t* start, int64_t* len) {
    if (!p->causal) { *start = 0; *len = p->N; return; }
    int64_t s = c * p->chunk, e = s + p->chunk;
    if (e > p->N) e = p->N;
    *start = s; *len = e - s;
}

typedef struct { uint64_t code; int64_t j; } code_pos;
static int cmp_code_pos(const void* a, const void* b) {
    const code_pos* x = (const code_pos*)a; const code_pos* y = (const code_pos*)b;
    if (x->code != y->code) return x->code < y->code ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

/* Step 4: sort each run by (code, position) -- "Sort the projected one-
 * dimensional keys in ascending order ... Divide the sorted keys into multiple
 * chunks" (Alg. P:1786-1790), ties by position (D19).             */
int oref_sort(const oref_problem* p, const uint64_t* kcode, uint64_t* scode, int32_t* perm) {
    const int64_t BH = p->B * p->H, N = p->N, C = run_count(p);
    if (p->causal && p->chunk < 1) return OREF_ERR_INVALID_ARG;
    #pragma omp parallel for schedule(dynamic)
    for (int64_t bh = 0; bh < BH; ++bh) {
        code_pos* buf = (code_pos*)malloc(sizeof(code_pos) * (size_t)N);
        for (int64_t c = 0; c < C; ++c) {
            int64_t s, len;
            run_span(p, c, &s, &len);
            for (int64_t r = 0; r < len; ++r) { buf[r].code = kcode[bh * N + s + r]; buf[r].j = s + r; }
            qsort(buf, (size_t)len, sizeof(code_pos), cmp_code_pos);
            for (int64_t r = 0; r < len; ++r) {
                scode[bh * N + s + r] = buf[r].code;
                perm[bh * N + s + r] = (int32_t)buf[r].j;
            }
        }
        free(buf);
    }
    return OREF_OK;
}

/* ------------------------------------------------------------------------ */
/* Step 5: candidate window in one sorted run.  Insertion point p = number of
 * run entries with code < qcode (torch.searchsorted default 'left', D3),
 * counted EXHAUSTIVELY (no binary search, north_star "brute-force"); window
 * w = min(W, len) centred on p and clamped into the run (D1, D2).    */
int64_t oref_insertion_point(const uint64_t* run, int64_t len, uint64_t qcode) {
    int64_t cnt = 0;
    for (int64_t r = 0; r < len; ++r) cnt += (run[r] < qcode);
    return cnt;
}
void oref_window_span(int64_t pins, int64_t len, int W, int64_t* s_out, int64_t* w_out) {
    int64_t w = W < len ? W : len;
    int64_t s = pins - W / 2;
    if (s < 0) s = 0;
    if (s > len - w) s = len - w;
    *s_out = s; *w_out = w;
}

/* Ranking distance in the kernel precision (see header, D23). */
static float rank_dist32(const float* q, const float* k, int dk) {
    float acc = 0.0f;
    for (int d = 0; d < dk; ++d) {
        float t = q[d] - k[d];
        float sq = t * t;
        acc = acc + sq;
    }
    return acc;
}

typedef struct { float D; int32_t j; } cand;
static int cmp_cand(const void* a, const void* b) {
    const cand* x = (const cand*)a; const cand* y = (const cand*)b;
    if (x->D != y->D) return x->D < y->D ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

/* Steps 5+6 for one query: union of the windows of every admissible run
 * (causal: runs c < floor(i/M), P:1335 / Alg. P:1792-1797 / D6), then the
 * first min(k, |C_i|) candidates by (D, j) ascending (D5, D17, D19).
 * Writes k entries of idx_row, padded with -1.  Returns |I_i|.            */
static int select_one(const oref_problem* p, int64_t bh, int64_t i, const float* Q, const float* K,
                      const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                      cand* buf, int32_t* idx_row) {
    const int64_t N = p->N;
    const int dk = p->d_k, W = eff_window(p), k = p->k;
    int64_t nruns = p->causal ? i / p->chunk : 1;
    int64_t nc = 0;
    const uint64_t qc = qcode[bh * N + i];
    const float* q = Q + (bh * N + i) * dk;
    for (int64_t c = 0; c < nruns; ++c) {
        int64_t s0, len;
        run_span(p, c, &s0, &len);
        const uint64_t* run = scode + bh * N + s0;
        int64_t pins = oref_insertion_point(run, len, qc);
        int64_t s, w;
        oref_window_span(pins, len, W, &s, &w);
        for (int64_t r = s; r < s + w; ++r) {
            int32_t j = perm[bh * N + s0 + r];
            buf[nc].j = j;
            buf[nc].D = rank_dist32(q, K + (bh * N + j) * dk, dk);
            ++nc;
        }
    }
    qsort(buf, (size_t)nc, sizeof(cand), cmp_cand);
    int nk = nc < k ? (int)nc : k;
    for (int r = 0; r < k; ++r) idx_row[r] = r < nk ? buf[r].j : -1;
    return nk;
}

/* Selection variant (reading D25): SPEC's query_topk
 * (S:224-228): the same per-run windows (steps 5, D1-D3), "merged across
 * chunks by |code - query_code| with ties broken by smaller source_index";
 * the first min(k, |C_i|) candidates by (|scode - qcode| as u64, j).        */
typedef struct { uint64_t d; int32_t j; } code_cand2;
static int cmp_code_cand2(const void* a, const void* b) {
    const code_cand2* x = (const code_cand2*)a; const code_cand2* y = (const code_cand2*)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

static void select_one_code(const oref_problem* p, int64_t bh, int64_t i, const uint64_t* qcode,
                            const uint64_t* scode, const int32_t* perm, code_cand2* buf, int32_t* idx_row) {
    const int64_t N = p->N;
    const int W = eff_window(p), k = p->k;
    const int64_t nruns = p->causal ? i / p->chunk : 1;
    const uint64_t qc = qcode[bh * N + i];
    int64_t nc = 0;
    for (int64_t c = 0; c < nruns; ++c) {
        int64_t s0, len;
        run_span(p, c, &s0, &len);
        const uint64_t* run = scode + bh * N + s0;
        int64_t s, w;
        oref_window_span(oref_insertion_point(run, len, qc), len, W, &s, &w);
        for (int64_t r = s; r < s + w; ++r) {
            const uint64_t kc = run[r];
            buf[nc].d = kc > qc ? kc - qc : qc - kc;
            buf[nc].j = perm[bh * N + s0 + r];
            ++nc;
        }
    }
    qsort(buf, (size_t)nc, sizeof(code_cand2), cmp_code_cand2);
    for (int r = 0; r < k; ++r) idx_row[r] = r < nc ? buf[r].j : -1;
}

int oref_select_code(const oref_problem* p, const uint64_t* qcode, const uint64_t* scode, const int32_t* perm,
                     int32_t* idx) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int W = eff_window(p);
    if (p->k < 1 || W < p->k || (p->causal && p->chunk < 1)) return OREF_ERR_INVALID_ARG;
    const int64_t maxc = (p->causal ? run_count(p) : 1) * (int64_t)W;
    #pragma omp parallel
    {
        code_cand2* buf = (code_cand2*)malloc(sizeof(code_cand2) * (size_t)(maxc + 1));
        #pragma omp for schedule(dynamic, 64)
        for (int64_t t = 0; t < BH * N; ++t) select_one_code(p, t / N, t % N, qcode, scode, perm, buf, idx + t * p->k);
        free(buf);
    }
    return OREF_OK;
}

/* Selection for every query (sel == NULL) or for the n_sel flat query ids
 * sel[t] = bh*N + i; idx is [n, k].                                         */
int oref_select(const oref_problem* p, const float* Q, const float* K, const uint64_t* qcode,
                const uint64_t* scode, const int32_t* perm, int32_t* idx,
                int64_t n_sel, const int64_t* sel) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int W = eff_window(p);
    if (p->k < 1 || W < p->k || (p->causal && p->chunk < 1)) return OREF_ERR_INVALID_ARG;
    const int64_t n = sel ? n_sel : BH * N;
    const int64_t maxc = (p->causal ? run_count(p) : 1) * (int64_t)W;
    #pragma omp parallel
    {
        cand* buf = (cand*)malloc(sizeof(cand) * (size_t)(maxc + 1));
        #pragma omp for schedule(dynamic, 64)
        for (int64_t t = 0; t < n; ++t) {
            int64_t flat = sel ? sel[t] : t;
            select_one(p, flat / N, flat % N, Q, K, qcode, scode, perm, buf, idx + t * p->k);
        }
        free(buf);
    }
    return OREF_OK;
}

/* ------------------------------------------------------------------------ */
/* Mean slot (D8): inclusive prefix mean of low-dim K and of V over positions
 * 0..i "using cumsum"; non-causal: mean over all N.     */
static void prefix_means(const oref_problem* p, const float* X, int64_t bh, int width, double* out) {
    const int64_t N = p->N;
    double* acc = (double*)calloc((size_t)width, sizeof(double));
    if (p->causal) {
        for (int64_t i = 0; i < N; ++i) {
            for (int d = 0; d < width; ++d) {
                acc[d] += (double)X[(bh * N + i) * width + d];
                out[i * width + d] = acc[d] / (double)(i + 1);
            }
        }
    } else {
        for (int64_t i = 0; i < N; ++i)
            for (int d = 0; d < width; ++d) acc[d] += (double)X[(bh * N + i) * width + d];
        for (int64_t i = 0; i < N; ++i)
            for (int d = 0; d < width; ++d) out[i * width + d] = acc[d] / (double)N;
    }
    free(acc);
}

static double dist64(const float* q, const float* k, int dk) {
    double acc = 0.0;
    for (int d = 0; d < dk; ++d) { double t = (double)q[d] - (double)k[d]; acc += t * t; }
    return acc;
}
static double dist64_mean(const float* q, const double* kb, int dk) {
    double acc = 0.0;
    for (int d = 0; d < dk; ++d) { double t = (double)q[d] - kb[d]; acc += t * t; }
    return acc;
}

/* Step 8: forward with a given index set.  Eq. 5: S_ij =
 * 1/(||q_i-k_j||^2 + eps) (gamma/pi cancels, eps = gamma^2, D13-D14);
 * Eq. 6 + appendix: Z_i = sum S, A = S/Z,
 * o_i = sum A v, with the mean slot scored like a key (D8).  Empty set and no
 * mean slot -> o = 0, Z = 0 (D7).  Computes queries sel (or all) of every
 * (b,h); idx rows are indexed like the output rows.                          */
static void forward_query(const oref_problem* p, int64_t bh, int64_t i, const float* Q, const float* K,
                          const float* V, double eps, const int32_t* row, const double* Kb, const double* Vb,
                          double* o, double* Zout) {
    const int64_t N = p->N;
    const int dk = p->d_k, dv = p->d_v, k = p->k;
    const float* q = Q + (bh * N + i) * dk;
    double Zi = 0.0;
    for (int r = 0; r < k; ++r) {
        if (row[r] < 0) continue;
        Zi += 1.0 / (dist64(q, K + (bh * N + row[r]) * dk, dk) + eps);
    }
    double Smu = 0.0;
    if (p->mean_slot) { Smu = 1.0 / (dist64_mean(q, Kb + i * dk, dk) + eps); Zi += Smu; }
    for (int d = 0; d < dv; ++d) o[d] = 0.0;
    if (Zi > 0.0) {
        for (int r = 0; r < k; ++r) {
            if (row[r] < 0) continue;
            int64_t j = row[r];
            double A = (1.0 / (dist64(q, K + (bh * N + j) * dk, dk) + eps)) / Zi;
            for (int d = 0; d < dv; ++d) o[d] += A * (double)V[(bh * N + j) * dv + d];
        }
        if (p->mean_slot) {
            double A = Smu / Zi;
            for (int d = 0; d < dv; ++d) o[d] += A * Vb[i * dv + d];
        }
    }
    *Zout = Zi;
}

/* Step 8: forward with a given index set.  Eq. 5: S_ij =
 * 1/(||q_i-k_j||^2 + eps) (gamma/pi cancels, eps = gamma^2, D13-D14);
 * Eq. 6 + appendix: Z_i = sum S, A = S/Z,
 * o_i = sum A v, with the mean slot scored like a key (D8).  Empty set and no
 * mean slot -> o = 0, Z = 0 (D7).  Computes the queries sel[t] = bh*N + i
 * (or all when sel == NULL); idx/O/Z rows are indexed like the outputs.     */
int oref_forward(const oref_problem* p, const float* Q, const float* K, const float* V, double eps,
                 const int32_t* idx, double* O, double* Z, int64_t n_sel, const int64_t* sel) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k, dv = p->d_v, k = p->k;
    if (!(eps > 0.0) || !isfinite(eps)) return OREF_ERR_NONFINITE;
    if (!sel) {
        /* queries are independent given the prefix means: OpenMP over the
         * queries of each (b,h) (every output row is computed by the same
         * serial code whichever thread runs it) */
        double* Kb = NULL; double* Vb = NULL;
        if (p->mean_slot) {
            Kb = (double*)malloc(sizeof(double) * (size_t)(N * dk));
            Vb = (double*)malloc(sizeof(double) * (size_t)(N * dv));
        }
        for (int64_t bh = 0; bh < BH; ++bh) {
            if (p->mean_slot) {
                prefix_means(p, K, bh, dk, Kb);
                prefix_means(p, V, bh, dv, Vb);
            }
            #pragma omp parallel for schedule(dynamic, 64)
            for (int64_t i = 0; i < N; ++i)
                forward_query(p, bh, i, Q, K, V, eps, idx + (bh * N + i) * k, Kb, Vb,
                              O + (bh * N + i) * dv, Z + bh * N + i);
        }
        free(Kb); free(Vb);
        return OREF_OK;
    }
    double* Kb = NULL; double* Vb = NULL; int64_t cur_bh = -1;
    if (p->mean_slot) {
        Kb = (double*)malloc(sizeof(double) * (size_t)(N * dk));
        Vb = (double*)malloc(sizeof(double) * (size_t)(N * dv));
    }
    for (int64_t t = 0; t < n_sel; ++t) {
        int64_t bh = sel[t] / N, i = sel[t] % N;
        if (p->mean_slot && bh != cur_bh) {
            prefix_means(p, K, bh, dk, Kb);
            prefix_means(p, V, bh, dv, Vb);
            cur_bh = bh;
        }
        forward_query(p, bh, i, Q, K, V, eps, idx + t * k, Kb, Vb, O + t * dv, Z + t);
    }
    free(Kb); free(Vb);
    return OREF_OK;
}

/* Step 9: backward with I_i held fixed (D16), every query of every (b,h).
 * Appendix summary P:2006-2045 with "dL/do_i . (v_j - o_i)/Z_i" read as a
 * d_v-wide dot product (D15):
 *   g_ij  = dO_i.(v_j - o_i)/Z_i
 *   dv_j += A_ij dO_i
 *   dq_i  = -2 sum_j g_ij (q_i - k_j)/delta^2
 *   dk_j += 2 g_ij (q_i - k_j)/delta^2
 *   deps  = -sum_i sum_j g_ij/delta^2
 * plus the mean slot as one more slot whose key/value are prefix means, its
 * gradients chained back with weight 1/(i+1) (causal) or 1/N (D8, S:323(a)).
 * Accumulation order: queries ascending, slots ascending, mean slot last.
 * Per (b,h), in two loops so the host cores can share the work without
 * changing any sum's order:
 *   (1) per query (OpenMP over i; each query writes only its own rows):
 *       Z_i, o_i, g_ij and delta_ij of every slot, dq_i, the mean slot's
 *       dKbar_i/dVbar_i;
 *   (2) the key-side sums dv_j, dk_j (OpenMP over disjoint key ranges, each
 *       thread walking ALL (i, slot) pairs in ascending order and applying
 *       those of its own keys -- every key's sum runs in ascending i), and
 *       deps over (i, slot) in ascending order (serial).                   */
int oref_backward(const oref_problem* p, const float* Q, const float* K, const float* V, double eps,
                  const int32_t* idx, const float* dO, double* dQ, double* dK, double* dV, double* d_eps) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k, dv = p->d_v, k = p->k;
    if (!(eps > 0.0) || !isfinite(eps)) return OREF_ERR_NONFINITE;
    double* Kb = NULL; double* Vb = NULL; double* dKb = NULL; double* dVb = NULL;
    if (p->mean_slot) {
        Kb = (double*)malloc(sizeof(double) * (size_t)(N * dk));
        Vb = (double*)malloc(sizeof(double) * (size_t)(N * dv));
        dKb = (double*)malloc(sizeof(double) * (size_t)(N * dk));
        dVb = (double*)malloc(sizeof(double) * (size_t)(N * dv));
    }
    /* per (query, slot) g and delta (slot k = the mean slot), per query Z and "attended" */
    double* gs = (double*)malloc(sizeof(double) * (size_t)(N * (k + 1)));
    double* ds = (double*)malloc(sizeof(double) * (size_t)(N * (k + 1)));
    double* Zs = (double*)malloc(sizeof(double) * (size_t)N);
    double deps = 0.0;
    for (int64_t bh = 0; bh < BH; ++bh) {
        double deps_bh = 0.0;
        if (p->mean_slot) {
            prefix_means(p, K, bh, dk, Kb);
            prefix_means(p, V, bh, dv, Vb);
            for (int64_t x = 0; x < N * dk; ++x) dKb[x] = 0.0;
            for (int64_t x = 0; x < N * dv; ++x) dVb[x] = 0.0;
        }
        for (int64_t x = 0; x < N * dk; ++x) { dQ[bh * N * dk + x] = 0.0; dK[bh * N * dk + x] = 0.0; }
        for (int64_t x = 0; x < N * dv; ++x) dV[bh * N * dv + x] = 0.0;
        /* (1) per query */
        #pragma omp parallel
        {
            double* o = (double*)malloc(sizeof(double) * (size_t)dv);
            #pragma omp for schedule(dynamic, 64)
            for (int64_t i = 0; i < N; ++i) {
                const int64_t fi = bh * N + i;
                const float* q = Q + fi * dk;
                const float* g_o = dO + fi * dv;
                const int32_t* row = idx + fi * k;
                /* forward quantities for this query */
                double Zi = 0.0, Smu = 0.0;
                for (int r = 0; r < k; ++r)
                    if (row[r] >= 0) Zi += 1.0 / (dist64(q, K + (bh * N + row[r]) * dk, dk) + eps);
                if (p->mean_slot) { Smu = 1.0 / (dist64_mean(q, Kb + i * dk, dk) + eps); Zi += Smu; }
                Zs[i] = Zi;
                if (!(Zi > 0.0)) continue;                      /* D7: nothing attended */
                for (int d = 0; d < dv; ++d) o[d] = 0.0;
                for (int r = 0; r < k; ++r) {
                    if (row[r] < 0) continue;
                    int64_t j = row[r];
                    double A = (1.0 / (dist64(q, K + (bh * N + j) * dk, dk) + eps)) / Zi;
                    for (int d = 0; d < dv; ++d) o[d] += A * (double)V[(bh * N + j) * dv + d];
                }
                if (p->mean_slot)
                    for (int d = 0; d < dv; ++d) o[d] += (Smu / Zi) * Vb[i * dv + d];
                /* gradients of the query side */
                for (int r = 0; r < k; ++r) {
                    if (row[r] < 0) continue;
                    int64_t j = row[r];
                    const float* kj = K + (bh * N + j) * dk;
                    double delta = dist64(q, kj, dk) + eps;
                    double dot = 0.0;
                    for (int d = 0; d < dv; ++d) dot += (double)g_o[d] * ((double)V[(bh * N + j) * dv + d] - o[d]);
                    double g = dot / Zi;
                    gs[i * (k + 1) + r] = g;
                    ds[i * (k + 1) + r] = delta;
                    for (int d = 0; d < dk; ++d) {
                        double diff = (double)q[d] - (double)kj[d];
                        dQ[fi * dk + d] += -2.0 * g * diff / (delta * delta);
                    }
                }
                if (p->mean_slot) {
                    const double* kb = Kb + i * dk;
                    double delta = dist64_mean(q, kb, dk) + eps;
                    double A = Smu / Zi;
                    double dot = 0.0;
                    for (int d = 0; d < dv; ++d) dot += (double)g_o[d] * (Vb[i * dv + d] - o[d]);
                    double g = dot / Zi;
                    gs[i * (k + 1) + k] = g;
                    ds[i * (k + 1) + k] = delta;
                    for (int d = 0; d < dv; ++d) dVb[i * dv + d] += A * (double)g_o[d];
                    for (int d = 0; d < dk; ++d) {
                        double diff = (double)q[d] - kb[d];
                        dQ[fi * dk + d] += -2.0 * g * diff / (delta * delta);
                        dKb[i * dk + d] += 2.0 * g * diff / (delta * delta);
                    }
                }
            }
            free(o);
        }
        /* (2) key side: dv_j, dk_j over the selecting queries in ascending i */
        #pragma omp parallel
        {
            int64_t nt = 1, t = 0;
#ifdef _OPENMP
            nt = omp_get_num_threads();
            t = omp_get_thread_num();
#endif
            const int64_t j0 = N * t / nt, j1 = N * (t + 1) / nt;
            for (int64_t i = 0; i < N; ++i) {
                if (!(Zs[i] > 0.0)) continue;
                const int64_t fi = bh * N + i;
                const float* q = Q + fi * dk;
                const float* g_o = dO + fi * dv;
                const int32_t* row = idx + fi * k;
                for (int r = 0; r < k; ++r) {
                    const int64_t j = row[r];
                    if (j < j0 || j >= j1) continue;            /* also skips -1 */
                    const float* kj = K + (bh * N + j) * dk;
                    const double g = gs[i * (k + 1) + r], delta = ds[i * (k + 1) + r];
                    const double A = (1.0 / delta) / Zs[i];
                    for (int d = 0; d < dv; ++d) dV[(bh * N + j) * dv + d] += A * (double)g_o[d];
                    for (int d = 0; d < dk; ++d) {
                        double diff = (double)q[d] - (double)kj[d];
                        dK[(bh * N + j) * dk + d] += 2.0 * g * diff / (delta * delta);
                    }
                }
            }
        }
        /* deps over (i, slot) ascending, mean slot last within a query */
        for (int64_t i = 0; i < N; ++i) {
            if (!(Zs[i] > 0.0)) continue;
            const int32_t* row = idx + (bh * N + i) * k;
            for (int r = 0; r < k; ++r) {
                if (row[r] < 0) continue;
                const double g = gs[i * (k + 1) + r], delta = ds[i * (k + 1) + r];
                deps_bh += -g / (delta * delta);
            }
            if (p->mean_slot) {
                const double g = gs[i * (k + 1) + k], delta = ds[i * (k + 1) + k];
                deps_bh += -g / (delta * delta);
            }
        }
        deps += deps_bh;
        if (p->mean_slot) {
            /* chain rule through the prefix means (S:323(a)):
             *   causal:     dK_t += sum_{i>=t} dKbar_i/(i+1)   (suffix sum, i descending)
             *   non-causal: dK_t += (1/N) sum_i dKbar_i                                   */
            double* acc = (double*)calloc((size_t)(dk + dv), sizeof(double));
            if (p->causal) {
                for (int64_t t = N - 1; t >= 0; --t) {
                    for (int d = 0; d < dk; ++d) acc[d] += dKb[t * dk + d] / (double)(t + 1);
                    for (int d = 0; d < dv; ++d) acc[dk + d] += dVb[t * dv + d] / (double)(t + 1);
                    for (int d = 0; d < dk; ++d) dK[(bh * N + t) * dk + d] += acc[d];
                    for (int d = 0; d < dv; ++d) dV[(bh * N + t) * dv + d] += acc[dk + d];
                }
            } else {
                for (int64_t i = 0; i < N; ++i) {
                    for (int d = 0; d < dk; ++d) acc[d] += dKb[i * dk + d];
                    for (int d = 0; d < dv; ++d) acc[dk + d] += dVb[i * dv + d];
                }
                for (int64_t t = 0; t < N; ++t) {
                    for (int d = 0; d < dk; ++d) dK[(bh * N + t) * dk + d] += acc[d] / (double)N;
                    for (int d = 0; d < dv; ++d) dV[(bh * N + t) * dv + d] += acc[dk + d] / (double)N;
                }
            }
            free(acc);
        }
    }
    /* D20: one scalar eps per call, gradient summed over all (b,h) in order */
    *d_eps = deps;
    free(gs); free(ds); free(Zs); free(Kb); free(Vb); free(dKb); free(dVb);
    return OREF_OK;
}

/* ------------------------------------------------------------------------ */
/* Score variants (reading D24).  The paper compares its
 * Cauchy Softmax with "Negative Euclidean, ... and Inverse Euclidean
 * operators" and with "Normalized Dot Prod" (Table
 * "similarity metrics"); SPEC fixes their formulas:
 *   1 NEG_EUCLID  S = exp(-D)                       ("Negative Euclidean with
 *                                                    traditional softmax")
 *   2 INV_EUCLID  S = 1/(sqrt(D) + 1e-6)            (stabiliser S:401)
 *   3 DOT         S = exp(q.k / sqrt(d_k))          ("dot_product")
 * with D = ||q - k||^2.  The top-k set is the same Euclidean selection for
 * every score ("We utilize Euclidean distance for k-NN searches"); only
 * the weights change: A = S/Z, Z = sum S, o = sum A v, the mean slot scored
 * like a key.  Z output: sum S for INV_EUCLID, log(sum S) for the two
 * exponential scores (the softmax normaliser in log form; the CUDA path keeps
 * it in log form to stay finite).  Backward, by the chain rule with
 * g_j = dL/dS_j = dO.(v_j - o)/Z (D15's dot product):
 *   dq  += g_j dS_j/dq,  dk_j += g_j dS_j/dk_j,  dv_j += A_j dO
 * where for the distance scores dS/dq = -dS/dk = S'(D) 2 (q - k) and for DOT
 * dS/dq = S k/sqrt(d_k), dS/dk = S q/sqrt(d_k).  INV_EUCLID at D = 0 (q == k)
 * is not differentiable; its (q - k) factor is 0 there and the gradient term is
 * taken as 0.  No eps: d_eps = 0.                                            */
enum { OREF_CAUCHY = 0, OREF_NEG_EUCLID = 1, OREF_INV_EUCLID = 2, OREF_DOT = 3 };

/* S of one slot and its partial derivatives: gq = dS/dq, gk = dS/dk (d_k each) */
static double score_slot(int score, const float* q, const double* kk, int dk, double* gq, double* gk) {
    double D = 0.0, dot = 0.0;
    for (int d = 0; d < dk; ++d) {
        double t = (double)q[d] - kk[d];
        D += t * t;
        dot += (double)q[d] * kk[d];
    }
    double S = 0.0, dSdD = 0.0;
    if (score == OREF_NEG_EUCLID) {
        S = exp(-D);
        dSdD = -S;
    } else if (score == OREF_INV_EUCLID) {
        double r = sqrt(D);
        S = 1.0 / (r + 1e-6);
        dSdD = r > 0.0 ? -S * S / (2.0 * r) : 0.0;
    } else {  /* OREF_DOT */
        double sc = 1.0 / sqrt((double)dk);
        S = exp(dot * sc);
        for (int d = 0; d < dk; ++d) { gq[d] = S * kk[d] * sc; gk[d] = S * (double)q[d] * sc; }
        return S;
    }
    for (int d = 0; d < dk; ++d) {
        double t = (double)q[d] - kk[d];
        gq[d] = dSdD * 2.0 * t;
        gk[d] = -dSdD * 2.0 * t;
    }
    return S;
}

static void key_row(const float* K, int64_t row, int dk, double* kk) {
    for (int d = 0; d < dk; ++d) kk[d] = (double)K[row * dk + d];
}

/* forward of every query with a given index set, score variant p->score != 0 */
int oref_forward_score(const oref_problem* p, const float* Q, const float* K, const float* V, const int32_t* idx,
                       double* O, double* Z) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k, dv = p->d_v, k = p->k;
    if (p->score < 1 || p->score > 3) return OREF_ERR_INVALID_ARG;
    #pragma omp parallel for schedule(dynamic)
    for (int64_t bh = 0; bh < BH; ++bh) {
        double* Kb = NULL; double* Vb = NULL;
        double kk[8], gq[8], gk[8];
        double* S = (double*)malloc(sizeof(double) * (size_t)(k + 1));
        if (p->mean_slot) {
            Kb = (double*)malloc(sizeof(double) * (size_t)(N * dk));
            Vb = (double*)malloc(sizeof(double) * (size_t)(N * dv));
            prefix_means(p, K, bh, dk, Kb);
            prefix_means(p, V, bh, dv, Vb);
        }
        for (int64_t i = 0; i < N; ++i) {
            const int64_t fi = bh * N + i;
            const float* q = Q + fi * dk;
            const int32_t* row = idx + fi * k;
            double Zi = 0.0;
            int any = 0;
            for (int r = 0; r < k; ++r) {
                if (row[r] < 0) continue;
                key_row(K, bh * N + row[r], dk, kk);
                S[r] = score_slot(p->score, q, kk, dk, gq, gk);
                Zi += S[r];
                any = 1;
            }
            if (p->mean_slot) {
                S[k] = score_slot(p->score, q, Kb + (p->causal ? i : 0) * dk, dk, gq, gk);
                Zi += S[k];
                any = 1;
            }
            for (int d = 0; d < dv; ++d) O[fi * dv + d] = 0.0;
            if (any) {
                for (int r = 0; r < k; ++r) {
                    if (row[r] < 0) continue;
                    for (int d = 0; d < dv; ++d) O[fi * dv + d] += (S[r] / Zi) * (double)V[(bh * N + row[r]) * dv + d];
                }
                if (p->mean_slot)
                    for (int d = 0; d < dv; ++d) O[fi * dv + d] += (S[k] / Zi) * Vb[(p->causal ? i : 0) * dv + d];
            }
            Z[fi] = !any ? 0.0 : (p->score == OREF_INV_EUCLID ? Zi : log(Zi));
        }
        free(S); free(Kb); free(Vb);
    }
    return OREF_OK;
}

/* backward of every query with a given index set, score variant p->score != 0 */
int oref_backward_score(const oref_problem* p, const float* Q, const float* K, const float* V, const int32_t* idx,
                        const float* dO, double* dQ, double* dK, double* dV, double* d_eps) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k, dv = p->d_v, k = p->k;
    if (p->score < 1 || p->score > 3) return OREF_ERR_INVALID_ARG;
    #pragma omp parallel for schedule(dynamic)
    for (int64_t bh = 0; bh < BH; ++bh) {
        double* Kb = NULL; double* Vb = NULL; double* dKb = NULL; double* dVb = NULL;
        double kk[8], gq[8], gk[8];
        double* S = (double*)malloc(sizeof(double) * (size_t)(k + 1));
        double* o = (double*)malloc(sizeof(double) * (size_t)dv);
        if (p->mean_slot) {
            Kb = (double*)malloc(sizeof(double) * (size_t)(N * dk));
            Vb = (double*)malloc(sizeof(double) * (size_t)(N * dv));
            dKb = (double*)calloc((size_t)(N * dk), sizeof(double));
            dVb = (double*)calloc((size_t)(N * dv), sizeof(double));
            prefix_means(p, K, bh, dk, Kb);
            prefix_means(p, V, bh, dv, Vb);
        }
        for (int64_t x = 0; x < N * dk; ++x) { dQ[bh * N * dk + x] = 0.0; dK[bh * N * dk + x] = 0.0; }
        for (int64_t x = 0; x < N * dv; ++x) dV[bh * N * dv + x] = 0.0;
        for (int64_t i = 0; i < N; ++i) {
            const int64_t fi = bh * N + i;
            const float* q = Q + fi * dk;
            const float* g_o = dO + fi * dv;
            const int32_t* row = idx + fi * k;
            const int64_t mi = p->causal ? i : 0;
            double Zi = 0.0;
            int any = 0;
            for (int r = 0; r < k; ++r) {
                if (row[r] < 0) continue;
                key_row(K, bh * N + row[r], dk, kk);
                S[r] = score_slot(p->score, q, kk, dk, gq, gk);
                Zi += S[r];
                any = 1;
            }
            if (p->mean_slot) { S[k] = score_slot(p->score, q, Kb + mi * dk, dk, gq, gk); Zi += S[k]; any = 1; }
            if (!any) continue;                               /* D7: nothing attended */
            for (int d = 0; d < dv; ++d) o[d] = 0.0;
            for (int r = 0; r < k; ++r) {
                if (row[r] < 0) continue;
                for (int d = 0; d < dv; ++d) o[d] += (S[r] / Zi) * (double)V[(bh * N + row[r]) * dv + d];
            }
            if (p->mean_slot)
                for (int d = 0; d < dv; ++d) o[d] += (S[k] / Zi) * Vb[mi * dv + d];
            for (int r = 0; r < k; ++r) {
                if (row[r] < 0) continue;
                const int64_t j = bh * N + row[r];
                key_row(K, j, dk, kk);
                score_slot(p->score, q, kk, dk, gq, gk);
                double dot = 0.0;
                for (int d = 0; d < dv; ++d) dot += (double)g_o[d] * ((double)V[j * dv + d] - o[d]);
                const double g = dot / Zi;
                for (int d = 0; d < dv; ++d) dV[j * dv + d] += (S[r] / Zi) * (double)g_o[d];
                for (int d = 0; d < dk; ++d) { dQ[fi * dk + d] += g * gq[d]; dK[j * dk + d] += g * gk[d]; }
            }
            if (p->mean_slot) {
                score_slot(p->score, q, Kb + mi * dk, dk, gq, gk);
                double dot = 0.0;
                for (int d = 0; d < dv; ++d) dot += (double)g_o[d] * (Vb[mi * dv + d] - o[d]);
                const double g = dot / Zi;
                for (int d = 0; d < dv; ++d) dVb[mi * dv + d] += (S[k] / Zi) * (double)g_o[d];
                for (int d = 0; d < dk; ++d) { dQ[fi * dk + d] += g * gq[d]; dKb[mi * dk + d] += g * gk[d]; }
            }
        }
        if (p->mean_slot) {
            /* the same chain rule through the prefix means as oref_backward (S:323(a)) */
            double* acc = (double*)calloc((size_t)(dk + dv), sizeof(double));
            if (p->causal) {
                for (int64_t t = N - 1; t >= 0; --t) {
                    for (int d = 0; d < dk; ++d) acc[d] += dKb[t * dk + d] / (double)(t + 1);
                    for (int d = 0; d < dv; ++d) acc[dk + d] += dVb[t * dv + d] / (double)(t + 1);
                    for (int d = 0; d < dk; ++d) dK[(bh * N + t) * dk + d] += acc[d];
                    for (int d = 0; d < dv; ++d) dV[(bh * N + t) * dv + d] += acc[dk + d];
                }
            } else {
                for (int d = 0; d < dk; ++d) acc[d] = dKb[d];
                for (int d = 0; d < dv; ++d) acc[dk + d] = dVb[d];
                for (int64_t t = 0; t < N; ++t) {
                    for (int d = 0; d < dk; ++d) dK[(bh * N + t) * dk + d] += acc[d] / (double)N;
                    for (int d = 0; d < dv; ++d) dV[(bh * N + t) * dv + d] += acc[dk + d] / (double)N;
                }
            }
            free(acc);
        }
        free(S); free(o); free(Kb); free(Vb); free(dKb); free(dVb);
    }
    *d_eps = 0.0;
    return OREF_OK;
}

/* Brute-force chunk-causal exact Euclidean kNN (no Morton code at all), same
 * ranking precision and tie rule as select_one.  Used by the recall workload
 * and by the "W >= M" special case.                                          */
int oref_bruteforce_knn(const oref_problem* p, const float* Q, const float* K, int32_t* idx) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int dk = p->d_k, k = p->k;
    #pragma omp parallel
    {
        cand* buf = (cand*)malloc(sizeof(cand) * (size_t)N);
        #pragma omp for schedule(dynamic, 64)
        for (int64_t flat = 0; flat < BH * N; ++flat) {
            int64_t bh = flat / N, i = flat % N;
            int64_t lim = p->causal ? (i / p->chunk) * p->chunk : N;
            for (int64_t j = 0; j < lim; ++j) {
                buf[j].j = (int32_t)j;
                buf[j].D = rank_dist32(Q + flat * dk, K + (bh * N + j) * dk, dk);
            }
            qsort(buf, (size_t)lim, sizeof(cand), cmp_cand);
            for (int r = 0; r < k; ++r) idx[flat * k + r] = r < lim ? buf[r].j : -1;
        }
        free(buf);
    }
    return OREF_OK;
}

/* Locality workload (Fig. 4 "overlap between the top-64
 * nearest neighbors before and after projection"
 * "top-64 nearest-by-|code difference| after Morton encoding").  For every
 * query i: the admissible keys (chunk-causal as in step 5, or all N),
 * optionally without j == i, ordered by (|kcode_j - qcode_i|, j) -- u64
 * absolute difference, ties by position (D19) -- first k, -1 padded.  Brute
 * force: every admissible key is scored and the list is sorted.            */
typedef struct { uint64_t d; int32_t j; } code_cand;
static int cmp_code_cand(const void* a, const void* b) {
    const code_cand* x = (const code_cand*)a; const code_cand* y = (const code_cand*)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

int oref_code_knn(const oref_problem* p, const uint64_t* qcode, const uint64_t* kcode, int exclude_self,
                  int32_t* idx) {
    const int64_t BH = p->B * p->H, N = p->N;
    const int k = p->k;
    #pragma omp parallel
    {
        code_cand* buf = (code_cand*)malloc(sizeof(code_cand) * (size_t)N);
        #pragma omp for schedule(dynamic, 64)
        for (int64_t flat = 0; flat < BH * N; ++flat) {
            const int64_t bh = flat / N, i = flat % N;
            const int64_t lim = p->causal ? (i / p->chunk) * p->chunk : N;
            const uint64_t qc = qcode[flat];
            int64_t n = 0;
            for (int64_t j = 0; j < lim; ++j) {
                if (exclude_self && j == i) continue;
                const uint64_t kc = kcode[bh * N + j];
                buf[n].d = kc > qc ? kc - qc : qc - kc;
                buf[n].j = (int32_t)j;
                ++n;
            }
            qsort(buf, (size_t)n, sizeof(code_cand), cmp_code_cand);
            for (int r = 0; r < k; ++r) idx[flat * k + r] = r < n ? buf[r].j : -1;
        }
        free(buf);
    }
    return OREF_OK;
}

int oref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
