// bwd_kernels.cuh -- the A8 query-side (K7) and A10 key-side (K9) kernel
// templates, shared by the per-(d_k, storage type) instantiation units of bwd_inst.cu
// (the many (d_k, lanes-per-row, registers) instantiations compile in
// parallel) and by bwd.cu, which holds the launch sequence.  See bwd.cu for
// the method and citations.
#pragma once

#include "common.cuh"
#include "internal.h"

namespace onedf {

constexpr int BWD_WARPS = 8;
constexpr int BWD_THREADS = BWD_WARPS * 32;
#ifndef ONEDF_KEY_U
#define ONEDF_KEY_U 4
#endif
#ifndef ONEDF_BWD_MINB
#define ONEDF_BWD_MINB 4
#endif

struct BwdArgs {
    const float* Q; const float* K; const void* V; const float* eps;     // V, dO: storage type TV (vdtype)
    const void* dO; const int32_t* idx;
    const float* Kbar; const float* Vbar; const int32_t* qorder;
    float* dQ; float2* muco; double* eps_q;
    int32_t* cursor; int32_t* rec_i; float2* rec_aw;      // key-major CSR records (csr.cu, SoA)
    int64_t N, total, nq, L;        // nq: schedule slots per (b,h) (N, or the owned chunks when sharded)
    int k, dv, causal, mean_slot, score;
    Shard sh;
    void* ws;
};

// Butterfly reduce-scatter of T partials over the P lanes of a lane group:
// afterwards the lane with in-group index l holds the full sum of partial
// t = l >> (log2 P - log2 T) in v[0].
template <int P, int T>
__device__ __forceinline__ void reduce_scatter(double (&v)[T]) {
    int live = T;
#pragma unroll
    for (int s = P / 2; s >= 1; s >>= 1) {
        if (live > 1) {
            const int half = live / 2;
            const bool upper = (lane_id() & s) != 0;
#pragma unroll
            for (int m = 0; m < T / 2; ++m) {
                if (m < half) {
                    const double send = upper ? v[m] : v[m + half];
                    const double keep = upper ? v[m + half] : v[m];
                    v[m] = keep + __shfl_xor_sync(FULL, send, s);
                }
            }
            live = half;
        } else {
            v[0] += __shfl_xor_sync(FULL, v[0], s);
        }
    }
}

// w of one slot (dq -= w (qt q - k), dk += w (q - kt k)) and its d_eps term,
// from the f64 weight S (exp-shifted for the softmax scores), A = S/Z and
// diff = dO.v - c (reading D24 for the variants).
template <int DK>
__device__ __forceinline__ void slot_w(int sc, const float* q, const float* kj, double ed, double S, double A,
                                       double invZ, double diff, double& w, double& de) {
    de = 0.0;
    if (sc == SC_CAUCHY) {
        const double delta = dist64<DK>(q, kj) + ed;
        const double g = diff * invZ;
        const double inv_d2 = 1.0 / (delta * delta);
        w = 2.0 * g * inv_d2;
        de = -(g * inv_d2);
    } else if (sc == SC_INV) {
        const double r = sqrt(dist64<DK>(q, kj));
        w = r > 0.0 ? diff * invZ * S * S / r : 0.0;   // not differentiable at q == k, where (q - k) = 0
    } else if (sc == SC_NEG) {
        w = 2.0 * A * diff;
    } else {
        w = A * diff * (1.0 / sqrt((double)DK));
    }
}

template <int DK, int P, int CH, int R, bool WHOLE, typename TV>
__global__ void __launch_bounds__(BWD_THREADS, ONEDF_BWD_MINB) bwd_query_kernel(const BwdArgs a) {
    constexpr int G = 32 / P;                    // rows per step
    constexpr int T = P < 8 ? P : 8;             // steps per block (live partials / loads in flight per lane)
    constexpr int RB = T * G;                    // rows per block
    constexpr int LOGP = P == 32 ? 5 : P == 16 ? 4 : P == 8 ? 3 : P == 4 ? 2 : P == 2 ? 1 : 0;
    constexpr int LOGT = T == 16 ? 4 : T == 8 ? 3 : T == 4 ? 2 : T == 2 ? 1 : 0;
    __shared__ double s_part[BWD_WARPS][32 * R];  // dO_i . v_j per slot (phase 1 -> phase 2)
    const int warp = threadIdx.x / 32, lane = lane_id();
    const int64_t slot = (int64_t)blockIdx.x * BWD_WARPS + warp;
    if (slot >= a.total) return;
    const int64_t N = a.N;
    const int64_t bh = slot / a.nq;
    int64_t pos;
    if (!a.sh.slot_pos(slot - bh * a.nq, N, pos)) return;      // sharded: padding of a short last chunk
    const int64_t i = a.qorder ? (int64_t)__ldg(a.qorder + bh * N + pos) : pos;
    const int64_t gq = bh * N + i;
    const int sc = a.score;
    const float e = __ldg(a.eps);
    if (sc == SC_CAUCHY && slot == 0 && lane == 0 && !(e > 0.f && isfinite(e))) set_flag(a.ws, ONEDF_OP_BWD, FLAG_BAD_EPS);
    const double ed = (double)e;
    const int dv = a.dv, k = a.k, nch = dv / 4;
    const int grp = lane / P, l = lane % P;
    // something attended (D7): the mean slot or a first selected key (idx ascending, -1 padded)
    const bool live = a.mean_slot || __ldg(a.idx + gq * k) >= 0;
    // the idx row, lane-parallel (slot e lives on lane e % 32, register e / 32)
    int jr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e2 = r * 32 + lane;
        jr[r] = (live && e2 < k) ? __ldg(a.idx + gq * k + e2) : -1;
    }
    float q[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) q[d] = __ldg(a.Q + gq * DK + d);

    // this lane's dO chunks (ch = l + h*P, h < CH)
    float4 g4[CH];
#pragma unroll
    for (int h = 0; h < CH; ++h) {
        const int ch = l + h * P;
        g4[h] = ch < nch ? ld4(static_cast<const TV*>(a.dO) + gq * dv, ch) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int64_t mrow = a.causal ? i : 0;
    const TV* Vb = static_cast<const TV*>(a.V) + bh * N * (int64_t)dv;
    const TV* Vl = Vb + 4 * l;                    // this lane's first chunk of row 0
    const int owner_t = l >> (LOGP - LOGT);
    const bool owner = (l & ((1 << (LOGP - LOGT)) - 1)) == 0;
    double* sp = s_part[warp];

    // ---------------- phase 1: dO_i . v_j for every slot (f64, exact f32 products)
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int h0 = 0; h0 < 32; h0 += RB) {
            const int e0 = r * 32 + h0;
            if (e0 >= k) break;                                  // warp-uniform
            double part[T];
            float4 x[T][CH];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int j = __shfl_sync(FULL, jr[r], (h0 + t * G + grp) & 31);
                // an unselected slot (j < 0) reads row 0; its dot is never used (phase 2 skips it)
                const int jj = j < 0 ? 0 : j;
                if (WHOLE) {
                    // P*CH == d_v/4: d_v is a constant and every chunk exists; lane base + row offset
                    const TV* vr = Vl + (int64_t)jj * (4 * P * CH);
#pragma unroll
                    for (int h = 0; h < CH; ++h) x[t][h] = ld4(vr, h * P);
                } else {
                    const TV* vr = Vb + (int64_t)jj * dv;
#pragma unroll
                    for (int h = 0; h < CH; ++h)
                        x[t][h] = l + h * P < nch ? ld4(vr, l + h * P) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int t = 0; t < T; ++t) {
                // exact f32 products summed in f64: these dots enter g = (dO.v_j - c)/Z, whose
                // cancellation when one weight dominates would amplify any rounding here (R3, R5)
                part[t] = 0.0;
#pragma unroll
                for (int h = 0; h < CH; ++h) {
                    part[t] = fma((double)x[t][h].x, (double)g4[h].x, part[t]);
                    part[t] = fma((double)x[t][h].y, (double)g4[h].y, part[t]);
                    part[t] = fma((double)x[t][h].z, (double)g4[h].z, part[t]);
                    part[t] = fma((double)x[t][h].w, (double)g4[h].w, part[t]);
                }
            }
            reduce_scatter<P, T>(part);
            const int row = e0 + owner_t * G + grp;
            if (owner && row < k) sp[row] = part[0];
        }
    }
    double dot_mu = 0.0;
    if (a.mean_slot) {
        double dpart = 0.0;
        const float* vbar = a.Vbar + (bh * (a.causal ? N : 1) + mrow) * (int64_t)dv;
#pragma unroll
        for (int h = 0; h < CH; ++h) {
            const int ch = l + h * P;
            if (grp == 0 && ch < nch) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(vbar) + ch);
                dpart = fma((double)g4[h].x, (double)x.x, dpart);
                dpart = fma((double)g4[h].y, (double)x.y, dpart);
                dpart = fma((double)g4[h].z, (double)x.z, dpart);
                dpart = fma((double)g4[h].w, (double)x.w, dpart);
            }
        }
        dot_mu = warp_sum(dpart);
    }
    __syncwarp();

    // ---------------- phase 2: weights, normaliser and c_i = dO_i . o_i recomputed in f64
    // from the slot dots (c = sum A_j (dO.v_j) + A_mu dO.Vbar): no f32-rounded O or Z
    // enters g_ij = (dO.v_j - c)/Z, which matters when one weight approaches 1.
    float kb[DK];
    double Smu = 0.0;
    if (a.mean_slot) {
#pragma unroll
        for (int d = 0; d < DK; ++d) kb[d] = __ldg(a.Kbar + (bh * (a.causal ? N : 1) + mrow) * DK + d);
        Smu = score_raw<DK>(sc, q, kb, ed);
    }
    double Sr[R], pr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        Sr[r] = 0.0;
        pr[r] = 0.0;
        if (jr[r] >= 0) {
            float kj[DK];
#pragma unroll
            for (int d = 0; d < DK; ++d) kj[d] = __ldg(a.K + (bh * N + jr[r]) * DK + d);
            Sr[r] = score_raw<DK>(sc, q, kj, ed);
            pr[r] = sp[r * 32 + lane];
        }
    }
    if (score_is_exp(sc)) {
        double m = -INFINITY;
#pragma unroll
        for (int r = 0; r < R; ++r) m = jr[r] >= 0 ? fmax(m, Sr[r]) : m;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
        if (a.mean_slot) m = fmax(m, Smu);
#pragma unroll
        for (int r = 0; r < R; ++r) Sr[r] = jr[r] >= 0 ? exp(Sr[r] - m) : 0.0;
        if (a.mean_slot) Smu = exp(Smu - m);
    }
    double zpart = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) zpart += Sr[r];
    const double Zi = warp_sum(zpart) + Smu;
    const double invZ = live && Zi > 0.0 ? 1.0 / Zi : 0.0;
    double cpart = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) cpart = fma(Sr[r] * invZ, pr[r], cpart);
    const double c = warp_sum(cpart) + (Smu * invZ) * dot_mu;
    const double qt = sc == SC_DOT ? 0.0 : 1.0;     // dq -= w (qt q - k): distance scores vs q.k
    double dq[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) dq[d] = 0.0;
    double deps = 0.0;
    int32_t* cur = a.cursor + bh * N;
    int32_t* rec_i = a.rec_i + bh * a.L;
    float2* rec_aw = a.rec_aw + bh * a.L;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int e2 = r * 32 + lane;
        if (e2 >= k) break;
        if (jr[r] >= 0) {
            float kj[DK];
#pragma unroll
            for (int d = 0; d < DK; ++d) kj[d] = __ldg(a.K + (bh * N + jr[r]) * DK + d);
            const double A = Sr[r] * invZ;
            double w, de;
            slot_w<DK>(sc, q, kj, ed, Sr[r], A, invZ, pr[r] - c, w, de);
#pragma unroll
            for (int d = 0; d < DK; ++d) dq[d] -= w * ((double)q[d] * qt - (double)kj[d]);
            deps += de;
            // append the record to key j's CSR segment (integer slot; the key side orders by i)
            const int32_t pos = atomicAdd(cur + jr[r], 1);
            rec_i[pos] = (int32_t)i;
            rec_aw[pos] = make_float2((float)A, (float)w);
        }
    }
    if (a.mean_slot) {
        const double A = Smu * invZ;
        double w, de;
        slot_w<DK>(sc, q, kb, ed, Smu, A, invZ, dot_mu - c, w, de);
        if (lane == 0) {
#pragma unroll
            for (int d = 0; d < DK; ++d) dq[d] -= w * ((double)q[d] * qt - (double)kb[d]);
            deps += de;
            a.muco[gq] = make_float2((float)A, (float)w);
        }
    } else if (lane == 0) {
        a.muco[gq] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int d = 0; d < DK; ++d) dq[d] = warp_sum(dq[d]);
    deps = warp_sum(deps);
    if (lane < DK) {
        double v = 0.0;
#pragma unroll
        for (int d = 0; d < DK; ++d) v = (lane == d) ? dq[d] : v;
        a.dQ[gq * DK + lane] = (float)v;
    }
    if (lane == 0) a.eps_q[gq] = deps;
}

struct KeyArgs {
    const float* Q; const float* K; const void* dO;        // dO: storage type TV; dK, dV written as f32
    const int32_t* offsets; const int32_t* rec_i; const float2* rec_aw; const int32_t* order;
    const int32_t* korder;
    float* dK; float* dV;
    int64_t N, L, total;
    int k, dv;
    double kt;           // dk += w (q - kt k): 1 for the distance scores, 0 for DOT
};


template <int R>
__device__ __forceinline__ void sort_prefix(uint32_t (&x)[KEY_REG_SEG / 32]) {
    uint32_t y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] = x[r];
    warp_sort_u32<R>(y);
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = y[r];
}

template <int DK, int P, int CH, bool WHOLE, typename TV>
__global__ void __launch_bounds__(BWD_THREADS, ONEDF_BWD_MINB) bwd_key_kernel(const KeyArgs a) {
    constexpr int G = 32 / P;
    constexpr int U = ONEDF_KEY_U;                // entries per lane group in flight
    __shared__ uint32_t s_key[BWD_WARPS][KEY_REG_SEG];
    const int warp = threadIdx.x / 32, lane = lane_id();
    const int64_t slot = (int64_t)blockIdx.x * BWD_WARPS + warp;
    if (slot >= a.total) return;
    const int64_t N = a.N, bh = slot / N;
    const int64_t j = a.korder ? (int64_t)__ldg(a.korder + slot) : slot % N;
    const int64_t gk = bh * N + j;
    const int32_t* off = a.offsets + bh * (N + 1);
    const int32_t s0 = __ldg(off + j), s1 = __ldg(off + j + 1);
    const int32_t len = s1 - s0;
    const int32_t* ri = a.rec_i + bh * a.L + s0;
    const float2* raw = a.rec_aw + bh * a.L + s0;
    const int dv = a.dv, nch = dv / 4;
    const int grp = lane / P, l = lane % P;
    if (len == 0) {
        // no query selected this key (e.g. the last chunk's keys, or another rank's queries):
        // its direct gradient is zero (the mean-slot scan adds its share afterwards)
        float4* dvrow = reinterpret_cast<float4*>(a.dV + gk * (int64_t)dv);
        for (int ch = lane; ch < nch; ch += 32) dvrow[ch] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (lane < DK) a.dK[gk * DK + lane] = 0.f;
        return;
    }

    // ---- fixed visiting order: ascending query position i (distinct within a segment)
    const bool small = !csr_long_segment(len, N);
    uint32_t* sk = s_key[warp];                   // sorted (i << KEY_POS_BITS | position) keys
    const int32_t* go = a.order + bh * a.L + s0;
    if (small) {
        uint32_t xs[KEY_REG_SEG / 32];
#pragma unroll
        for (int r = 0; r < KEY_REG_SEG / 32; ++r) {
            const int e = r * 32 + lane;
            xs[r] = e < len ? ((uint32_t)__ldg(ri + e) << KEY_POS_BITS) | (uint32_t)e : ~0u;
        }
        if (len <= 32) sort_prefix<1>(xs);
        else if (len <= 64) sort_prefix<2>(xs);
        else if (len <= 128) sort_prefix<4>(xs);
        else if (KEY_REG_SEG <= 256 || len <= 256) sort_prefix<8>(xs);
        else sort_prefix<(KEY_REG_SEG > 256 ? 16 : 8)>(xs);
#pragma unroll
        for (int r = 0; r < KEY_REG_SEG / 32; ++r)
            if (r * 32 < len) sk[r * 32 + lane] = xs[r];
        __syncwarp();
    }
    // long segments were ordered beforehand by csr_long_order_kernel into `order` (go)

    float kj[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) kj[d] = __ldg(a.K + gk * DK + d);
    double dk[DK];
#pragma unroll
    for (int d = 0; d < DK; ++d) dk[d] = 0.0;
    double acc[CH][4];
#pragma unroll
    for (int h = 0; h < CH; ++h)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[h][c] = 0.0;
    const TV* dOb = static_cast<const TV*>(a.dO) + bh * N * (int64_t)dv;
    const TV* dOl = dOb + 4 * l;                  // this lane's first chunk of row 0
    const float* Qb = a.Q + bh * N * DK;

    for (int32_t b0 = 0; b0 < len; b0 += 32) {
        const int32_t t = b0 + lane;
        const bool has = t < len;
        int iq = 0;
        float2 aw = make_float2(0.f, 0.f);
        float qi[DK];
        if (has) {
            int e;
            if (small) {
                const uint32_t v = sk[t];
                e = (int)(v & ((1u << KEY_POS_BITS) - 1));
                iq = (int)(v >> KEY_POS_BITS);
            } else {
                e = __ldg(go + t);
                iq = __ldg(ri + e);
            }
            aw = __ldg(raw + e);
#pragma unroll
            for (int d = 0; d < DK; ++d) qi[d] = __ldg(Qb + (int64_t)iq * DK + d);
        }
        const int n = min(32, len - b0);
        // dV: group g takes entries g, g+G, ... of this chunk, U at a time
        for (int t0 = 0; t0 < n; t0 += G * U) {
            float4 x[U][CH];
            float Au[U];
            if (WHOLE && t0 + G * U <= n) {
                // d_v = 4*P*CH and all U entries of every group present: lane base + row offset, no masks
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int src = t0 + u * G + grp;
                    const int iu = __shfl_sync(FULL, iq, src);
                    Au[u] = __shfl_sync(FULL, aw.x, src);
                    const TV* rp = dOl + (int64_t)iu * (4 * P * CH);
#pragma unroll
                    for (int h = 0; h < CH; ++h) x[u][h] = ld4(rp, h * P);
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int src = t0 + u * G + grp;
                    const int iu = __shfl_sync(FULL, iq, src & 31);
                    Au[u] = __shfl_sync(FULL, aw.x, src & 31);
                    const bool ok = src < n;
                    if (!ok) Au[u] = 0.f;
#pragma unroll
                    for (int h = 0; h < CH; ++h) {
                        const int ch = l + h * P;
                        x[u][h] = (ok && ch < nch) ? ld4(dOb + (int64_t)iu * dv, ch) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            }
            // the U = 4 entries summed in f32 (sum4, fixed order), promoted once per value (reading R5)
            // each group of 4 entries (u = 4m .. 4m+3: entries t0 + 8m .. t0 + 8m + 7 of the chunk) is
            // summed in f32 (sum4, fixed order) and promoted once per value (reading R5); groups in
            // ascending entry order, a group past the chunk's last entry skipped -- the same sums
            // in the same order for any U
            static_assert(U % 4 == 0, "the f32 group of the dV gather is 4 entries");
#pragma unroll
            for (int m = 0; m < U; m += 4) {
                if (m > 0 && t0 + m * G >= n) break;
#pragma unroll
                for (int h = 0; h < CH; ++h) {
                    acc[h][0] += (double)sum4(Au[m], x[m][h].x, Au[m + 1], x[m + 1][h].x, Au[m + 2], x[m + 2][h].x,
                                              Au[m + 3], x[m + 3][h].x);
                    acc[h][1] += (double)sum4(Au[m], x[m][h].y, Au[m + 1], x[m + 1][h].y, Au[m + 2], x[m + 2][h].y,
                                              Au[m + 3], x[m + 3][h].y);
                    acc[h][2] += (double)sum4(Au[m], x[m][h].z, Au[m + 1], x[m + 1][h].z, Au[m + 2], x[m + 2][h].z,
                                              Au[m + 3], x[m + 3][h].z);
                    acc[h][3] += (double)sum4(Au[m], x[m][h].w, Au[m + 1], x[m + 1][h].w, Au[m + 2], x[m + 2][h].w,
                                              Au[m + 3], x[m + 3][h].w);
                }
            }
        }
        // dK: the lane owning the entry, f64, fixed entry -> lane map
        if (has) {
#pragma unroll
            for (int d = 0; d < DK; ++d) dk[d] += (double)aw.y * ((double)qi[d] - a.kt * (double)kj[d]);
        }
    }
#pragma unroll
    for (int o = P; o < 32; o <<= 1)
#pragma unroll
        for (int h = 0; h < CH; ++h)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[h][c] += __shfl_xor_sync(FULL, acc[h][c], o);
    if (grp == 0) {
        float* dvrow = a.dV + gk * (int64_t)dv;
#pragma unroll
        for (int h = 0; h < CH; ++h) {
            const int ch = l + h * P;
            if (ch < nch)
                reinterpret_cast<float4*>(dvrow)[ch] =
                    make_float4((float)acc[h][0], (float)acc[h][1], (float)acc[h][2], (float)acc[h][3]);
        }
    }
#pragma unroll
    for (int d = 0; d < DK; ++d) dk[d] = warp_sum(dk[d]);
    if (lane < DK) {
        double v = 0.0;
#pragma unroll
        for (int d = 0; d < DK; ++d) v = (lane == d) ? dk[d] : v;
        a.dK[gk * DK + lane] = (float)v;
    }
}


// per-(d_k, storage type) launchers (explicitly instantiated by bwd_inst.cu's units)
template <int DK, typename TV>
void launch_bwd_query_dk(const BwdArgs& a, int P, int nch, int dv, int k, unsigned grid, cudaStream_t st);
template <int DK, typename TV>
void launch_bwd_key_dk(const KeyArgs& ka, int P, int dv, unsigned grid, cudaStream_t st);

}  // namespace onedf
