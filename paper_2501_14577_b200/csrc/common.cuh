// common.cuh -- shared device helpers for the onedf sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "onedf.h"

namespace onedf {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARP = 32;

// Flag bits written into the header of a workspace (see onedf.h "Errors"):
// one 32-bit word per op (ONEDF_OP_ENCODE .. ONEDF_OP_BWD), each zeroed only
// by its own op, so a workspace shared by the whole pipeline keeps every op's
// flags until that op runs again.
enum : unsigned { FLAG_NONFINITE_INPUT = 1u, FLAG_BAD_EPS = 2u };
constexpr int FLAG_WORDS = 4;

// Every workspace starts with this many bytes of header (flag word + pad).
constexpr size_t WS_HEADER = 256;

__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Carves consecutive 256-B aligned regions out of a workspace.
struct Carver {
    char* base;
    size_t off;
    __host__ Carver(void* b) : base((char*)b), off(WS_HEADER) {}
    template <typename T>
    __host__ T* take(size_t count) {
        off = align_up(off, 256);
        T* p = base ? (T*)(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
    __host__ size_t bytes() const { return align_up(off, 256); }
};

// Record of one sorted key: d_k coordinates, the original position (int bits),
// padded to a multiple of 4 floats so one run entry is 1-3 float4 loads.
template <int DK>
struct RecW { static constexpr int value = (DK + 1 + 3) / 4 * 4; };

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------- value rows (V, O, dO, dV)
// Storage type of the d_v-wide rows (onedf_problem.vdtype, reading D26): float,
// or bfloat16 widened exactly on load and rounded once (RN) from f64 on store.
// A row is addressed in chunks of 4 values (16 B float / 8 B bf16).
using bf16 = __nv_bfloat16;

__device__ __forceinline__ float4 ld4(const float* p, int64_t c4) {
    return __ldg(reinterpret_cast<const float4*>(p) + c4);
}
__device__ __forceinline__ float4 ld4(const bf16* p, int64_t c4) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p) + c4);
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                       __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}
// one value (the column scans)
__device__ __forceinline__ float ld1(const float* p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ float ld1(const bf16* p, int64_t i) {
    return __uint_as_float((unsigned)__ldg(reinterpret_cast<const unsigned short*>(p) + i) << 16);
}

__device__ __forceinline__ void st4(float* p, int64_t c4, double a, double b, double c, double d) {
    reinterpret_cast<float4*>(p)[c4] = make_float4((float)a, (float)b, (float)c, (float)d);
}
__device__ __forceinline__ unsigned bf16_bits(double x) {
    return (unsigned)__bfloat16_as_ushort(__double2bfloat16(x));     // cvt.rn.bf16.f64: one rounding
}
__device__ __forceinline__ void st4(bf16* p, int64_t c4, double a, double b, double c, double d) {
    reinterpret_cast<uint2*>(p)[c4] = make_uint2(bf16_bits(a) | (bf16_bits(b) << 16), bf16_bits(c) | (bf16_bits(d) << 16));
}
__device__ __forceinline__ void st1(float* p, int64_t i, double x) { p[i] = (float)x; }
__device__ __forceinline__ void st1(bf16* p, int64_t i, double x) { p[i] = __double2bfloat16(x); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
    return __shfl_sync(FULL, v, src);
}

// f32 ranking distance in the pinned order ((0 + t0^2) + t1^2) + ...; the
// _rn intrinsics forbid FMA contraction (reading D23).
template <int DK>
__device__ __forceinline__ float rank_dist32(const float* q, const float* k) {
    // 0 + t0^2 == t0^2 exactly (t0^2 >= +0), so the chain starts at t0^2
    const float t0 = __fsub_rn(q[0], k[0]);
    float acc = __fmul_rn(t0, t0);
#pragma unroll
    for (int d = 1; d < DK; ++d) {
        float t = __fsub_rn(q[d], k[d]);
        acc = __fadd_rn(acc, __fmul_rn(t, t));
    }
    return acc;
}

// Sum of 4 f32 products in the fixed order ((a0 b0 + a1 b1) + a2 b2) + a3 b3 with explicit
// roundings (no contraction choice left to the compiler): the f32 group of the gathers, which the
// caller adds into an f64 accumulator -- one f32->f64 conversion per 4 products (reading R5).
__device__ __forceinline__ float sum4(float a0, float b0, float a1, float b1, float a2, float b2, float a3,
                                      float b3) {
    float s = __fmul_rn(a0, b0);
    s = __fmaf_rn(a1, b1, s);
    s = __fmaf_rn(a2, b2, s);
    return __fmaf_rn(a3, b3, s);
}

// f64 squared distance used for the Cauchy weights (exact products of f32 data).
template <int DK>
__device__ __forceinline__ double dist64(const float* q, const float* k) {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < DK; ++d) {
        double t = (double)q[d] - (double)k[d];
        acc = fma(t, t, acc);
    }
    return acc;
}

// ---------------------------------------------------------------- warp sorting of u64 keys
__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) { return a < b ? b : a; }

// Ascending bitonic sort of one key per lane (element e = lane).
__device__ __forceinline__ unsigned long long warp_sort32(unsigned long long x) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const unsigned long long y = __shfl_xor_sync(FULL, x, stride);
            const bool up = (lane & size) == 0 || size == 32;
            const bool lower = (lane & stride) == 0;
            x = (lower == up) ? umin64(x, y) : umax64(x, y);
        }
    }
    return x;
}

// Ascending bitonic sort of 32*R keys spread over the warp (element e = r*32 + lane).
template <int R>
__device__ __forceinline__ void warp_sort(unsigned long long (&x)[R]) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 32 * R; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
                const int rs = stride / 32;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if ((r & rs) == 0) {
                        const bool up = ((r * 32) & size) == 0;
                        const unsigned long long a = x[r], b = x[r + rs];
                        const unsigned long long lo = umin64(a, b), hi = umax64(a, b);
                        x[r] = up ? lo : hi;
                        x[r + rs] = up ? hi : lo;
                    }
                }
            } else {
                const bool lower = (lane & stride) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const bool up = size >= 32 ? ((r * 32) & size) == 0 : (lane & size) == 0;
                    const unsigned long long y = __shfl_xor_sync(FULL, x[r], stride);
                    x[r] = (lower == up) ? umin64(x[r], y) : umax64(x[r], y);
                }
            }
        }
    }
}

// Ascending bitonic sort of 32*R u32 keys spread over the warp (element e = r*32 + lane).
template <int R>
__device__ __forceinline__ void warp_sort_u32(uint32_t (&x)[R]) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 32 * R; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
                const int rs = stride / 32;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if ((r & rs) == 0) {
                        const bool up = ((r * 32) & size) == 0;
                        const uint32_t a = x[r], b = x[r + rs];
                        const uint32_t lo = min(a, b), hi = max(a, b);
                        x[r] = up ? lo : hi;
                        x[r + rs] = up ? hi : lo;
                    }
                }
            } else {
                const bool lower = (lane & stride) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const bool up = size >= 32 ? ((r * 32) & size) == 0 : (lane & size) == 0;
                    const uint32_t y = __shfl_xor_sync(FULL, x[r], stride);
                    x[r] = (lower == up) ? min(x[r], y) : max(x[r], y);
                }
            }
        }
    }
}

// Sequence sharding (onedf.h "Sequence sharding"): chunk c of every (b,h)
// belongs to rank owner(c) (zig-zag over 2*world); a rank computes the
// queries of its chunks.  world <= 1: everything is owned.
struct Shard {
    int32_t rank = 0, world = 1;
    int64_t M = 1, C = 1;          // chunk length, chunks per (b,h)
    __host__ __device__ static int32_t owner(int64_t c, int32_t world) {
        const int64_t g = c % (2 * (int64_t)world);
        return (int32_t)(g < world ? g : 2 * (int64_t)world - 1 - g);
    }
    __host__ __device__ bool on() const { return world > 1; }
    __host__ __device__ bool owns_row(int64_t i) const { return world <= 1 || owner(i / M, world) == rank; }
    // t-th owned chunk in ascending order
    __host__ __device__ int64_t chunk_of(int64_t t) const {
        const int64_t P2 = 2 * (int64_t)world;
        return P2 * (t / 2) + ((t & 1) ? P2 - 1 - rank : rank);
    }
    __host__ int64_t n_owned() const {
        if (world <= 1) return C;
        int64_t t = 0;
        while (chunk_of(t) < C) ++t;
        return t;
    }
    // query-schedule slots per (b,h): all N, or the owned chunks padded to M
    __host__ int64_t slots(int64_t N) const { return world <= 1 ? N : n_owned() * M; }
    // slot s of a (b,h) -> schedule position (chunk-major); false for padding
    __device__ __forceinline__ bool slot_pos(int64_t s, int64_t N, int64_t& pos) const {
        if (world <= 1) { pos = s; return true; }
        const int64_t t = s / M;
        pos = chunk_of(t) * M + (s - t * M);
        return pos < N;
    }
};

// Attention scores (onedf.h ONEDF_SCORE_*, reading D24).  score_raw is the
// weight S itself for the sum-normalised scores (CAUCHY, INV_EUCLID) and the
// logit x (S = exp(x)) for the softmax scores (NEG_EUCLID, DOT).
enum : int { SC_CAUCHY = 0, SC_NEG = 1, SC_INV = 2, SC_DOT = 3 };
__host__ __device__ inline bool score_is_exp(int sc) { return sc == SC_NEG || sc == SC_DOT; }

template <int DK, typename KT>
__device__ __forceinline__ double dot64(const float* q, const KT* k) {
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < DK; ++d) acc = fma((double)q[d], (double)k[d], acc);
    return acc;
}

template <int DK>
__device__ __forceinline__ double score_raw(int sc, const float* q, const float* k, double eps) {
    if (sc == SC_DOT) return dot64<DK>(q, k) * (1.0 / sqrt((double)DK));
    const double D = dist64<DK>(q, k);
    if (sc == SC_CAUCHY) return 1.0 / (D + eps);
    if (sc == SC_INV) return 1.0 / (sqrt(D) + 1e-6);
    return -D;
}

__device__ __forceinline__ void set_flag(void* ws, int op, unsigned bit) {
    atomicOr((unsigned*)ws + op, bit);
}

}  // namespace onedf

// value storage type of a problem (onedf.h ONEDF_DTYPE_*) as a C++ type TV
#define ONEDF_DISPATCH_TV(vdtype, ...)                                       \
    if ((vdtype) == ONEDF_DTYPE_BF16) { using TV = onedf::bf16; __VA_ARGS__; } \
    else { using TV = float; __VA_ARGS__; }

#define ONEDF_DISPATCH_DK(dk, ...)                        \
    switch (dk) {                                         \
        case 1: { constexpr int DK = 1; __VA_ARGS__; } break; \
        case 2: { constexpr int DK = 2; __VA_ARGS__; } break; \
        case 3: { constexpr int DK = 3; __VA_ARGS__; } break; \
        case 4: { constexpr int DK = 4; __VA_ARGS__; } break; \
        case 5: { constexpr int DK = 5; __VA_ARGS__; } break; \
        case 6: { constexpr int DK = 6; __VA_ARGS__; } break; \
        case 7: { constexpr int DK = 7; __VA_ARGS__; } break; \
        default: { constexpr int DK = 8; __VA_ARGS__; } break; \
    }
