// Shared device helpers for the dreg B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dreg_cuda.h"

namespace dregb {

constexpr int kMaxStages = 12;      // radix stages per line FFT
constexpr int kMaxRadix = 64;       // largest prime factor handled by the generic butterfly
constexpr int kMaxPartials = 4096;  // per-pair partial-sum slots per reduction

// Per-axis line-FFT plan (host-built, passed by value).  Stage s of the DIF
// forward transform uses radix[s] on sub-blocks of n1[s]*radix[s] elements;
// twiddle W_{n_s}^{j1 k} = W_n^{j1 k tws[s]} is read from the axis table.
// Division by a run-time constant via multiply-high (valid for x < 2^31).
struct FastDiv {
    unsigned int d, mul, shift;
    void init(unsigned int dv) {
        d = dv;
        unsigned int l = 0;
        while ((1u << l) < dv) ++l;
        mul = (unsigned int)((((unsigned long long)1 << 32) * (((unsigned long long)1 << l) - dv)) / dv + 1);
        shift = l;
    }
    __device__ __forceinline__ unsigned int div(unsigned int x) const {
        return (__umulhi(x, mul) + x) >> shift;
    }
};

struct AxisPlan {
    int n;
    int nst;
    int radix[kMaxStages];
    int n1[kMaxStages];
    int tws[kMaxStages];
    FastDiv fn1[kMaxStages];
};

// Per-pair device state driving the warp loop of register_pair
// (registration.cpp:245-271) without host synchronisation.
struct PairState {
    int active;          // level still iterating warps
    int cur;             // accepted phi / warped buffer index
    int solve_done;      // current solve met tol (admm.cpp:304-307)
    int iterations;      // iterations of the current solve
    int status;          // DREG_OK / DREG_NUMERIC
    int velocity_count;  // registration.hpp:42
    int warps;           // accepted warps at the current level
    int level;
    int solves;            // compose/decide passes (= solve_velocity calls)
    unsigned int counter;  // last-block reduction ticket
    int done_iter;         // iteration at which solve_done was raised
    double sad_prev;
    double final_change;
    float lo, hi;          // shared intensity range (registration.cpp:157-166)
    double folding;        // interior voxels with det J <= 0 of the final phi (metrics.cpp:211-228)
    double min_det;        // interior min det J (fp32-cast values, metrics.cpp:222)
    int solver_iterations[DREG_MAX_LEVELS][DREG_MAX_WARPS];
    double mean_sad[DREG_MAX_LEVELS][DREG_MAX_WARPS + 1];
    int level_warps[DREG_MAX_LEVELS];
};

// fp32 complex arithmetic.  DREG_PACKED selects the sm_100 packed forms (FADD2 /
// FMUL2 / FFMA2, one instruction per complex add): 0 = scalar, 1 = packed adds,
// 2 = packed adds and multiplies.  On B200 a packed op issues at half the scalar
// rate (tools/pipebench: 4 scalar vs 2 packed warp-instructions/clk/SM, 128 fp32
// lanes/clk/SM either way), so packing saves issue slots, not FP-pipe time.
#ifndef DREG_PACKED
#define DREG_PACKED 0
#endif
#if DREG_PACKED >= 1
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// a + s * (b.y, b.x): s = (1, -1) gives a - i b, s = (-1, 1) gives a + i b (exact: |s| = 1)
__device__ __forceinline__ float2 cadd_swp(float2 a, float2 b, float2 s) {
    return __ffma2_rn(make_float2(b.y, b.x), s, a);
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cadd_swp(float2 a, float2 b, float2 s) {
    return make_float2(a.x + s.x * b.y, a.y + s.y * b.x);
}
#endif
#if DREG_PACKED >= 2
// a * b given br = (-b.y, b.x) = i b (precomputed for table twiddles)
__device__ __forceinline__ float2 cmul_r(float2 a, float2 b, float2 br) {
    return __ffma2_rn(make_float2(a.y, a.y), br, __fmul2_rn(make_float2(a.x, a.x), b));
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return cmul_r(a, b, make_float2(-b.y, b.x)); }
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), make_float2(b.x, -b.y)));
}
// a * w and a * conj(w) for a twiddle-table entry t = (w.x, w.y, -w.y, w.x): two
// instructions each (the swaps are operand modifiers)
__device__ __forceinline__ float2 cmul_t(float2 a, float4 t) {
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(t.z, t.w), __fmul2_rn(make_float2(a.x, a.x), make_float2(t.x, t.y)));
}
__device__ __forceinline__ float2 cmulc_t(float2 a, float4 t) {
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(t.y, t.x), __fmul2_rn(make_float2(a.x, a.x), make_float2(t.w, t.z)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
#else
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
    return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
#endif
// Twiddle-table entry type of the plane kernel: (w, i w) as float4 when multiplies are
// packed (two instructions per twiddle), plain float2 otherwise (half the LDS width).
#if DREG_PACKED >= 2
using TwEntry = float4;
__device__ __forceinline__ float4 tw_entry(float2 w) { return make_float4(w.x, w.y, -w.y, w.x); }
#else
using TwEntry = float2;
__device__ __forceinline__ float2 tw_entry(float2 w) { return w; }
#endif
__device__ __forceinline__ float2 cmul_t(float2 a, float2 t) { return cmul(a, t); }
__device__ __forceinline__ float2 cmulc_t(float2 a, float2 t) { return cmulc(a, t); }
// 1/d for normal positive d without the IEEE slow path of __frcp_rn: MUFU.RCP plus
// one Newton step (<= 1 ulp); used for the regulariser multiplier, d >= theta > 0.
__device__ __forceinline__ float rcp_nr(float d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return fmaf(r, fmaf(-d, r, 1.0f), r);
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// Barrier policies: the whole CTA, or one warp group on a named barrier (bar.sync id, n).
struct BlockSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
template <int ID, int N>
struct NamedSync {
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory"); }
};

// Deterministic reduction of doubles over a group of NT threads (gtid in [0, NT),
// warp-aligned), fixed tree order.  Result valid in gtid 0.
template <int NT, class Sync>
__device__ __forceinline__ double group_sum(double v, double* red, int gtid, Sync sync) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = gtid & 31, wid = gtid >> 5;
    sync();
    if (lane == 0) red[wid] = v;
    sync();
    double s = 0.0;
    if (gtid == 0) {
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += red[w];
    }
    return s;
}
template <int NT, class Sync>
__device__ __forceinline__ double group_min(double v, double* red, int gtid, Sync sync) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
    const int lane = gtid & 31, wid = gtid >> 5;
    sync();
    if (lane == 0) red[wid] = v;
    sync();
    double s = 1.0e300;
    if (gtid == 0) {
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s = fmin(s, red[w]);
    }
    return s;
}

// Deterministic block reduction of doubles (fixed tree order).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
    return group_sum<NT>(v, red, (int)threadIdx.x, BlockSync{});
}
template <int NT>
__device__ __forceinline__ double block_min(double v, double* red) {
    return group_min<NT>(v, red, (int)threadIdx.x, BlockSync{});
}

// Deterministic cross-block reduction, K sums per block (fixed per-thread strides +
// fixed tree => run-to-run bit-identical).  Every thread of the group must call it.
// gtid 0 writes vals[] as this block's partials into part[k * kMaxPartials + slot];
// the group that arrives last reduces all partials and returns true (totals valid in
// gtid 0 only).  s_last: one shared int owned by the group.
template <int NT, int K, class Sync>
__device__ __forceinline__ bool group_reduce_partials(const double (&vals)[K], double* part, unsigned int* counter,
                                                      unsigned int nblocks, double (&tot)[K], double* red,
                                                      int* s_last, int gtid, Sync sync, unsigned slot,
                                                      unsigned min_mask = 0u) {
    if (gtid == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) part[(size_t)k * kMaxPartials + slot] = vals[k];
        __threadfence();
        const unsigned int t = atomicAdd(counter, 1u);
        *s_last = (t == nblocks - 1);
    }
    sync();
    if (!*s_last) return false;
    __threadfence();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const bool is_min = (min_mask >> k) & 1u;
        double acc = is_min ? 1e300 : 0.0;
        for (unsigned b = gtid; b < nblocks; b += NT) {
            const double v = __ldcg(part + (size_t)k * kMaxPartials + b);
            acc = is_min ? fmin(acc, v) : acc + v;
        }
        tot[k] = is_min ? group_min<NT>(acc, red, gtid, sync) : group_sum<NT>(acc, red, gtid, sync);
    }
    if (gtid == 0) *counter = 0u;
    return true;
}

template <int NT, int K>
__device__ __forceinline__ bool reduce_partials(const double (&vals)[K], double* part, unsigned int* counter,
                                                unsigned int nblocks, double (&tot)[K], double* red,
                                                unsigned min_mask = 0u, int slot = -1) {
    __shared__ int s_last;
    return group_reduce_partials<NT, K>(vals, part, counter, nblocks, tot, red, &s_last, (int)threadIdx.x,
                                        BlockSync{}, slot < 0 ? blockIdx.x : (unsigned)slot, min_mask);
}

// Last-block ticket: returns true in thread 0 of the block that finishes last
// among `nblocks` (per pair).  Callers then reduce the partials in fixed order,
// which keeps every reduction run-to-run bit-deterministic.
__device__ __forceinline__ bool last_block_ticket(unsigned int* counter, unsigned int nblocks) {
    __threadfence();
    const unsigned int t = atomicAdd(counter, 1u);
    const bool last = (t == nblocks - 1);
    if (last) {
        *counter = 0u;
        __threadfence();
    }
    return last;
}

}  // namespace dregb
