// Compile-time-specialised yz-plane spectral kernel (the w-update core,
// admm.cpp:83-95) for power-of-two planes that fit one CTA's shared memory.
//
// Each axis transform is two register-resident DIF stages (radix R1, then R2 on
// contiguous blocks), so a plane makes 6 shared-memory round trips per w-update:
//   global -> [y1] -> smem -> [y2] -> smem -> [z1] -> smem
//          -> [z2 * m z2^-1] -> smem -> [z1^-1] -> smem -> [y2^-1] -> smem -> [y1^-1] -> global
// The forward z2 stage, the regulariser multiply and the adjoint z2 stage touch the
// same elements, so they fuse in registers.  Outputs stay digit-reversed between the
// forward and adjoint halves; the multiplier is indexed through position tables.
//
// Shared layout: element (y, z) at z*P + y + y/R2y, P = NY + NY/R2y rounded to 8 mod 16
// complex: conflict-free for the strided stage-1 rows, the contiguous stage-2 blocks
// (one pad per block) and for column access (consecutive y per half-warp).
#pragma once

#include "fft_device.cuh"
#include "launch.h"

namespace dregb {

template <bool INV, class C>
__device__ __forceinline__ C cmul_tw(C a, C w) {
    return INV ? cmulc(a, w) : cmul(a, w);
}

// 16-point DFT in natural order: j = j1 + 4 j2, k = k2 + 4 k1.
template <bool INV, class C>
__device__ __forceinline__ void dft16(C* x) {
    using R = typename CT<C>::R;
    const R c1 = (R)0.92387953251128675612818318939679, s1 = (R)0.38268343236508977172845998403040;
    const R h = (R)0.70710678118654752440084436210485;
    // W16^e, e = 0..9 (forward sign)
    const C W[10] = {CT<C>::make(1, 0),  CT<C>::make(c1, -s1), CT<C>::make(h, -h),   CT<C>::make(s1, -c1),
                     CT<C>::make(0, -1), CT<C>::make(-s1, -c1), CT<C>::make(-h, -h), CT<C>::make(-c1, -s1),
                     CT<C>::make(-1, 0), CT<C>::make(-c1, s1)};
    C a[4][4];
#pragma unroll
    for (int j1 = 0; j1 < 4; ++j1) {
#pragma unroll
        for (int j2 = 0; j2 < 4; ++j2) a[j1][j2] = x[j1 + 4 * j2];
        dft4<INV>(a[j1]);
    }
#pragma unroll
    for (int j1 = 1; j1 < 4; ++j1)
#pragma unroll
        for (int k2 = 1; k2 < 4; ++k2)
            a[j1][k2] = (j1 * k2 == 4) ? rot_mi<INV>(a[j1][k2]) : cmul_tw<INV>(a[j1][k2], W[j1 * k2]);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
        C b[4] = {a[0][k2], a[1][k2], a[2][k2], a[3][k2]};
        dft4<INV>(b);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) x[k2 + 4 * k1] = b[k1];
    }
}

template <bool INV, int R, class C>
__device__ __forceinline__ void rdft(C* x) {
    static_assert(R == 2 || R == 4 || R == 8 || R == 16, "rdft: radix 2, 4, 8 or 16");
    if constexpr (R == 2) dft2<INV>(x);
    else if constexpr (R == 4) dft4<INV>(x);
    else if constexpr (R == 8) dft8<INV>(x);
    else dft16<INV>(x);
}

template <int NY, int R2Y>
struct PlaneLayout {
    static constexpr int base = NY + NY / R2Y;
    static constexpr int P = base + ((8 - (base % 16) + 16) % 16);
    __device__ static __forceinline__ int at(int y, int z) { return z * P + y + y / R2Y; }
};

template <int NY, int NZ, int R1Y, int R1Z, int NT, int MODE>
__global__ void __launch_bounds__(NT, (NY * NZ <= 8192) ? 3 : 1) plane_fast_kernel(PArgs a) {
    constexpr int R2Y = NY / R1Y, R2Z = NZ / R1Z;
    using Lay = PlaneLayout<NY, R2Y>;
    const int pair = blockIdx.y;
    PairState* st = a.F.st + pair;
    if (!st->active || st->status) return;
    if (st->solve_done && (!a.need_tail || a.k > st->done_iter)) return;

    extern __shared__ __align__(16) unsigned char smem[];
    float2* buf = reinterpret_cast<float2*>(smem);
    double* red = reinterpret_cast<double*>(buf + NZ * Lay::P);
    TwEntry* twy = reinterpret_cast<TwEntry*>(red + 32);  // tables staged once per CTA
    TwEntry* twz = twy + NY;
    float* sys = reinterpret_cast<float*>(twz + NZ);
    float* szs = sys + NY;
    const int tid = threadIdx.x;
    const int hx = a.F.hx;
    const int c = blockIdx.x / hx, p = blockIdx.x - c * hx;
    float2* Sp = a.F.S + ((size_t)pair * 3 * hx + (size_t)c * hx + p) * (size_t)a.F.lines;
    for (int i = tid; i < NY; i += NT) {
        twy[i] = tw_entry(__ldg(a.twy + i));
        sys[i] = __ldg(a.sy_fast + i);
    }
    for (int i = tid; i < NZ; i += NT) {
        twz[i] = tw_entry(__ldg(a.twz + i));
        szs[i] = __ldg(a.sz_fast + i);
    }
    __syncthreads();

    // y stage 1 (DIF radix R1Y, n1 = R2Y), straight from global
#pragma unroll
    for (int b = tid; b < NZ * R2Y; b += NT) {
        const int j1 = b % R2Y, z = b / R2Y;
        float2 x[R1Y];
#pragma unroll
        for (int t = 0; t < R1Y; ++t) x[t] = __ldg(Sp + z * NY + j1 + R2Y * t);
        rdft<false, R1Y>(x);
#pragma unroll
        for (int k = 1; k < R1Y; ++k) x[k] = cmul_t(x[k], twy[j1 * k]);
#pragma unroll
        for (int k = 0; k < R1Y; ++k) buf[Lay::at(j1 + R2Y * k, z)] = x[k];
    }
    __syncthreads();
    // y stage 2 (radix R2Y on contiguous blocks)
    for (int b = tid; b < NZ * R1Y; b += NT) {
        const int blk = b % R1Y, z = b / R1Y;
        float2 x[R2Y];
#pragma unroll
        for (int e = 0; e < R2Y; ++e) x[e] = buf[Lay::at(blk * R2Y + e, z)];
        rdft<false, R2Y>(x);
#pragma unroll
        for (int e = 0; e < R2Y; ++e) buf[Lay::at(blk * R2Y + e, z)] = x[e];
    }
    __syncthreads();
    // z stage 1 (DIF radix R1Z, n1 = R2Z)
    for (int b = tid; b < NY * R2Z; b += NT) {
        const int y = b % NY, j1 = b / NY;
        float2 x[R1Z];
#pragma unroll
        for (int t = 0; t < R1Z; ++t) x[t] = buf[Lay::at(y, j1 + R2Z * t)];
        rdft<false, R1Z>(x);
#pragma unroll
        for (int k = 1; k < R1Z; ++k) x[k] = cmul_t(x[k], twz[j1 * k]);
#pragma unroll
        for (int k = 0; k < R1Z; ++k) buf[Lay::at(y, j1 + R2Z * k)] = x[k];
    }
    __syncthreads();
    // z stage 2 + multiplier + adjoint z stage 2 (or the energy sum)
    const float sxp = __ldg(a.sx + p);
    const int order = a.order;
    double acc = 0.0;
    for (int b = tid; b < NY * R1Z; b += NT) {
        const int y = b % NY, blk = b / NY;
        float2 x[R2Z];
#pragma unroll
        for (int e = 0; e < R2Z; ++e) x[e] = buf[Lay::at(y, blk * R2Z + e)];
        rdft<false, R2Z>(x);
        const float sy = sys[y];
        if (MODE == 0) {
            const float sxy = sxp + sy;
#pragma unroll
            for (int e = 0; e < R2Z; ++e) {
                // theta / (lambda (2 s)^n + theta) / N, s = 3 - cos - cos - cos (regularizer.cpp:69-73)
                const float base = 2.0f * (sxy + szs[blk * R2Z + e]);
                const float b2 = base * base;
                float K = (order & 1) ? base : 1.0f;
                K *= order >= 2 ? b2 : 1.0f;
                K *= order >= 4 ? b2 : 1.0f;
                K *= order >= 6 ? b2 : 1.0f;
                const float m = a.scale * rcp_nr(fmaf(a.lambda, K, a.theta));
                x[e] = cscale(x[e], m);
            }
            rdft<true, R2Z>(x);
#pragma unroll
            for (int e = 0; e < R2Z; ++e) buf[Lay::at(y, blk * R2Z + e)] = x[e];
        } else {
#pragma unroll
            for (int e = 0; e < R2Z; ++e) {
                const double base = 2.0 * ((double)sxp + (double)sy + (double)szs[blk * R2Z + e]);
                double K = base;
                for (int q = 1; q < a.order; ++q) K *= base;
                acc += K * ((double)x[e].x * x[e].x + (double)x[e].y * x[e].y);
            }
        }
    }
    if (MODE == 1) {
        const bool self_conj = (p == 0) || (2 * p == a.F.M);
        const double vals[1] = {block_sum<NT>(acc, red) * (self_conj ? 1.0 : 2.0)};
        double tot[1];
        if (reduce_partials<NT, 1>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot,
                                      red) &&
            tid == 0)
            a.energy_out[pair] = 0.5 * tot[0] / (double)a.F.N;
        return;
    }
    __syncthreads();
    // adjoint z stage 1
    for (int b = tid; b < NY * R2Z; b += NT) {
        const int y = b % NY, j1 = b / NY;
        float2 x[R1Z];
#pragma unroll
        for (int k = 0; k < R1Z; ++k) x[k] = buf[Lay::at(y, j1 + R2Z * k)];
#pragma unroll
        for (int k = 1; k < R1Z; ++k) x[k] = cmulc_t(x[k], twz[j1 * k]);
        rdft<true, R1Z>(x);
#pragma unroll
        for (int t = 0; t < R1Z; ++t) buf[Lay::at(y, j1 + R2Z * t)] = x[t];
    }
    __syncthreads();
    // adjoint y stage 2
    for (int b = tid; b < NZ * R1Y; b += NT) {
        const int blk = b % R1Y, z = b / R1Y;
        float2 x[R2Y];
#pragma unroll
        for (int e = 0; e < R2Y; ++e) x[e] = buf[Lay::at(blk * R2Y + e, z)];
        rdft<true, R2Y>(x);
#pragma unroll
        for (int e = 0; e < R2Y; ++e) buf[Lay::at(blk * R2Y + e, z)] = x[e];
    }
    __syncthreads();
    // adjoint y stage 1, straight to global
#pragma unroll 2
    for (int b = tid; b < NZ * R2Y; b += NT) {
        const int j1 = b % R2Y, z = b / R2Y;
        float2 x[R1Y];
#pragma unroll
        for (int k = 0; k < R1Y; ++k) x[k] = buf[Lay::at(j1 + R2Y * k, z)];
#pragma unroll
        for (int k = 1; k < R1Y; ++k) x[k] = cmulc_t(x[k], twy[j1 * k]);
        rdft<true, R1Y>(x);
#pragma unroll
        for (int t = 0; t < R1Y; ++t) Sp[z * NY + j1 + R2Y * t] = x[t];
    }
}

// Register-blocked yz-plane kernel (radix-8 / radix-R1Z first stages).  Thread
// (y1, z1) holds the 8 x R1Z sub-grid {(y1 + R2Y*t, z1 + R2Z*u)} in registers, so the
// first DIF stage of BOTH axes runs straight out of the global load and the last
// adjoint stage of both axes straight into the global store:
//   global -> [y1, z1] -> smem -> [y2] -> smem -> [z2 * m z2^-1] -> smem
//          -> [y2^-1] -> smem -> [z1^-1, y1^-1] -> global
// i.e. 4 shared-memory round trips instead of plane_fast_kernel's 6, and each
// thread loads its first-stage twiddles once per plane instead of once per
// butterfly.  Positions and multiplier tables are those of plane_fast_kernel with
// R1Y = 8 and the same R1Z (same digit-reversed placement), so results agree to
// rounding.
//
// The multiplier theta / (lambda K_n + theta) / N is evaluated as
// 1 / ((lambda N / theta) K_n + N) with K_n = (2 s)^n, the doubled position tables
// staged in shared memory and n a compile-time constant (ORD 1..3; 0 = run-time n).
template <int ORD>
__device__ __forceinline__ float kn_pow(float base, int order) {
    if constexpr (ORD == 1) return base;
    else if constexpr (ORD == 2) return base * base;
    else if constexpr (ORD == 3) return base * (base * base);
    else {
        const float b2 = base * base;
        float K = (order & 1) ? base : 1.0f;
        K *= order >= 2 ? b2 : 1.0f;
        K *= order >= 4 ? b2 : 1.0f;
        K *= order >= 6 ? b2 : 1.0f;
        return K;
    }
}

//
// MODE 2 is the spectral-state iteration: the plane holds V^_j = r2c_x(v_j);
// the ADMM state lives here, in the 3-D Fourier domain, as U_j = FFT(v_j + b_hat_{j-1})
// (two iterates, ping-pong).  With m = theta / (lambda K_n + theta) the reference's
// w_j = m U_j and b_j = (1 - m) U_j (admm.cpp:66-101,142-153), so with the extrapolated
// Ut_j = U_j + c_{j-1} (U_j - U_{j-1}) (admm.cpp:130-139, linear in w and b alike)
//     b_hat_j = (1 - m) Ut_j,   w_hat_j - b_hat_j = (2 m - 1) Ut_j.
// One pass:  U_j = yzFFT(V^_j) + (1 - m) Ut_{j-1};  store U_j over U_{j-2};
//            plane <- yzFFT^-1((2 m - 1) Ut_j / N)   (= the v-update's argument, x-spectrum).
// Element (b, e) of a plane's state sits at e * (NY * R1Z) + b (coalesced per e).
// UPF = state elements per load batch: batch 0 is issued before the forward radix-R2Z, batch
// n + 1 before batch n is consumed (register software pipeline); MINB = CTAs per SM.
template <int NY, int NZ, int R1Z, int MODE, int ORD, int MINB = ((NY * NZ <= 8192) ? 3 : 1), int UPF = 4>
__global__ void __launch_bounds__((NY / 8) * (NZ / R1Z), MINB) plane_reg_kernel(PArgs a) {
    constexpr int R2Y = NY / 8, R2Z = NZ / R1Z, NT = R2Y * R2Z;
    static_assert(R2Y <= 16 && R2Z <= 16 && (R1Z == 2 || R1Z == 4 || R1Z == 8), "radix split outside rdft<>");
    using Lay = PlaneLayout<NY, R2Y>;
    const int pair = blockIdx.y;
    if (a.pf_ahead && threadIdx.x == 0) {
        // L2 prefetch of the plane the CTA starting about one wave later will load
        // (blocks are dispatched in linear order as resident slots free up)
        // (a negative DREG_PLANE_PF prefetches unconditionally: the A/B knob for the check below)
        const unsigned lin = blockIdx.y * gridDim.x + blockIdx.x + (unsigned)(a.pf_ahead < 0 ? -a.pf_ahead : a.pf_ahead);
        if (lin < gridDim.x * gridDim.y) {
            // only for a plane that will be transformed: the CTAs of finished pairs exit below, and a
            // 64 KB prefetch from each of them made an all-finished launch cost 0.5 ms of HBM time
            const PairState* ts = a.F.st + lin / gridDim.x;
            const bool live = ts->active && !ts->status && !(ts->solve_done && (!a.need_tail || a.k > ts->done_iter));
            if (live || a.pf_ahead < 0) {
                const float2* nxt = a.F.S + (size_t)lin * (size_t)a.F.lines;  // plane index pair*3*hx + c*hx + p
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"((unsigned)(NY * NZ * 8)) : "memory");
            }
        }
    }
    PairState* st = a.F.st + pair;
    if (!st->active || st->status) return;
    if (st->solve_done && (!a.need_tail || a.k > st->done_iter)) return;

    extern __shared__ __align__(16) unsigned char smem[];
    float2* buf = reinterpret_cast<float2*>(smem);
    double* red = reinterpret_cast<double*>(buf + NZ * Lay::P);
    float2* twy = reinterpret_cast<float2*>(red + 32);
    float2* twz = twy + NY;
    float* sys = reinterpret_cast<float*>(twz + NZ);
    float* szs = sys + NY;
    const int tid = threadIdx.x;
    const int hx = a.F.hx;
    const int c = blockIdx.x / hx, p = blockIdx.x - c * hx;
    float2* Sp = a.F.S + ((size_t)pair * 3 * hx + (size_t)c * hx + p) * (size_t)a.F.lines;
    const int y1 = tid % R2Y, z1 = tid / R2Y;
    if (MODE == 2 && tid == 0 && a.ss_prefetch) {
        // this plane's state iterates are needed after the forward transforms: bring them to L2 now
        const size_t pl = ((size_t)pair * 3 * hx + (size_t)c * hx + p) * (size_t)(NY * NZ);
        if (a.has1)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.U1 + pl), "r"((unsigned)(NY * NZ * 8)) : "memory");
        if (a.has0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.U0 + pl), "r"((unsigned)(NY * NZ * 8)) : "memory");
    }

    // stage A: global -> registers (all loads in flight at once)
    float2 x[R1Z][8];  // [z sub-index][y sub-index]
#pragma unroll
    for (int u = 0; u < R1Z; ++u)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const float2* src = Sp + (z1 + R2Z * u) * NY + y1 + R2Y * t;
            // MODE 2 streams five half-spectra through L2: every line is touched once (evict first)
            x[u][t] = (MODE == 2 && a.ss_stream) ? __ldcs(src) : __ldg(src);
        }
    // position tables doubled (exact) for the multiplier base 2 (sx + sy + sz)
    const float dbl = MODE != 1 ? 2.0f : 1.0f;
    for (int i = tid; i < NY; i += NT) {
        twy[i] = __ldg(a.twy + i);
        sys[i] = dbl * __ldg(a.sy_fast + i);
    }
    for (int i = tid; i < NZ; i += NT) {
        twz[i] = __ldg(a.twz + i);
        szs[i] = dbl * __ldg(a.sz_fast + i);
    }
    // y stage 1: radix 8 over t, twiddle W_NY^(y1 k)
#pragma unroll
    for (int u = 0; u < R1Z; ++u) dft8<false>(x[u]);
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        const float2 w = __ldg(a.twy + y1 * k);
#pragma unroll
        for (int u = 0; u < R1Z; ++u) x[u][k] = cmul(x[u][k], w);
    }
    // z stage 1: radix R1Z over u, twiddle W_NZ^(z1 k)
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        float2 col[R1Z];
#pragma unroll
        for (int u = 0; u < R1Z; ++u) col[u] = x[u][t];
        rdft<false, R1Z>(col);
#pragma unroll
        for (int u = 0; u < R1Z; ++u) x[u][t] = col[u];
    }
#pragma unroll
    for (int k = 1; k < R1Z; ++k) {
        const float2 w = __ldg(a.twz + z1 * k);
#pragma unroll
        for (int t = 0; t < 8; ++t) x[k][t] = cmul(x[k][t], w);
    }
#pragma unroll
    for (int u = 0; u < R1Z; ++u)
#pragma unroll
        for (int t = 0; t < 8; ++t) buf[Lay::at(y1 + R2Y * t, z1 + R2Z * u)] = x[u][t];
    __syncthreads();
    // y stage 2 (radix R2Y on contiguous blocks)
    for (int b = tid; b < NZ * 8; b += NT) {
        const int blk = b % 8, z = b / 8;
        float2 v[R2Y];
#pragma unroll
        for (int e = 0; e < R2Y; ++e) v[e] = buf[Lay::at(blk * R2Y + e, z)];
        rdft<false, R2Y>(v);
#pragma unroll
        for (int e = 0; e < R2Y; ++e) buf[Lay::at(blk * R2Y + e, z)] = v[e];
    }
    __syncthreads();
    // z stage 2 + multiplier + adjoint z stage 2 (or the energy sum)
    const float sxp = dbl * __ldg(a.sx + p);
    const int order = a.order;
    const float lam_n = a.lam_n, n_f = a.n_f;
    double acc = 0.0;
    for (int b = tid; b < NY * R1Z; b += NT) {
        const int y = b % NY, blk = b / NY;
        float2 v[R2Z];
        float2 u1[R2Z], u0[R2Z];  // MODE 2: U_{j-1}, U_{j-2} of this thread's elements
        const float2* U1 = nullptr;
        float2* U0 = nullptr;
        auto load_state = [&](int e0) {
#pragma unroll
            for (int q = 0; q < UPF; ++q) {
                const int e = e0 + q;
                u1[e] = a.has1 ? __ldcs(U1 + (size_t)e * (NY * R1Z)) : make_float2(0.f, 0.f);
                u0[e] = a.has0 ? __ldcs(U0 + (size_t)e * (NY * R1Z)) : u1[e];
            }
        };
        if (MODE == 2) {
            const size_t pl = ((size_t)pair * 3 * hx + (size_t)c * hx + p) * (size_t)(NY * NZ) + b;
            U1 = a.U1 + pl;  // U_{j-1}
            U0 = a.U0 + pl;  // U_{j-2} in, U_j out
            load_state(0);   // in flight across the shared-memory loads and the forward radix
        }
#pragma unroll
        for (int e = 0; e < R2Z; ++e) v[e] = buf[Lay::at(y, blk * R2Z + e)];
        rdft<false, R2Z>(v);
        const float sy = sys[y];
        if (MODE == 2) {
            const float sxy = sxp + sy;  // doubled
            const float cc = a.c_cur, cp = a.c_prev, inv_n = a.inv_nf;
#pragma unroll
            for (int e0 = 0; e0 < R2Z; e0 += UPF) {
                if (e0 + UPF < R2Z) load_state(e0 + UPF);
#pragma unroll
                for (int q = 0; q < UPF; ++q) {
                    const int e = e0 + q;
                    // q_ = (lambda N / theta) K_n:  1 - m = q_ r,  (2 m - 1) / N = (N - q_) r / N,  r = 1 / (q_ + N)
                    const float qk = lam_n * kn_pow<ORD>(sxy + szs[blk * R2Z + e], order);
                    const float r = rcp_nr(qk + n_f);
                    const float m1 = qk * r, m2 = (n_f - qk) * r * inv_n;
                    const float2 utp = make_float2(fmaf(cp, u1[e].x - u0[e].x, u1[e].x), fmaf(cp, u1[e].y - u0[e].y, u1[e].y));
                    const float2 un = make_float2(fmaf(m1, utp.x, v[e].x), fmaf(m1, utp.y, v[e].y));
                    __stcs(U0 + (size_t)e * (NY * R1Z), un);
                    v[e] = make_float2(m2 * fmaf(cc, un.x - u1[e].x, un.x), m2 * fmaf(cc, un.y - u1[e].y, un.y));
                }
            }
            rdft<true, R2Z>(v);
#pragma unroll
            for (int e = 0; e < R2Z; ++e) buf[Lay::at(y, blk * R2Z + e)] = v[e];
        } else if (MODE == 0) {
            const float sxy = sxp + sy;  // doubled
#pragma unroll
            for (int e = 0; e < R2Z; ++e) {
                // theta / (lambda (2 s)^n + theta) / N, s = 3 - cos - cos - cos (regularizer.cpp:69-73)
                const float K = kn_pow<ORD>(sxy + szs[blk * R2Z + e], order);
                v[e] = cscale(v[e], rcp_nr(fmaf(lam_n, K, n_f)));
            }
            rdft<true, R2Z>(v);
#pragma unroll
            for (int e = 0; e < R2Z; ++e) buf[Lay::at(y, blk * R2Z + e)] = v[e];
        } else {
#pragma unroll
            for (int e = 0; e < R2Z; ++e) {
                const double base = 2.0 * ((double)sxp + (double)sy + (double)szs[blk * R2Z + e]);
                double K = base;
                for (int q = 1; q < a.order; ++q) K *= base;
                acc += K * ((double)v[e].x * v[e].x + (double)v[e].y * v[e].y);
            }
        }
    }
    if (MODE == 1) {
        const bool self_conj = (p == 0) || (2 * p == a.F.M);
        const double vals[1] = {block_sum<NT>(acc, red) * (self_conj ? 1.0 : 2.0)};
        double tot[1];
        if (reduce_partials<NT, 1>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot,
                                      red) &&
            tid == 0)
            a.energy_out[pair] = 0.5 * tot[0] / (double)a.F.N;
        return;
    }
    __syncthreads();
    // adjoint y stage 2
    for (int b = tid; b < NZ * 8; b += NT) {
        const int blk = b % 8, z = b / 8;
        float2 v[R2Y];
#pragma unroll
        for (int e = 0; e < R2Y; ++e) v[e] = buf[Lay::at(blk * R2Y + e, z)];
        rdft<true, R2Y>(v);
#pragma unroll
        for (int e = 0; e < R2Y; ++e) buf[Lay::at(blk * R2Y + e, z)] = v[e];
    }
    __syncthreads();
    // stage E: adjoint z stage 1 and y stage 1 in registers, straight to global
#pragma unroll
    for (int u = 0; u < R1Z; ++u)
#pragma unroll
        for (int t = 0; t < 8; ++t) x[u][t] = buf[Lay::at(y1 + R2Y * t, z1 + R2Z * u)];
#pragma unroll
    for (int k = 1; k < R1Z; ++k) {
        const float2 w = twz[z1 * k];
#pragma unroll
        for (int t = 0; t < 8; ++t) x[k][t] = cmulc(x[k][t], w);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        float2 col[R1Z];
#pragma unroll
        for (int u = 0; u < R1Z; ++u) col[u] = x[u][t];
        rdft<true, R1Z>(col);
#pragma unroll
        for (int u = 0; u < R1Z; ++u) x[u][t] = col[u];
    }
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        const float2 w = twy[y1 * k];
#pragma unroll
        for (int u = 0; u < R1Z; ++u) x[u][k] = cmulc(x[u][k], w);
    }
#pragma unroll
    for (int u = 0; u < R1Z; ++u) {
        dft8<true>(x[u]);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            float2* dst = Sp + (z1 + R2Z * u) * NY + y1 + R2Y * t;
            if (MODE == 2 && a.ss_stream) __stcs(dst, x[u][t]);
            else *dst = x[u][t];
        }
    }
}

}  // namespace dregb
