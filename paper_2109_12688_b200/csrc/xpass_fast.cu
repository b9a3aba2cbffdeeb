// Compile-time-specialised fused x-pass for x extents M = 16 R2 (line FFT length
// L = M/2 = 8 R2, R2 in {4, 8, 16}: M = 64, 128, 256), TL = 32 x-lines per CTA.
// Same per-voxel semantics as xpass_kernel (admm_kernels.cu; reference
// admm.cpp:23-63,130-153,155-170 and fft.cpp r2c/c2r along x); the difference is the
// FFT plumbing:
//
//  * one cp.async wave stages all three components' spectrum rows, transposed,
//    straight into the FFT buffer (no separate staging buffer, no per-component waits);
//  * the c2r pre-processing (E + iO from X[k], conj X[L-k]) is fused with the first
//    adjoint stage (radix R2 on contiguous position blocks) in registers;
//  * the r2c post-processing is fused with the last forward stage: with
//    L = 8 R2 digit reversal, position block b holds the frequencies k = b (mod 8), so
//    blocks {j, 8-j} hold every partner pair (k, L-k) and one thread finishes both.
// Position of frequency k = 8 p1 + b is R2 b + p1 (same scheme as fft_device.cuh).
#include <algorithm>
#include <type_traits>

#include <cstdlib>
#include "fft_device.cuh"
#include "kernels.cuh"
#include "launch.h"
#include "plane_fast.cuh"
#include "pointwise.cuh"

namespace dregb {

namespace {

constexpr int kFT = 256;  // threads
constexpr int kFTL = 32;  // x-lines per CTA
constexpr int kR1 = 8;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int n = valid ? 8 : 0;  // src-size 0 => zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// HINT 1: streaming loads, no L1 allocation, 256-byte L2 prefetch granule
template <int N, int HINT = 0>
__device__ __forceinline__ void ldvN(const float* p, float* out) {
    if constexpr (N == 4 && HINT == 2) {  // HINT 2: evict-first streaming load (ld.global.cs)
        const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
        out[0] = t.x;
        out[1] = t.y;
        out[2] = t.z;
        out[3] = t.w;
    } else if constexpr (N == 4 && HINT == 1) {
        asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(out[0]), "=f"(out[1]), "=f"(out[2]), "=f"(out[3])
                     : "l"(p));
    } else if constexpr (N == 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        out[0] = t.x;
        out[1] = t.y;
        out[2] = t.z;
        out[3] = t.w;
    } else if constexpr (N == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        out[0] = t.x;
        out[1] = t.y;
    } else {
        out[0] = p[0];
    }
}
template <int N>
__device__ __forceinline__ void stvN(float* p, const float* in) {
    if constexpr (N == 4) *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
    else if constexpr (N == 2) *reinterpret_cast<float2*>(p) = make_float2(in[0], in[1]);
    else p[0] = in[0];
}

}  // namespace

template <class C>
__device__ __forceinline__ float ld_real(const C* line, int x) {
    return (float)reinterpret_cast<const decltype(C::x)*>(line)[x];
}

// u = v + b_hat: formed in the transform's precision (fp64 in precise mode, exactly
// like the reference's real[i] = double(v) + double(b_hat), admm.cpp:77-80)
template <class C>
__device__ __forceinline__ void st_real_sum(C* line, int x, float v, float b) {
    using R = decltype(C::x);
    reinterpret_cast<R*>(line)[x] = (R)v + (R)b;
}

// VEC consecutive reals of a line starting at even x: 64-bit shared accesses (x even)
template <int VEC, class C>
__device__ __forceinline__ void ld_reals(const C* line, int x, float* out) {
    if constexpr (sizeof(C) == 8 && VEC >= 2) {
#pragma unroll
        for (int q = 0; q < VEC; q += 2) {
            const float2 t = line[(x + q) >> 1];
            out[q] = t.x;
            out[q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < VEC; ++q) out[q] = ld_real(line, x + q);
    }
}
template <int VEC, class C>
__device__ __forceinline__ void st_reals_sum(C* line, int x, const float* v, const float* b) {
    if constexpr (sizeof(C) == 8 && VEC >= 2) {
#pragma unroll
        for (int q = 0; q < VEC; q += 2) line[(x + q) >> 1] = make_float2(v[q] + b[q], v[q + 1] + b[q + 1]);
    } else {
#pragma unroll
        for (int q = 0; q < VEC; ++q) st_real_sum(line, x + q, v[q], b[q]);
    }
}

// ---- tile phases (shared by the one-tile-per-CTA kernel and the pipelined kernel) ----
// A tile is TL = 32 consecutive x-lines of one pair, all three components; buf holds
// [3][TL][PM] complex.  `tid` is the thread's index inside the kFT-thread group that
// runs the phase; `sync` is that group's barrier.

// cp.async all three components' spectrum rows (transposed) into buf; caller waits.
// A thread keeps its line l = tid % 32 and walks the (component, x-bin) rows with
// incremental addresses (the index arithmetic was 24 integer instructions per 8-byte
// copy, 17% of the spectral-state x-pass's issue slots).
template <int R2, class C, int NF = kFT>
__device__ __forceinline__ void stage_spectrum(C* buf, const C* S, long long lines, long long L0, int nl,
                                               int tid) {
    constexpr int HX = kR1 * R2 + 1, PM = HX, TL = kFTL;
    static_assert(NF % TL == 0, "a thread keeps its line");
    constexpr int STEP = NF / TL;
    const int l = tid & (TL - 1);
    const bool ok = l < nl;
    const int w = tid >> 5;  // first x-bin of this thread; it then walks p = w, w + STEP, ...
    const size_t sstep = (size_t)STEP * lines;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const C* src = S + ((size_t)c * HX + w) * lines + L0 + (ok ? l : 0);
        C* dst = buf + (c * TL + l) * PM + w;
#pragma unroll
        for (int i = 0; i < (HX + STEP - 1) / STEP; ++i, src += sstep, dst += STEP) {
            if (w + i * STEP < HX) {
                if constexpr (sizeof(C) == 16) *dst = ok ? *src : CT<C>::make(0, 0);  // fp64 storage
                else cp_async8(dst, src, ok);
            }
        }
    }
}

// phase 1: c2r of the staged spectrum -> w_{k-1} (real, natural order) in buf.
template <int R2, class C, class Sync, int NF = kFT>
__device__ __forceinline__ void c2r_tile(C* buf, const C* twx, const C* xtw, int tid, Sync sync) {
    constexpr int L = kR1 * R2, PM = L + 1, TL = kFTL;
    // (a) pre-process + adjoint of the last DIF stage.  In place with cross-task reads
    // inside a line, so each round covers whole lines (LPR lines x 4 block pairs) and
    // separates all reads from all writes.  Line fastest: a half-warp touches 16 lines
    // at one block offset; the odd pitch (2 PM = 130 words = 2 mod 32) spreads them
    // over all 32 banks.
    constexpr int LPR = NF / (kR1 / 2);
#pragma unroll 1
    for (int r0 = 0; r0 < 3 * TL; r0 += LPR) {
        const int line = r0 + tid % LPR, j = tid / LPR;  // line = c * TL + l
        const bool act = line < 3 * TL;
        const C* X = buf + line * PM;
        C z[2][R2];
        if constexpr (sizeof(C) == 8) {
            // fp32: bins k and L - k need the same two inputs A = X[k], B = X[L-k] and share
            // s = A + conj(B), d = A - conj(B), o = d conj(W_M^k) (W_M^{L-k} = -conj(W_M^k)):
            // Z'[k] = (s.x - o.y, s.y + o.x), Z'[L-k] = (s.x + o.y, o.x - s.y) -- half the loads
            // and half the arithmetic of treating the two bins separately.
            auto joint = [&](int k, C& zk, C& zp) {
                const C A = X[k], B = X[L - k], w = xtw[k];
                const C s = CT<C>::make(A.x + B.x, A.y - B.y), d = CT<C>::make(A.x - B.x, A.y + B.y);
                const C o = CT<C>::make(fmaf(d.x, w.x, d.y * w.y), fmaf(d.y, w.x, -(d.x * w.y)));
                zk = CT<C>::make(s.x - o.y, s.y + o.x);
                zp = CT<C>::make(s.x + o.y, o.x - s.y);
            };
            auto single = [&](int k, C& zk) {  // self-paired bins (k = 0 with L, k = L/2)
                C A = X[k];
                C B = X[L - k];
                if (k == 0) {
                    A.y = 0;
                    B.y = 0;
                }
                B.y = -B.y;
                const C e = cadd(A, B);
                const C o = cmulc(csub(A, B), xtw[k]);
                zk = CT<C>::make(e.x - o.y, e.y + o.x);
            };
            if (act) {
                if (j != 0) {  // blocks j and 8 - j: bin 8 p1 + j pairs with 8 (R2-1-p1) + (8 - j)
#pragma unroll
                    for (int p1 = 0; p1 < R2; ++p1) joint(kR1 * p1 + j, z[0][p1], z[1][R2 - 1 - p1]);
                } else {  // block 0 pairs p1 with R2 - p1 (0 and R2/2 are self-paired); block 4 pairs p1 with R2-1-p1
                    single(0, z[0][0]);
                    single(kR1 * (R2 / 2), z[0][R2 / 2]);
#pragma unroll
                    for (int p1 = 1; p1 < R2 / 2; ++p1) joint(kR1 * p1, z[0][p1], z[0][R2 - p1]);
#pragma unroll
                    for (int p1 = 0; p1 < R2 / 2; ++p1) joint(kR1 * p1 + kR1 / 2, z[1][p1], z[1][R2 - 1 - p1]);
                }
                rdft<true, R2>(z[0]);
                rdft<true, R2>(z[1]);
            }
        } else if (act) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int b = q == 0 ? j : (j == 0 ? kR1 / 2 : kR1 - j);
#pragma unroll
                for (int p1 = 0; p1 < R2; ++p1) {
                    const int k = kR1 * p1 + b;
                    C A = X[k];
                    C B = X[L - k];
                    if (k == 0) {
                        A.y = 0;
                        B.y = 0;
                    }
                    B.y = -B.y;
                    const C e = cadd(A, B);
                    const C o = cmulc(csub(A, B), xtw[k]);
                    z[q][p1] = CT<C>::make(e.x - o.y, e.y + o.x);
                }
                rdft<true, R2>(z[q]);
            }
        }
        sync();  // every read of these lines done before any write
        if (act) {
            C* Y = buf + line * PM;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int b = q == 0 ? j : (j == 0 ? kR1 / 2 : kR1 - j);
#pragma unroll
                for (int e = 0; e < R2; ++e) Y[R2 * b + e] = z[q][e];
            }
        }
    }
    sync();
    // (b) adjoint of the first DIF stage: conj twiddle, inverse radix 8 over stride R2
    for (int t = tid; t < 3 * TL * R2; t += NF) {
        const int line = t % (3 * TL), j1 = t / (3 * TL);  // line fastest (conflict-free)
        C* Y = buf + line * PM;
        C x[kR1];
#pragma unroll
        for (int k = 0; k < kR1; ++k) x[k] = Y[j1 + R2 * k];
#pragma unroll
        for (int k = 1; k < kR1; ++k) x[k] = cmulc(x[k], twx[j1 * k]);
        dft8<true>(x);
#pragma unroll
        for (int s = 0; s < kR1; ++s) Y[j1 + R2 * s] = x[s];
    }
    sync();
}

// phase 2: point-wise ADMM updates (fp32) of one tile; accumulates change / residual /
// data-term partials of this thread.
template <int MODE, int DT, int R2, int VEC, int UNR, class C, int NTP = kFT, int HINT = 0>
__device__ __forceinline__ void pointwise_tile(const XArgs& a, C* __restrict__ buf, int pair, long long L0, int nl, int tid,
                                               float& fc, float& fr, float& fo) {
    constexpr int L = kR1 * R2, PM = L + 1, M = 2 * L, TL = kFTL;
    const long long N = a.F.N;
    // the field arrays and the shared-memory tile never alias: __restrict__ lets the unrolled loop
    // hoist the next iteration's global loads above this iteration's shared-memory stores
    float* __restrict__ V = a.F.V + (size_t)pair * 3 * N;
    float* __restrict__ BO = a.F.BH + (size_t)pair * 3 * N;  // b_{k-2} in, b_k out (the dual iterates ping-pong)
    float* __restrict__ WP = a.F.WP + (size_t)pair * 3 * N;
    const float* __restrict__ BP = a.F.BP + (size_t)pair * 3 * N;  // b_{k-1}
    const float* __restrict__ G = a.F.G + (size_t)pair * 3 * N;
    const float* __restrict__ Dd = a.F.D + (size_t)pair * N;
    const float thf = (float)a.sp.theta, ithf = (float)(1.0 / a.sp.theta), epsf = (float)a.sp.epsilon;
    const float cf = (float)a.coef, cpf = (float)a.coef_prev;
    const bool accel = a.sp.accelerate != 0;
    const bool hp = a.coef_prev != 0.0;  // b_hat_{k-1} differs from b_{k-1}
    const size_t base = (size_t)L0 * M;
    const int nvox = nl * M;
#pragma unroll UNR
    for (int i0 = tid * VEC; i0 < nvox; i0 += NTP * VEC) {
        const int l = i0 / M, x0 = i0 - l * M;
        const size_t gi = base + i0;
        float w[3][VEC], vp[3][VEC], bo[3][VEC], wp[3][VEC], bp[3][VEC], g[3][VEC], dv[VEC];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (MODE != X_FIRST && MODE != X_SSN) ldvN<VEC, HINT>(V + (size_t)c * N + gi, vp[c]);
            if (MODE == X_GENERAL) ldvN<VEC, HINT>(BP + (size_t)c * N + gi, bp[c]);        // b_{k-1}
            if (MODE == X_GENERAL && hp) ldvN<VEC, HINT>(BO + (size_t)c * N + gi, bo[c]);  // b_{k-2}
            if (MODE == X_GENERAL && accel) ldvN<VEC, HINT>(WP + (size_t)c * N + gi, wp[c]);
            if (MODE != X_TAIL) ldvN<VEC, HINT>(G + (size_t)c * N + gi, g[c]);
        }
        if (MODE != X_TAIL) ldvN<VEC, HINT>(Dd + gi, dv);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const C* wl = buf + (c * TL + l) * PM;
            if (MODE != X_FIRST) ld_reals<VEC>(wl, x0, w[c]);
#pragma unroll
            for (int jj = 0; jj < VEC; ++jj) {
                if (MODE == X_FIRST) {
                    w[c][jj] = 0.f;
                    vp[c][jj] = 0.f;
                }
                if (MODE == X_SSN) vp[c][jj] = 0.f;
                // b_hat_{k-1} = b_{k-1} + c_{k-2} (b_{k-1} - b_{k-2}) (admm.cpp:130-139), re-formed from
                // the two stored dual iterates -- the bits the previous pass computed -- instead of a
                // stored b_hat field (saves one 12 B/voxel write per iteration)
                if (MODE != X_GENERAL) bo[c][jj] = 0.f;
                else bo[c][jj] = hp ? fmaf(cpf, bp[c][jj] - bo[c][jj], bp[c][jj]) : bp[c][jj];
            }
        }
        if (MODE == X_TAIL) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int jj = 0; jj < VEC; ++jj) {
                    const float dd = vp[c][jj] - w[c][jj];
                    fr = fmaf(dd, dd, fr);
                }
            continue;
        }
        float wh[3][VEC], bh[3][VEC], vn[3][VEC];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int jj = 0; jj < VEC; ++jj) {
                if (MODE == X_FIRST) {
                    wh[c][jj] = 0.f;
                    bh[c][jj] = 0.f;
                    continue;
                }
                if (MODE == X_SS || MODE == X_SSN) {  // the staged field is w_hat - b_hat; u = v
                    wh[c][jj] = w[c][jj];
                    bh[c][jj] = 0.f;
                    continue;
                }
                const float dd = vp[c][jj] - w[c][jj];
                fr = fmaf(dd, dd, fr);
                const float b = bo[c][jj] + dd;  // dual update (admm.cpp:142-153)
                if (MODE == X_GENERAL && accel) {
                    wh[c][jj] = fmaf(cf, w[c][jj] - wp[c][jj], w[c][jj]);  // admm.cpp:130-139
                    bh[c][jj] = fmaf(cf, b - bp[c][jj], b);
                } else {
                    wh[c][jj] = w[c][jj];
                    bh[c][jj] = b;
                }
                bo[c][jj] = b;
            }
#pragma unroll
        for (int jj = 0; jj < VEC; ++jj) {
            const float whj[3] = {wh[0][jj], wh[1][jj], wh[2][jj]};
            const float bhj[3] = {bh[0][jj], bh[1][jj], bh[2][jj]};
            const float gj[3] = {g[0][jj], g[1][jj], g[2][jj]};
            float vj[3];
            v_update_voxel_f32<DT, (MODE == X_SS || MODE == X_SSN) && DT == 2>(whj, bhj, gj, dv[jj], thf, ithf, epsf, vj);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                vn[c][jj] = vj[c];
                if (MODE != X_SSN) fc += fabsf(vj[c] - vp[c][jj]);
            }
            if (a.sp.log_objective) {
                const float rho = fmaf(gj[0], vj[0], fmaf(gj[1], vj[1], gj[2] * vj[2])) + dv[jj];
                fo += DT == 1 ? fabsf(rho) : 0.5f * rho * rho;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            constexpr bool SS = MODE == X_SS || MODE == X_SSN;
            if (MODE != X_FIRST && !SS && accel) stvN<VEC>(WP + (size_t)c * N + gi, w[c]);
            if (MODE != X_FIRST && !SS) stvN<VEC>(BO + (size_t)c * N + gi, bo[c]);  // b_k over b_{k-2}
            if (MODE != X_SSN || a.ss_last) stvN<VEC>(V + (size_t)c * N + gi, vn[c]);
            if constexpr (SS && sizeof(C) == 8 && VEC >= 2) {  // u = v: no b_hat to add
#pragma unroll
                for (int q = 0; q < VEC; q += 2) (buf + (c * TL + l) * PM)[(x0 + q) >> 1] = make_float2(vn[c][q], vn[c][q + 1]);
            } else
                st_reals_sum<VEC>(buf + (c * TL + l) * PM, x0, vn[c], bh[c]);
        }
    }
}

// phase 2 for the l1 data term: the same updates in fp64 with the reference's rounding
// points -- b = float(b_hat + v - w) (admm.cpp:142-153), w_hat / b_hat =
// float(a + c (a - a_prev)) (:130-139), the v-update from the unrounded warped and
// target values (v_update_voxel_exact) -- and fp64 change / residual / objective sums.
// The shrinkage's branch |zhat| <= 1 amplifies any rounding difference, so the l1 path
// spends the extra fp64 issue (it is not the bench path).
template <int MODE, int DT, int R2, int VEC, int UNR, class C, int NTP = kFT, int HINT = 0>
__device__ __forceinline__ void pointwise_tile_exact(const XArgs& a, C* buf, int pair, long long L0, int nl, int tid,
                                                     double& fc, double& fr, double& fo) {
    constexpr int L = kR1 * R2, PM = L + 1, M = 2 * L, TL = kFTL;
    const long long N = a.F.N;
    float* V = a.F.V + (size_t)pair * 3 * N;
    float* BO = a.F.BH + (size_t)pair * 3 * N;  // b_{k-2} in, b_k out (the dual iterates ping-pong)
    float* WP = a.F.WP + (size_t)pair * 3 * N;
    const float* BP = a.F.BP + (size_t)pair * 3 * N;  // b_{k-1}
    const float* G = a.F.G + (size_t)pair * 3 * N;
    const float* Wd = a.F.D + (size_t)pair * N;  // l1: D holds the warped image itself
    const float* Td = a.F.T + (size_t)pair * N;
    const double theta = a.sp.theta, eps = a.sp.epsilon, coef = a.coef, coefp = a.coef_prev;
    const bool accel = a.sp.accelerate != 0;
    const bool hp = a.coef_prev != 0.0;
    const size_t base = (size_t)L0 * M;
    const int nvox = nl * M;
#pragma unroll UNR
    for (int i0 = tid * VEC; i0 < nvox; i0 += NTP * VEC) {
        const int l = i0 / M, x0 = i0 - l * M;
        const size_t gi = base + i0;
        float w[3][VEC], vp[3][VEC], bo[3][VEC], wp[3][VEC], bp[3][VEC], g[3][VEC], wv[VEC], tv[VEC];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (MODE != X_FIRST) ldvN<VEC, HINT>(V + (size_t)c * N + gi, vp[c]);
            if (MODE == X_GENERAL) ldvN<VEC, HINT>(BP + (size_t)c * N + gi, bp[c]);        // b_{k-1}
            if (MODE == X_GENERAL && hp) ldvN<VEC, HINT>(BO + (size_t)c * N + gi, bo[c]);  // b_{k-2}
            if (MODE == X_GENERAL && accel) ldvN<VEC, HINT>(WP + (size_t)c * N + gi, wp[c]);
            if (MODE != X_TAIL) ldvN<VEC, HINT>(G + (size_t)c * N + gi, g[c]);
        }
        if (MODE != X_TAIL) {
            ldvN<VEC, HINT>(Wd + gi, wv);
            ldvN<VEC, HINT>(Td + gi, tv);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const C* wl = buf + (c * TL + l) * PM;
            if (MODE != X_FIRST) ld_reals<VEC>(wl, x0, w[c]);  // w = float(c2r), as stored by w_update_into
#pragma unroll
            for (int jj = 0; jj < VEC; ++jj) {
                if (MODE == X_FIRST) {
                    w[c][jj] = 0.f;
                    vp[c][jj] = 0.f;
                }
                // b_hat_{k-1} = float(b_{k-1} + c_{k-2} (b_{k-1} - b_{k-2})) (admm.cpp:130-139): the
                // reference's own expression on the stored fp32 iterates, so the same bits
                if (MODE != X_GENERAL) bo[c][jj] = 0.f;
                else if (hp) {
                    const double db1 = (double)bp[c][jj];
                    bo[c][jj] = (float)__dadd_rn(db1, __dmul_rn(coefp, __dsub_rn(db1, (double)bo[c][jj])));
                } else bo[c][jj] = bp[c][jj];
            }
        }
        if (MODE == X_TAIL) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int jj = 0; jj < VEC; ++jj) {
                    const double dd = (double)vp[c][jj] - (double)w[c][jj];
                    fr += dd * dd;
                }
            continue;
        }
        float wh[3][VEC], bh[3][VEC], vn[3][VEC];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int jj = 0; jj < VEC; ++jj) {
                if (MODE == X_FIRST) {
                    wh[c][jj] = 0.f;
                    bh[c][jj] = 0.f;
                    continue;
                }
                const double dv = (double)vp[c][jj], dw = (double)w[c][jj];
                const double dd = dv - dw;
                fr += dd * dd;
                const float b = (float)__dsub_rn(__dadd_rn((double)bo[c][jj], dv), dw);
                if (MODE == X_GENERAL && accel) {
                    wh[c][jj] = (float)__dadd_rn(dw, __dmul_rn(coef, __dsub_rn(dw, (double)wp[c][jj])));
                    const double db = (double)b;
                    bh[c][jj] = (float)__dadd_rn(db, __dmul_rn(coef, __dsub_rn(db, (double)bp[c][jj])));
                } else {
                    wh[c][jj] = w[c][jj];
                    bh[c][jj] = b;
                }
                bo[c][jj] = b;
            }
#pragma unroll
        for (int jj = 0; jj < VEC; ++jj) {
            const float whj[3] = {wh[0][jj], wh[1][jj], wh[2][jj]};
            const float bhj[3] = {bh[0][jj], bh[1][jj], bh[2][jj]};
            const float gj[3] = {g[0][jj], g[1][jj], g[2][jj]};
            float vj[3];
            v_update_voxel_exact<DT>(whj, bhj, gj, wv[jj], tv[jj], theta, eps, vj);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                vn[c][jj] = vj[c];
                fc += fabs((double)vj[c] - (double)vp[c][jj]);
            }
            if (a.sp.log_objective) {
                const double rho = data_residual_exact(gj, vj, wv[jj], tv[jj]);
                fo += DT == 1 ? fabs(rho) : 0.5 * rho * rho;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (MODE != X_FIRST && accel) stvN<VEC>(WP + (size_t)c * N + gi, w[c]);
            if (MODE != X_FIRST) stvN<VEC>(BO + (size_t)c * N + gi, bo[c]);  // b_k over b_{k-2}
            stvN<VEC>(V + (size_t)c * N + gi, vn[c]);
            st_reals_sum<VEC>(buf + (c * TL + l) * PM, x0, vn[c], bh[c]);  // u = v + b_hat (admm.cpp:77-80)
        }
    }
}

// phase 2 dispatch: fp32 (l2, the bench path) or the exact fp64 form (l1)
template <int MODE, int DT, int R2, int VEC, int UNR, class C, int NTP = kFT, int HINT = 0, class Acc>
__device__ __forceinline__ void pointwise_any(const XArgs& a, C* buf, int pair, long long L0, int nl, int tid, Acc& fc,
                                              Acc& fr, Acc& fo) {
    if constexpr (DT == 1 || sizeof(C) == 16)  // l1, or the precise (fp64 transform) mode
        pointwise_tile_exact<MODE, DT, R2, VEC, UNR, C, NTP, HINT>(a, buf, pair, L0, nl, tid, fc, fr, fo);
    else
        pointwise_tile<MODE, DT, R2, VEC, UNR, C, NTP, HINT>(a, buf, pair, L0, nl, tid, fc, fr, fo);
}

template <int DT, class C = float2>
using AccT = typename std::conditional<DT == 1 || sizeof(C) == 16, double, float>::type;

// phase 3: r2c of u (real, natural order in buf) -> spectrum rows in global.
template <int R2, class C, class Sync, int NF = kFT, bool STREAM = false>
__device__ __forceinline__ void r2c_tile(C* buf, const C* twx, const C* xtw, C* S, long long lines,
                                         long long L0, int nl, int tid, Sync sync) {
    constexpr int L = kR1 * R2, HX = L + 1, PM = L + 1, TL = kFTL;
    if (nl < TL) {
        for (int idx = tid; idx < 3 * TL * PM; idx += NF) {
            const int l = (idx / PM) & (TL - 1);
            if (l >= nl) buf[idx] = CT<C>::make(0, 0);
        }
    }
    sync();
    // (a) first DIF stage: radix 8 over stride R2, twiddle W_L^{j1 k}
    for (int t = tid; t < 3 * TL * R2; t += NF) {
        const int line = t % (3 * TL), j1 = t / (3 * TL);  // line fastest (conflict-free)
        C* Y = buf + line * PM;
        C x[kR1];
#pragma unroll
        for (int s = 0; s < kR1; ++s) x[s] = Y[j1 + R2 * s];
        dft8<false>(x);
#pragma unroll
        for (int k = 1; k < kR1; ++k) x[k] = cmul(x[k], twx[j1 * k]);
#pragma unroll
        for (int k = 0; k < kR1; ++k) Y[j1 + R2 * k] = x[k];
    }
    sync();
    // (b) last DIF stage on block pairs {j, 8-j} + r2c post-processing -> global
    constexpr int TASKS = 3 * (kR1 / 2) * TL;  // (c, j) outer, line fastest (coalesced stores)
    for (int t = tid; t < TASKS; t += NF) {
        const int l = t & (TL - 1);
        const int cj = t >> 5;
        const int c = cj >> 2, j = cj & 3;
        if (l >= nl) continue;
        const C* Y = buf + (c * TL + l) * PM;
        const int b0 = j, b1 = j == 0 ? kR1 / 2 : kR1 - j;
        C z0[R2], z1[R2];
#pragma unroll
        for (int e = 0; e < R2; ++e) {
            z0[e] = Y[R2 * b0 + e];
            z1[e] = Y[R2 * b1 + e];
        }
        rdft<false, R2>(z0);
        rdft<false, R2>(z1);
        C* Sc = S + (size_t)c * HX * lines + L0 + l;
        auto put = [&](int k, C out) {
            if constexpr (STREAM && sizeof(C) == 8) __stcs(Sc + (size_t)k * lines, out);  // read once, by the plane pass
            else Sc[(size_t)k * lines] = out;
        };
        auto emit = [&](int k, C zk, C zpartner) {
            const C zc = cconj(zpartner);
            const C ee = CT<C>::make((zk.x + zc.x) * 0.5f, (zk.y + zc.y) * 0.5f);
            const C oo = CT<C>::make((zk.y - zc.y) * 0.5f, -(zk.x - zc.x) * 0.5f);
            put(k, cadd(ee, cmul(xtw[k], oo)));
        };
        if constexpr (sizeof(C) == 8) {
            // fp32: X[k] and X[L-k] share s = Z[k] + conj(Z[L-k]), d = Z[k] - conj(Z[L-k]):
            // X[k] = s/2 + (t1, t2), X[L-k] = (s.x/2 - t1, t2 - s.y/2), (t1, t2) = W_M^k (d.y, -d.x) / 2
            auto joint = [&](int k, C a_, C b_) {
                const C w = xtw[k];
                const C s_ = CT<C>::make(a_.x + b_.x, a_.y - b_.y), d = CT<C>::make(a_.x - b_.x, a_.y + b_.y);
                const float hx_ = 0.5f * w.x, hy_ = 0.5f * w.y;
                const float t1 = fmaf(hx_, d.y, hy_ * d.x), t2 = fmaf(hy_, d.y, -(hx_ * d.x));
                const float sx = 0.5f * s_.x, sy = 0.5f * s_.y;
                put(k, CT<C>::make(sx + t1, sy + t2));
                put(L - k, CT<C>::make(sx - t1, t2 - sy));
            };
            if (j != 0) {
#pragma unroll
                for (int p1 = 0; p1 < R2; ++p1) joint(kR1 * p1 + b0, z0[p1], z1[R2 - 1 - p1]);
            } else {
                emit(0, z0[0], z0[0]);
                emit(L, z0[0], z0[0]);  // Nyquist bin k = L (Z[L] = Z[0])
                emit(kR1 * (R2 / 2), z0[R2 / 2], z0[R2 / 2]);
#pragma unroll
                for (int p1 = 1; p1 < R2 / 2; ++p1) joint(kR1 * p1, z0[p1], z0[R2 - p1]);
#pragma unroll
                for (int p1 = 0; p1 < R2 / 2; ++p1) joint(kR1 * p1 + kR1 / 2, z1[p1], z1[R2 - 1 - p1]);
            }
        } else {
#pragma unroll
            for (int p1 = 0; p1 < R2; ++p1) {
                if (j == 0) {
                    // block 0: partner of k = 8 p1 is L - k = 8 (R2 - p1) in block 0
                    emit(kR1 * p1, z0[p1], z0[(R2 - p1) & (R2 - 1)]);
                    // block 4 is self-paired: partner index R2 - 1 - p1
                    emit(kR1 * p1 + kR1 / 2, z1[p1], z1[R2 - 1 - p1]);
                } else {
                    emit(kR1 * p1 + b0, z0[p1], z1[R2 - 1 - p1]);
                    emit(kR1 * p1 + b1, z1[p1], z0[R2 - 1 - p1]);
                }
            }
            if (j == 0) emit(L, z0[0], z0[0]);  // Nyquist bin k = L (Z[L] = Z[0])
        }
    }
}

// Per-pair reduction of one tile's partials (slot = tile index within the pair) and
// the solve-level bookkeeping done by the pair's last tile.
template <int MODE, class Sync, int NTP = kFT>
__device__ __forceinline__ void finish_tile(const XArgs& a, int pair, unsigned slot, unsigned ntiles, double fc,
                                            double fr, double fo, double* red, int* s_last, int tid, Sync sync) {
    PairState* st = a.F.st + pair;
    const double vals[3] = {group_sum<NTP>(fc, red, tid, sync), group_sum<NTP>(fr, red, tid, sync),
                            group_sum<NTP>(fo, red, tid, sync)};
    double tot[3];
    if (group_reduce_partials<NTP, 3>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, ntiles, tot,
                                      red, s_last, tid, sync, slot) &&
        tid == 0) {
        const long long N = a.F.N;
        double* dg = a.F.diag ? a.F.diag + (size_t)pair * a.F.diag_stride * 3 : nullptr;
        if (MODE == X_TAIL) {
            const int it = st->iterations;
            if (dg && it >= 1) dg[(it - 1) * 3 + 1] = sqrt(tot[1]);
        } else {
            const double change = tot[0] / (3.0 * (double)N);
            if (dg) {
                dg[a.k * 3 + 0] = change;
                if (a.k >= 1) dg[(a.k - 1) * 3 + 1] = sqrt(tot[1]);
                dg[a.k * 3 + 2] = tot[2];
            }
            st->iterations = a.k + 1;
            st->final_change = change;
            if (change <= a.sp.tol) {
                st->done_iter = a.k;
                __threadfence();
                st->solve_done = 1;
            }
        }
    }
}

template <int MODE, int DT, int R2, int VEC = 2, int UNR = 2, class C = float2, int MINB = 3>
__global__ void __launch_bounds__(kFT, (sizeof(C) == 8) ? MINB : 2) xpass_fast_kernel(XArgs a) {
    constexpr int L = kR1 * R2;
    constexpr int HX = L + 1;
    constexpr int PM = L + 1;  // odd line pitch (complex)
    constexpr int TL = kFTL;
    const int pair = blockIdx.y;
    PairState* st = a.F.st + pair;
    if (!st->active || st->status) return;
    if ((MODE <= X_GENERAL || MODE == X_SS || MODE == X_SSN) && st->solve_done) return;

    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool F64 = sizeof(C) == 16;
    C* buf = reinterpret_cast<C*>(smem);                  // [3][TL][PM]
    C* twx = buf + 3 * TL * PM;                           // W_L^e
    C* xtw = twx + L;                                     // W_M^k, k in [0, HX]
    double* red = reinterpret_cast<double*>(xtw + HX + 1);
    __shared__ int s_last;
    const C* twx_g;
    const C* xtw_g;
    if constexpr (F64) {
        twx_g = a.twx64;
        xtw_g = a.xtw64;
    } else {
        twx_g = a.twx;
        xtw_g = a.xtw;
    }
    const int tid = threadIdx.x;
    const long long lines = a.F.lines;
    const long long L0 = (long long)blockIdx.x * TL;
    const int nl = (int)min((long long)TL, lines - L0);
    const BlockSync sync{};

    if (MODE != X_FIRST) stage_spectrum<R2>(buf, spectrum_of<C>(a.F, pair), lines, L0, nl, tid);
    for (int i = tid; i < L; i += kFT) twx[i] = twx_g[i];
    for (int i = tid; i <= HX; i += kFT) xtw[i] = xtw_g[i];
    if (!F64 && MODE != X_FIRST) cp_async_wait_all();
    __syncthreads();
    if (MODE != X_FIRST) c2r_tile<R2>(buf, twx, xtw, tid, sync);
    AccT<DT, C> fc = 0, fr = 0, fo = 0;
    pointwise_any<MODE, DT, R2, VEC, UNR>(a, buf, pair, L0, nl, tid, fc, fr, fo);
    if (MODE != X_TAIL)
        r2c_tile<R2>(buf, twx, xtw, spectrum_of<C>(a.F, pair), lines, L0, nl, tid, sync);
    if (MODE == X_SSN) {  // no norms: only the iteration count
        if (blockIdx.x == 0 && tid == 0) st->iterations = a.k + 1;
        return;
    }
    finish_tile<MODE>(a, pair, blockIdx.x, gridDim.x, fc, fr, fo, red, &s_last, tid, sync);
}

// ---- warp-specialised persistent x-pass (X_GENERAL, fp32) ----------------------------
// Threads [0, kFT) are the FFT group: c2r of tile i in ring buffer i % NB, then the
// cp.async prefetch of tile i+1's spectrum, then the r2c of tile i-1.  The remaining
// NPW warps are the point-wise group: the ADMM update of tile i, streaming the
// 112 B/voxel of field state.  Hand-off through named barriers:
//   W_READY(b): FFT arrives after c2r into buffer b; point-wise syncs before reading w.
//   U_READY(b): point-wise arrives after writing u; FFT syncs before the r2c.
// NB = 3: tile i+1 is staged while tile i is updated and tile i-1 transformed back, so
// the x-FFT work and the spectrum latency overlap the HBM stream instead of
// serialising with it (the one-tile kernel's critical path).  Each CTA owns a
// contiguous range of (pair, tile) tiles; the change / residual / data-term partials of
// a run of consecutive tiles of one pair are reduced once per run (fp64 per-thread sums,
// fixed tree) and the pair's ticket counts tiles, so the per-pair totals are
// deterministic for a given SM count.
// Named barriers: 1 = FFT (c2r) group, 2 = point-wise group, then NB ids each for W and U, one for
// the r2c group of the split form and NB for FREE -- 4 + 3 NB <= 16 ids, so the ring holds at most 4 tiles.
constexpr int kBarFFT = 1, kBarPW = 2, kBarW = 3;
template <int NB> struct RingBars {
    static constexpr int U = kBarW + NB, FFTB = kBarW + 2 * NB, F = kBarW + 2 * NB + 1;
    static_assert(F + NB <= 16, "named barrier ids");
};

// named barrier base + b with a compile-time id (a run-time id makes ptxas reserve all 16)
template <int BASE, int N, bool ARRIVE>
__device__ __forceinline__ void ring_bar(int b) {
#define DREG_RB(ID)                                                                  \
    if (ARRIVE) asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory"); \
    else asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
    switch (b) {
        case 0: DREG_RB(BASE + 0) break;
        case 1: DREG_RB(BASE + 1) break;
        case 2: DREG_RB(BASE + 2) break;
        default: DREG_RB(BASE + 3) break;
    }
#undef DREG_RB
}

// NB = 2 (two tile buffers, MINB = 2 CTAs per SM): the next tile is staged only after the
// previous one is transformed back, and the co-resident CTA covers that latency.
// SPLIT: the FFT warps form two groups, one staging + inverse-transforming tile i + 1 while the
// other forward-transforms tile i - 1 (and the point-wise group updates tile i), so the three
// stages of the ring run concurrently instead of the FFT group alternating between two of them;
// FREE(b) (r2c group arrives, c2r group waits) returns a buffer for restaging.
template <int DT, int R2, int NB, int NPW, int VEC, int UNR, int FW = 8, int HINT = 0, int MODE = X_GENERAL, int MINB = 1,
          bool SPLIT = false>
__global__ void __launch_bounds__(32 * (FW + NPW), MINB) xpass_pipe_kernel(XArgs a, int tiles_per_pair, int npairs) {
    constexpr int L = kR1 * R2, HX = L + 1, PM = L + 1, TL = kFTL;
    constexpr int BUF = 3 * TL * PM;
    constexpr int NF = 32 * FW, NTP = 32 * NPW, NALL = NF + NTP;
    static_assert(NB == 3 || NB == 2 || (NB == 4 && SPLIT), "ring of three tile buffers (two: unsplit; four: split form)");
    constexpr int kBarU = RingBars<NB>::U, kBarFFTB = RingBars<NB>::FFTB, kBarF = RingBars<NB>::F;
    extern __shared__ __align__(16) unsigned char smem[];
    float2* ring = reinterpret_cast<float2*>(smem);  // [NB][3][TL][PM]
    float2* twx = ring + NB * BUF;
    float2* xtw = twx + L;
    double* red = reinterpret_cast<double*>(xtw + HX + 1);  // [3][NPW]
    static_assert(3 * NPW <= 64, "red[] size");
    int* plist = reinterpret_cast<int*>(red + 64);  // [npairs] schedulable pairs, ascending
    __shared__ int tile_of[NB];
    __shared__ int s_np;
    // Only the pairs still iterating are spread over the grid (pairs stop at different
    // warps; a static split over all pairs would leave the CTAs of finished pairs idle
    // while the rest do full work).  The predicate uses flags that cannot change during
    // this launch: a solve_done raised by this launch carries done_iter == k (written
    // first, fenced), so every CTA derives the same list.
    if (threadIdx.x < 32) {
        int n = 0;
        for (int p0 = 0; p0 < npairs; p0 += 32) {
            const int p = p0 + (int)threadIdx.x;
            bool ok = false;
            if (p < npairs) {
                const volatile PairState* st = a.F.st + p;
                ok = a.pipe_all || (st->active && !st->status);  // pipe_all: A/B knob, static split
                if (ok && !a.pipe_all && st->solve_done) {
                    __threadfence();
                    ok = st->done_iter >= a.k;
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (ok) plist[n + __popc(m & ((1u << threadIdx.x) - 1u))] = p;
            n += __popc(m);
        }
        if (threadIdx.x == 0) s_np = n;
    }
    __syncthreads();
    const long long lines = a.F.lines;
    const int T = tiles_per_pair;
    const int total = T * s_np;  // tiles in schedulable-slot order: slot-major
    const int G = gridDim.x;
    // contiguous tile range of this CTA
    auto range_start = [&](int cta) { return (int)(((long long)cta * total) / G); };
    const int g_end = range_start(blockIdx.x + 1);
    const bool fft_group = threadIdx.x < NF;
    const int tid = fft_group ? (int)threadIdx.x : (int)threadIdx.x - NF;
    auto runnable_from = [&](int g) {  // pair flags are stable while any of its tiles is pending
        while (g < g_end) {
            const int slot = g / T;
            const PairState* st = a.F.st + plist[slot];
            if (st->active && !st->status && !st->solve_done) return g;
            g = (slot + 1) * T;
        }
        return -1;
    };
    auto stage = [&](int g, float2* buf) {
        const int pair = plist[g / T], tile = g - (g / T) * T;
        const long long L0 = (long long)tile * TL;
        const int nl = (int)min((long long)TL, lines - L0);
        stage_spectrum<R2, float2, NF>(buf, a.F.S + (size_t)pair * 3 * HX * lines, lines, L0, nl, tid);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    if (SPLIT && fft_group) {
        static_assert(!SPLIT || ((NB == 3 || NB == 4) && FW % 2 == 0), "split FFT groups: ring of three or four, even warp count");
        constexpr int NA = NF / 2;  // threads per FFT sub-group
        // W: c2r group arrives, point-wise waits; U: point-wise arrives, r2c group waits
        if (tid < NA) {
            const NamedSync<kBarFFT, NA> sync{};
            for (int i = tid; i < L; i += NA) twx[i] = a.twx[i];
            for (int i = tid; i <= HX; i += NA) xtw[i] = a.xtw[i];
            auto stage_a = [&](int g, float2* buf) {
                const int pair = plist[g / T], tile = g - (g / T) * T;
                const long long L0 = (long long)tile * TL;
                const int nl = (int)min((long long)TL, lines - L0);
                if (!DREG_SKIP(a, 4)) stage_spectrum<R2, float2, NA>(buf, a.F.S + (size_t)pair * 3 * HX * lines, lines, L0, nl, tid);
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            int cur = runnable_from(range_start(blockIdx.x));
            if (cur >= 0) stage_a(cur, ring);
            for (int i = 0;; ++i) {
                const int b = i % NB;
                const int next = cur >= 0 ? runnable_from(cur + 1) : -1;
                if (cur >= 0) {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                    sync();
                    if (!DREG_SKIP(a, 1)) c2r_tile<R2, float2, NamedSync<kBarFFT, NA>, NA>(ring + b * BUF, twx, xtw, tid, sync);
                }
                if (tid == 0) tile_of[b] = cur;
                ring_bar<kBarW, NA + NTP, true>(b);
                if (cur < 0) break;
                // slot i + 1 (the next tile, or the end marker) reuses the buffer, tile_of[] entry and
                // W barrier of tile i - 2: wait until the r2c group (hence the point-wise group) is done with it
                const int nb = (i + 1) % NB;
                if (i + 1 >= NB) ring_bar<kBarF, NF, false>(nb);
                if (next >= 0) stage_a(next, ring + nb * BUF);
                cur = next;
            }
        } else {
            const int tb = tid - NA;
            const NamedSync<kBarFFTB, NA> sync{};
            int n_tiles = 0;
            for (int g = runnable_from(range_start(blockIdx.x)); g >= 0; g = runnable_from(g + 1)) ++n_tiles;
            // this group trails the point-wise group, whose tickets may raise solve_done for a
            // pair it has finished: the tile ids come from tile_of[], not from the pair flags
            for (int i = 0; i < n_tiles; ++i) {
                const int b = i % NB;
                ring_bar<kBarU, NA + NTP, false>(b);
                const int cur = tile_of[b];
                const int pair = plist[cur / T], tile = cur - (cur / T) * T;
                const long long L0 = (long long)tile * TL;
                const int nl = (int)min((long long)TL, lines - L0);
                // the last spectral-state iteration's v is the solve's result: nothing reads its spectrum
                if (!((MODE == X_SS || MODE == X_SSN) && a.ss_last) && !DREG_SKIP(a, 1))
                    r2c_tile<R2, float2, NamedSync<kBarFFTB, NA>, NA, HINT == 2>(
                        ring + b * BUF, twx, xtw, a.F.S + (size_t)pair * 3 * HX * lines, lines, L0, nl, tb, sync);
                if (i + NB <= n_tiles) ring_bar<kBarF, NF, true>(b);  // slot i + NB (a tile or the end marker) reuses b
            }
        }
    } else if (fft_group) {
        const NamedSync<kBarFFT, NF> sync{};
        for (int i = tid; i < L; i += NF) twx[i] = a.twx[i];
        for (int i = tid; i <= HX; i += NF) xtw[i] = a.xtw[i];
        int cur = runnable_from(range_start(blockIdx.x));
        if (cur >= 0) stage(cur, ring);
        int prev = -1;
        for (int i = 0;; ++i) {
            const int b = i % NB;
            float2* buf = ring + b * BUF;
            const int next = cur >= 0 ? runnable_from(cur + 1) : -1;
            if (cur >= 0) {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
                sync();  // staged spectrum (and, first round, the tables) visible to the group
                if (!DREG_SKIP(a, 1)) c2r_tile<R2, float2, NamedSync<kBarFFT, NF>, NF>(buf, twx, xtw, tid, sync);
            }
            if (tid == 0) tile_of[b] = cur;
            ring_bar<kBarW, NALL, true>(b);
            // prefetch tile i+1 into buffer (i+1) % NB: it held tile i-2, transformed back last round
            if (NB == 3 && next >= 0) stage(next, ring + ((i + 1) % NB) * BUF);
            if (prev >= 0) {
                const int pb = (i + NB - 1) % NB;
                ring_bar<kBarU, NALL, false>(pb);
                const int pair = plist[prev / T], tile = prev - (prev / T) * T;
                const long long L0 = (long long)tile * TL;
                const int nl = (int)min((long long)TL, lines - L0);
                if (!DREG_SKIP(a, 1) && !((MODE == X_SS || MODE == X_SSN) && a.ss_last))
                    r2c_tile<R2, float2, NamedSync<kBarFFT, NF>, NF>(ring + pb * BUF, twx, xtw, a.F.S + (size_t)pair * 3 * HX * lines, lines, L0, nl,
                                 tid, sync);
                sync();  // buffer pb is restaged next round by this group
            }
            if (NB == 2 && next >= 0) stage(next, ring + ((i + 1) % NB) * BUF);  // the buffer just transformed back
            if (cur < 0) break;
            prev = cur;
            cur = next;
        }
    } else {
        const NamedSync<kBarPW, NTP> sync{};
        // per-thread fp64 sums over the tiles of the current run (consecutive tiles of one pair)
        double acc[3] = {0.0, 0.0, 0.0};
        int run_start = -1;
        for (int i = 0;; ++i) {
            const int b = i % NB;
            ring_bar<kBarW, SPLIT ? NF / 2 + NTP : NALL, false>(b);
            const int cur = tile_of[b];
            if (cur < 0) break;
            const int slot = cur / T, pair = plist[slot], tile = cur - slot * T;
            const long long L0 = (long long)tile * TL;
            const int nl = (int)min((long long)TL, lines - L0);
            AccT<DT> fc = 0, fr = 0, fo = 0;
            if (!DREG_SKIP(a, 2))
                pointwise_any<MODE, DT, R2, VEC, UNR, float2, NTP, HINT>(a, ring + b * BUF, pair, L0, nl, tid, fc,
                                                                         fr, fo);
            ring_bar<kBarU, SPLIT ? NF / 2 + NTP : NALL, true>(b);
            if (MODE == X_SSN) {  // no norms to reduce: only the iteration count is kept
                if (tile == 0 && tid == 0) a.F.st[pair].iterations = a.k + 1;
                continue;
            }
            if (run_start < 0) run_start = tile;
            acc[0] += (double)fc;
            acc[1] += (double)fr;
            acc[2] += (double)fo;
            // the run ends at the pair's last tile or the end of this CTA's range
            if (tile != T - 1 && cur + 1 != g_end) continue;
            if (DREG_SKIP(a, 8)) {
                acc[0] = acc[1] = acc[2] = 0.0;
                run_start = -1;
                continue;
            }
            // group sums (fixed tree), then the pair-level ticket weighted by the run length
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], o);
            sync();  // red[] free (previous run's readers done)
            if ((tid & 31) == 0)
#pragma unroll
                for (int k = 0; k < 3; ++k) red[k * NPW + (tid >> 5)] = acc[k];
            sync();
            PairState* st = a.F.st + pair;
            if (tid == 0) {
                double* part = a.F.part + (size_t)pair * 3 * kMaxPartials;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    double v = 0.0;
                    for (int w = 0; w < NPW; ++w) v += red[k * NPW + w];
                    part[(size_t)k * kMaxPartials + run_start] = v;
                }
                const unsigned run_len = (unsigned)(tile + 1 - run_start);
                __threadfence();
                const unsigned t = atomicAdd(&st->counter, run_len);
                if (t + run_len == (unsigned)T) {
                    __threadfence();
                    // runs of this pair, in CTA order: deterministic sum
                    double tot[3] = {0.0, 0.0, 0.0};
                    const int p0 = slot * T;
                    for (int c = 0; c < G; ++c) {
                        const int s0 = max(range_start(c), p0), s1 = min(range_start(c + 1), p0 + T);
                        if (s0 >= s1) continue;
#pragma unroll
                        for (int k = 0; k < 3; ++k) tot[k] += __ldcg(part + (size_t)k * kMaxPartials + (s0 - p0));
                    }
                    st->counter = 0u;
                    const long long N = a.F.N;
                    double* dg = a.F.diag ? a.F.diag + (size_t)pair * a.F.diag_stride * 3 : nullptr;
                    const double change = tot[0] / (3.0 * (double)N);
                    if (dg) {
                        dg[a.k * 3 + 0] = change;
                        if (a.k >= 1) dg[(a.k - 1) * 3 + 1] = sqrt(tot[1]);
                        dg[a.k * 3 + 2] = tot[2];
                    }
                    st->iterations = a.k + 1;
                    st->final_change = change;
                    if (change <= a.sp.tol) {
                        st->done_iter = a.k;  // before the flag: see the schedulable-pair scan
                        __threadfence();
                        st->solve_done = 1;
                    }
                }
            }
            acc[0] = acc[1] = acc[2] = 0.0;
            run_start = -1;
        }
    }
}

template <int R2, class C = float2>
static size_t fast_smem() {
    constexpr int L = kR1 * R2;
    return sizeof(C) * (3 * kFTL * (L + 1) + L + L + 2) + sizeof(double) * 32;
}

bool xpass_fast_eligible(const XArgs& a) {
    if (!a.fast_x || a.odd || a.f64) return false;
    const int M = a.F.M;
    return M == 64 || M == 128 || M == 256;
}

template <int MODE, int DT, int R2>
static cudaError_t launch_fast_x(const XArgs& a, int npairs, cudaStream_t s) {
    const dim3 grid((unsigned)((a.F.lines + kFTL - 1) / kFTL), (unsigned)npairs);
    const size_t smem = a.precise ? fast_smem<R2, double2>() : fast_smem<R2>();
    void (*k)(XArgs) = xpass_fast_kernel<MODE, DT, R2>;
    if (a.precise) k = xpass_fast_kernel<MODE, DT, R2, 2, 2, double2>;
    else switch (a.fx_variant) {
        case 41: k = xpass_fast_kernel<MODE, DT, R2, 4, 1>; break;
        case 21: k = xpass_fast_kernel<MODE, DT, R2, 2, 1>; break;
        case 24: k = xpass_fast_kernel<MODE, DT, R2, 2, 4>; break;
        case 11: k = xpass_fast_kernel<MODE, DT, R2, 1, 1>; break;
        case 14: k = xpass_fast_kernel<MODE, DT, R2, 1, 4>; break;
        case 224: k = xpass_fast_kernel<MODE, DT, R2, 2, 2, float2, 4>; break;
        case 214: k = xpass_fast_kernel<MODE, DT, R2, 2, 1, float2, 4>; break;
        default: break;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k<<<grid, kFT, smem, s>>>(a);
    return cudaGetLastError();
}

template <int DT, int R2, int NPW, int VEC, int UNR, int FW = 8, int HINT = 0, int MODE = X_GENERAL, int NB = 3, int MINB = 1,
          bool SPLIT = false>
static cudaError_t launch_pipe_t(const XArgs& a, int npairs, cudaStream_t s) {
    constexpr int L = kR1 * R2;
    const size_t smem = sizeof(float2) * ((size_t)NB * 3 * kFTL * (L + 1) + L + L + 2) + sizeof(double) * 64 +
                        sizeof(int) * (size_t)npairs;
    void (*k)(XArgs, int, int) = xpass_pipe_kernel<DT, R2, NB, NPW, VEC, UNR, FW, HINT, MODE, MINB, SPLIT>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = (int)((a.F.lines + kFTL - 1) / kFTL);
    // DREG_XPASS_SMS (experiment knob): persistent CTAs, i.e. SMs the x-pass occupies
    const char* lim = std::getenv("DREG_XPASS_SMS");
    if (lim && std::atoi(lim) > 0) sms = std::min(sms, std::atoi(lim));
    const int grid = std::min(tiles * npairs, sms * MINB);
    k<<<grid, 32 * (FW + NPW), smem, s>>>(a, tiles, npairs);
    return cudaGetLastError();
}

template <int DT, int R2>
static cudaError_t launch_pipe_r(const XArgs& a, int npairs, cudaStream_t s) {
    switch (a.pipe) {  // FFT warps * 10000 + point-wise warps * 100 + VEC * 10 + unroll
        case 80841: return launch_pipe_t<DT, R2, 8, 4, 1, 8>(a, npairs, s);
        case 41221: return launch_pipe_t<DT, R2, 12, 2, 1, 4>(a, npairs, s);
        case 40842: return launch_pipe_t<DT, R2, 8, 4, 2, 4>(a, npairs, s);
        default: return launch_pipe_t<DT, R2, 8, 4, 1, 4>(a, npairs, s);  // 40841: measured best at M = 128
    }
}

template <int MODE, int R2, int VEC, int UNR, int MINB>
static cudaError_t launch_fast_ss(const XArgs& a, int npairs, cudaStream_t s) {
    const dim3 grid((unsigned)((a.F.lines + kFTL - 1) / kFTL), (unsigned)npairs);
    const size_t smem = fast_smem<R2>();
    void (*k)(XArgs) = xpass_fast_kernel<MODE, 2, R2, VEC, UNR, float2, MINB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k<<<grid, kFT, smem, s>>>(a);
    return cudaGetLastError();
}

// spectral-state x-pass (l2 only): the point-wise group streams 40 B/voxel instead of 100,
// so the warp split is tuned separately (DREG_PIPE_SS: FFT warps * 10000 + point-wise
// warps * 100 + VEC * 10 + unroll)
template <int R2, int MODE>
static cudaError_t launch_pipe_ss(const XArgs& a, int npairs, cudaStream_t s) {
    switch (a.pipe_ss) {  // the measured alternatives (profiles/r2c_ss_sweep.md); the rest of the sweep was dropped
        case 3: return launch_fast_ss<MODE, R2, 2, 2, 3>(a, npairs, s);  // one tile per CTA, 3 CTAs per SM
        case 80841: return launch_pipe_t<2, R2, 8, 4, 1, 8, 0, MODE>(a, npairs, s);   // 8 FFT + 8 point-wise warps
        case 120442: return launch_pipe_t<2, R2, 4, 4, 2, 12, 0, MODE>(a, npairs, s);  // 12 FFT + 4 point-wise, unsplit
        case 2060242: return launch_pipe_t<2, R2, 2, 4, 2, 6, 0, MODE, 2, 2>(a, npairs, s);  // two CTAs per SM, two buffers each
        case 1120841: return launch_pipe_t<2, R2, 8, 4, 1, 12, 0, MODE, 3, 1, true>(a, npairs, s);  // split, 8 point-wise warps
        case 41120841: return launch_pipe_t<2, R2, 8, 4, 1, 12, 0, MODE, 4, 1, true>(a, npairs, s);  // ring of four tiles
        case 1240841: return launch_pipe_t<2, R2, 8, 4, 1, 24, 0, MODE, 3, 1, true>(a, npairs, s);  // 12 + 12 FFT, 8 point-wise
        // 12 FFT warps cover a tile's 96 lines x 4 block pairs / 384 r2c tasks in one round each, split
        // into a c2r group and an r2c group (6 + 6); 4 point-wise warps with four iterations of grad /
        // diff loads in flight (the loop is unrolled 4x over __restrict__ pointers): 1120444
        default: return launch_pipe_t<2, R2, 4, 4, 4, 12, 0, MODE, 3, 1, true>(a, npairs, s);
    }
}

template <int MODE, int DT>
static cudaError_t launch_fast_r(const XArgs& a, int npairs, cudaStream_t s) {
    switch (a.F.M) {
        case 64: return launch_fast_x<MODE, DT, 4>(a, npairs, s);
        case 128: return launch_fast_x<MODE, DT, 8>(a, npairs, s);
        default: return launch_fast_x<MODE, DT, 16>(a, npairs, s);
    }
}

bool xpass_ss_eligible(const XArgs& a) {
    return xpass_fast_eligible(a) && a.pipe && !a.precise && a.sp.data_term == 2 && (a.F.M == 64 || a.F.M == 128);
}

cudaError_t launch_xpass_fast(const XArgs& a, int mode, int npairs, cudaStream_t s) {
    const bool l1 = a.sp.data_term == 1;
    if (mode == X_SS || mode == X_SSN) {
        if (!xpass_ss_eligible(a)) return cudaErrorInvalidConfiguration;
        if (a.F.M == 128) return mode == X_SS ? launch_pipe_ss<8, X_SS>(a, npairs, s) : launch_pipe_ss<8, X_SSN>(a, npairs, s);
        return mode == X_SS ? launch_pipe_ss<4, X_SS>(a, npairs, s) : launch_pipe_ss<4, X_SSN>(a, npairs, s);
    }
    if (mode == X_GENERAL && a.pipe && !a.precise && a.F.M == 128)
        return l1 ? launch_pipe_r<1, 8>(a, npairs, s) : launch_pipe_r<2, 8>(a, npairs, s);
    if (mode == X_GENERAL && a.pipe && !a.precise && a.F.M == 64)
        return l1 ? launch_pipe_r<1, 4>(a, npairs, s) : launch_pipe_r<2, 4>(a, npairs, s);
    // M = 256 (config 5): a tile is 99 KB, so the ring has two buffers; the point-wise group's
    // 100 B/voxel stream is the long stage and covers the later restaging (DREG_PIPE256=0: one tile per CTA)
    if (mode == X_GENERAL && a.pipe && a.pipe256 && !a.precise && a.F.M == 256 && !l1)
        return a.pipe256 == 2 ? launch_pipe_t<2, 16, 8, 4, 2, 4, 0, X_GENERAL, 2, 1>(a, npairs, s)  // two iterations of loads in flight
                              : launch_pipe_t<2, 16, 8, 4, 1, 4, 0, X_GENERAL, 2, 1>(a, npairs, s);
    switch (mode) {
        case X_FIRST: return l1 ? launch_fast_r<X_FIRST, 1>(a, npairs, s) : launch_fast_r<X_FIRST, 2>(a, npairs, s);
        case X_SECOND: return l1 ? launch_fast_r<X_SECOND, 1>(a, npairs, s) : launch_fast_r<X_SECOND, 2>(a, npairs, s);
        case X_GENERAL: return l1 ? launch_fast_r<X_GENERAL, 1>(a, npairs, s) : launch_fast_r<X_GENERAL, 2>(a, npairs, s);
        default: return l1 ? launch_fast_r<X_TAIL, 1>(a, npairs, s) : launch_fast_r<X_TAIL, 2>(a, npairs, s);
    }
}

}  // namespace dregb
