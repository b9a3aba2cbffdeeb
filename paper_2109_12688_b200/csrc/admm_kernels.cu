// Accelerated-ADMM inner loop kernels (reference admm.cpp:252-314).
//
// One ADMM iteration k is two launches:
//   xpass(k)  -- per tile of x-lines: c2r of the filtered spectrum -> w_{k-1};
//                dual update b_{k-1} (admm.cpp:142-153); constraint residual
//                (:163-170); Nesterov extrapolation of w and b (:130-139, :294-297);
//                closed-form v-update (:23-63); change norm (:155-161);
//                u_k = v_k + b_hat_k; r2c along x -> spectrum (plane-major).
//   plane(k)  -- per (component, x-frequency) plane: y/z DIF FFT, multiply by
//                theta / (lambda K_n + theta) / N (:83-95, regularizer.cpp:51-79),
//                y/z inverse.
// so the spectrum makes exactly one HBM round trip between launches and every
// real-space field is touched once per iteration.
#include "fft_device.cuh"
#include "kernels.cuh"
#include "launch.h"
#include "pointwise.cuh"
#include "plane_fast.cuh"

namespace dregb {

constexpr int kXThreads = 256;
constexpr int kPThreads = 512;

// C = float2 (fp32 x-FFT) or double2 (precise mode: fp64 butterflies and twiddles)
template <class C>
struct XSmem {
    C* twx;
    C* xtw;
    int* xpos;
    C* buf;
    C* Xs;
    double* red;
};

template <class C>
__device__ __forceinline__ XSmem<C> carve_x(unsigned char* smem, int L, int hx, int TL, int PM) {
    XSmem<C> s;
    size_t off = 0;
    s.twx = reinterpret_cast<C*>(smem + off);
    off += sizeof(C) * L;
    s.xtw = reinterpret_cast<C*>(smem + off);
    off += sizeof(C) * (hx + 1);
    s.buf = reinterpret_cast<C*>(smem + off);
    off += sizeof(C) * 3 * TL * PM;
    s.Xs = reinterpret_cast<C*>(smem + off);
    off += sizeof(C) * hx * TL;
    s.red = reinterpret_cast<double*>(smem + off);
    off += sizeof(double) * 32;
    s.xpos = reinterpret_cast<int*>(smem + off);
    return s;
}

size_t xpass_smem_bytes_c(int L, int hx, int TL, int PM, size_t csz) {
    return csz * (L + hx + 1 + 3 * (size_t)TL * PM + (size_t)hx * TL) + sizeof(double) * 32 + sizeof(int) * L;
}

size_t xpass_smem_bytes(int L, int hx, int TL, int PM) { return xpass_smem_bytes_c(L, hx, TL, PM, sizeof(float2)); }

template <int VEC>
__device__ __forceinline__ void ldv(const float* p, float* out) {
    if constexpr (VEC == 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        out[0] = t.x; out[1] = t.y; out[2] = t.z; out[3] = t.w;
    } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) out[j] = p[j];
    }
}
template <int VEC>
__device__ __forceinline__ void stv(float* p, const float* in) {
    if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
    } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) p[j] = in[j];
    }
}

template <int MODE, int DT, int VEC, bool F64 = false, int MINB = 3, class C = float2>
__global__ void __launch_bounds__(kXThreads, (VEC == 4 && F64) ? 2 : MINB) xpass_kernel(XArgs a) {
    using R = decltype(C::x);
    const int pair = blockIdx.y;
    PairState* st = a.F.st + pair;
    if (!st->active || st->status) return;
    constexpr bool UTIL = (MODE == X_FWD || MODE == X_INV);
    if (MODE <= X_GENERAL && st->solve_done) return;
    if (UTIL && st->solve_done && a.k > st->done_iter) return;

    extern __shared__ __align__(16) unsigned char smem[];
    const int L = a.px.n, M = a.F.M, hx = a.F.hx, TL = a.TL, PM = a.PM;
    XSmem<C> sm = carve_x<C>(smem, L, hx, TL, PM);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const long long lines = a.F.lines;
    const long long L0 = (long long)blockIdx.x * TL;
    const int nl = (int)min((long long)TL, lines - L0);
    const long long N = a.F.N;
    const int lt = 31 - __clz(TL);  // TL is a power of two
    const int tm = TL - 1;

    const C* twx_g;
    const C* xtw_g;
    if constexpr (sizeof(C) == 16) {
        twx_g = a.twx64;
        xtw_g = a.xtw64;
    } else {
        twx_g = a.twx;
        xtw_g = a.xtw;
    }
    for (int i = tid; i < L; i += nthr) {
        sm.twx[i] = twx_g[i];
        sm.xpos[i] = a.xpos[i];
    }
    for (int i = tid; i <= hx; i += nthr) sm.xtw[i] = xtw_g[i];
    __syncthreads();

    float* V = a.F.V + (size_t)pair * 3 * N;
    float* BH = a.F.BH + (size_t)pair * 3 * N;  // iterations: b_{k-2} in, b_k out (X_FWD: b_hat input)
    float* WP = a.F.WP + (size_t)pair * 3 * N;
    const float* BP = a.F.BP + (size_t)pair * 3 * N;  // b_{k-1}
    const float* G = a.F.G + (size_t)pair * 3 * N;
    const float* Dd = a.F.D + (size_t)pair * N;
    C* S = spectrum_of<C>(a.F, pair);  // fp32 storage, fp64 in precise mode

    if (a.prefetch && (MODE == X_GENERAL || MODE == X_SECOND)) {
        // Stream this tile's field rows into L2 while the spectrum loads and the
        // inverse x-FFT run (cp.async.bulk.prefetch: no registers, no smem).
        const unsigned bytes = (unsigned)(nl * M * sizeof(float));
        const size_t off = (size_t)L0 * M;
        if (tid < 16) {
            const float* base;
            const int f = tid / 3, c = tid - 3 * (tid / 3);
            if (tid == 15) base = Dd + off;
            else if (f == 0) base = V + (size_t)c * N + off;
            else if (f == 1) base = G + (size_t)c * N + off;
            else if (f == 2) base = (MODE == X_GENERAL ? BH : V) + (size_t)c * N + off;
            else if (f == 3) base = (MODE == X_GENERAL ? WP : V) + (size_t)c * N + off;
            else base = (MODE == X_GENERAL ? BP : V) + (size_t)c * N + off;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base), "r"(bytes) : "memory");
        }
    }

    // ---- phase 1: x c2r of the filtered spectrum -> w_{k-1} (real, in smem) ----
    if (MODE != X_FIRST && MODE != X_FWD) {
        for (int c = 0; c < 3; ++c) {
            const C* Sc = S + (size_t)c * hx * lines;
            for (int idx = tid; idx < hx * TL; idx += nthr) {
                const int p = idx >> lt, l = idx & tm;
                sm.Xs[idx] = l < nl && !DREG_SKIP(a, 4) ? Sc[(size_t)p * lines + L0 + l] : CT<C>::make(0, 0);
            }
            __syncthreads();
            C* bc = sm.buf + (size_t)c * TL * PM;
            if (!a.odd) {
                // Z'[k] = E + i O with E = X[k] + conj(X[L-k]), O = (X[k] - conj(X[L-k])) W_M^{-k};
                // imaginary parts of the self-conjugate bins ignored (1-D c2r semantics).
                for (int idx = tid; idx < L * TL; idx += nthr) {
                    const int k = idx >> lt, l = idx & tm;
                    C A = sm.Xs[k * TL + l];
                    C B = sm.Xs[(L - k) * TL + l];
                    if (k == 0) { A.y = 0.f; B.y = 0.f; }
                    B.y = -B.y;
                    const C e = cadd(A, B);
                    const C o = cmulc(csub(A, B), sm.xtw[k]);
                    bc[l * PM + sm.xpos[k]] = CT<C>::make(e.x - o.y, e.y + o.x);
                }
            } else {
                for (int idx = tid; idx < M * TL; idx += nthr) {
                    const int k = idx >> lt, l = idx & tm;
                    C X;
                    if (k < hx) {
                        X = sm.Xs[k * TL + l];
                        if (k == 0) X.y = 0.f;
                    } else {
                        X = cconj(sm.Xs[(M - k) * TL + l]);
                    }
                    bc[l * PM + sm.xpos[k]] = X;
                }
            }
            __syncthreads();
        }
        if (!DREG_SKIP(a, 1)) fft_lines<true>(sm.buf, 3 * TL, a.fd_lines, PM, 1, a.px, sm.twx, tid, nthr);
    }

    if constexpr (UTIL) {
        const size_t base = (size_t)L0 * M;
        const int nvox = nl * M;
        for (int i = tid; i < 3 * nvox; i += nthr) {
            const int c = i / nvox, r = i - c * nvox;
            const int l = r / M, x = r - l * M;
            C* bl = sm.buf + (size_t)(c * TL + l) * PM;
            const size_t gi = (size_t)c * N + base + r;
            if (MODE == X_FWD) {
                const R u = a.add_bh ? (R)V[gi] + (R)BH[gi] : (R)V[gi];  // admm.cpp:77-80
                if (!a.odd) reinterpret_cast<R*>(bl)[x] = u;
                else bl[x] = CT<C>::make(u, 0);
            } else {
                WP[gi] = (float)(!a.odd ? reinterpret_cast<const R*>(bl)[x] : bl[x].x);
            }
        }
        if (MODE == X_INV) return;
    }

    // ---- phase 2: point-wise ADMM updates on the tile ----
    const double theta = a.sp.theta, inv_theta = 1.0 / a.sp.theta, eps = a.sp.epsilon;
    const double coef = a.coef, coefp = a.coef_prev;
    const bool accel = a.sp.accelerate != 0;
    const bool hp = a.coef_prev != 0.0;  // b_hat_{k-1} differs from b_{k-1}
    double s_change = 0.0, s_res = 0.0, s_obj = 0.0;
    const size_t base = (size_t)L0 * M;
    const int nvox = nl * M;
    if constexpr (!F64) {
        // fp32 arithmetic, fp32 per-thread partial sums (a thread covers <= ~64 voxels)
        const float thf = (float)theta, ithf = (float)inv_theta, epsf = (float)eps, cf = (float)coef;
        const float cpf = (float)coefp;
        float fc = 0.f, fr = 0.f, fo = 0.f;
#pragma unroll 2
        for (int i0 = tid * VEC; i0 < (UTIL || DREG_SKIP(a, 2) ? 0 : nvox); i0 += nthr * VEC) {
            const int l = i0 / M, x0 = i0 - l * M;
            const size_t gi = base + i0;
            float w[3][VEC], vp[3][VEC], bo[3][VEC], wp[3][VEC], bp[3][VEC], g[3][VEC], dv[VEC];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (MODE != X_FIRST) ldv<VEC>(V + (size_t)c * N + gi, vp[c]);
                if (MODE == X_GENERAL) ldv<VEC>(BP + (size_t)c * N + gi, bp[c]);
                if (MODE == X_GENERAL && hp) ldv<VEC>(BH + (size_t)c * N + gi, bo[c]);
                if (MODE == X_GENERAL && accel) ldv<VEC>(WP + (size_t)c * N + gi, wp[c]);
                if (MODE != X_TAIL) ldv<VEC>(G + (size_t)c * N + gi, g[c]);
            }
            if (MODE != X_TAIL) ldv<VEC>(Dd + gi, dv);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const C* bl = sm.buf + (size_t)(c * TL + l) * PM;
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    w[c][j] = MODE == X_FIRST ? 0.f : (float)(!a.odd ? reinterpret_cast<const R*>(bl)[x0 + j] : bl[x0 + j].x);
                    if (MODE == X_FIRST) vp[c][j] = 0.f;
                    // b_hat_{k-1} re-formed from the stored dual iterates b_{k-1}, b_{k-2} (admm.cpp:130-139)
                    if (MODE != X_GENERAL) bo[c][j] = 0.f;
                    else bo[c][j] = hp ? fmaf(cpf, bp[c][j] - bo[c][j], bp[c][j]) : bp[c][j];
                }
            }
            if (MODE == X_TAIL) {
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int j = 0; j < VEC; ++j) {
                        const float dd = vp[c][j] - w[c][j];
                        fr = fmaf(dd, dd, fr);
                    }
                continue;
            }
            float wh[3][VEC], bh[3][VEC], vn[3][VEC];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    if (MODE == X_FIRST) {
                        wh[c][j] = 0.f;
                        bh[c][j] = 0.f;
                        continue;
                    }
                    const float dd = vp[c][j] - w[c][j];
                    fr = fmaf(dd, dd, fr);
                    const float b = bo[c][j] + dd;  // dual update (admm.cpp:142-153)
                    if (MODE == X_GENERAL && accel) {
                        wh[c][j] = fmaf(cf, w[c][j] - wp[c][j], w[c][j]);  // extrapolate (admm.cpp:130-139)
                        bh[c][j] = fmaf(cf, b - bp[c][j], b);
                    } else {
                        wh[c][j] = w[c][j];
                        bh[c][j] = b;
                    }
                    bo[c][j] = b;
                }
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const float whj[3] = {wh[0][j], wh[1][j], wh[2][j]};
                const float bhj[3] = {bh[0][j], bh[1][j], bh[2][j]};
                const float gj[3] = {g[0][j], g[1][j], g[2][j]};
                float vj[3];
                v_update_voxel_f32<DT>(whj, bhj, gj, dv[j], thf, ithf, epsf, vj);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    vn[c][j] = vj[c];
                    fc += fabsf(vj[c] - vp[c][j]);
                }
                if (a.sp.log_objective) {
                    const float rho = fmaf(gj[0], vj[0], fmaf(gj[1], vj[1], gj[2] * vj[2])) + dv[j];
                    fo += DT == 1 ? fabsf(rho) : 0.5f * rho * rho;
                }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (MODE != X_FIRST && accel) stv<VEC>(WP + (size_t)c * N + gi, w[c]);
                if (MODE != X_FIRST) stv<VEC>(BH + (size_t)c * N + gi, bo[c]);  // b_k over b_{k-2}
                stv<VEC>(V + (size_t)c * N + gi, vn[c]);
                C* bl = sm.buf + (size_t)(c * TL + l) * PM;
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    const R u = (R)vn[c][j] + (R)bh[c][j];
                    if (!a.odd) reinterpret_cast<R*>(bl)[x0 + j] = u;
                    else bl[x0 + j] = CT<C>::make(u, 0);
                }
            }
        }
        s_change = fc;
        s_res = fr;
        s_obj = fo;
    } else {
    for (int i0 = tid * VEC; i0 < (UTIL || DREG_SKIP(a, 2) ? 0 : nvox); i0 += nthr * VEC) {
        const int l = i0 / M, x0 = i0 - l * M;
        const size_t gi = base + i0;
        float w[3][VEC], vp[3][VEC];
        if (MODE != X_FIRST) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const C* bl = sm.buf + (size_t)(c * TL + l) * PM;
                if (!a.odd) {
                    const R* wl = reinterpret_cast<const R*>(bl);
#pragma unroll
                    for (int j = 0; j < VEC; ++j) w[c][j] = (float)wl[x0 + j];  // w stored as float (admm.cpp:97-99)
                } else {
#pragma unroll
                    for (int j = 0; j < VEC; ++j) w[c][j] = (float)bl[x0 + j].x;
                }
                ldv<VEC>(V + (size_t)c * N + gi, vp[c]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int j = 0; j < VEC; ++j) vp[c][j] = 0.f;
        }
        if (MODE == X_TAIL) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    const double dd = (double)vp[c][j] - (double)w[c][j];
                    s_res += dd * dd;
                }
            continue;
        }
        float wh[3][VEC], bh[3][VEC];
        if (MODE == X_FIRST) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int j = 0; j < VEC; ++j) { wh[c][j] = 0.f; bh[c][j] = 0.f; }
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float bo[VEC], bp[VEC];
                if (MODE == X_GENERAL) {
                    // b_hat_{k-1} = float(b_{k-1} + c_{k-2} (b_{k-1} - b_{k-2})) (admm.cpp:130-139),
                    // the reference's expression on the stored fp32 iterates: the same bits
                    ldv<VEC>(BP + (size_t)c * N + gi, bp);
                    if (hp) {
                        ldv<VEC>(BH + (size_t)c * N + gi, bo);
#pragma unroll
                        for (int j = 0; j < VEC; ++j) {
                            const double ab = bp[j];
                            bo[j] = (float)__dadd_rn(ab, __dmul_rn(coefp, __dsub_rn(ab, (double)bo[j])));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) bo[j] = bp[j];
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < VEC; ++j) bo[j] = 0.f;
                }
                float b[VEC];
#pragma unroll
                for (int j = 0; j < VEC; ++j) {
                    // dual_update: b = b_hat + v - w  (admm.cpp:142-153)
                    b[j] = (float)((double)bo[j] + (double)vp[c][j] - (double)w[c][j]);
                    const double dd = (double)vp[c][j] - (double)w[c][j];
                    s_res += dd * dd;
                }
                if (accel && MODE == X_GENERAL) {
                    float wp[VEC];
                    ldv<VEC>(WP + (size_t)c * N + gi, wp);
#pragma unroll
                    for (int j = 0; j < VEC; ++j) {  // av + scale * (av - b), unfused like the reference
                        const double aw = w[c][j], ab = b[j];
                        wh[c][j] = (float)__dadd_rn(aw, __dmul_rn(coef, __dsub_rn(aw, (double)wp[j])));
                        bh[c][j] = (float)__dadd_rn(ab, __dmul_rn(coef, __dsub_rn(ab, (double)bp[j])));
                    }
                } else {
                    // coefficient is exactly 0 (first step, or accelerate off)
#pragma unroll
                    for (int j = 0; j < VEC; ++j) { wh[c][j] = w[c][j]; bh[c][j] = b[j]; }
                }
                if (accel) stv<VEC>(WP + (size_t)c * N + gi, w[c]);
                stv<VEC>(BH + (size_t)c * N + gi, b);  // b_k over b_{k-2}
            }
        }
        float g[3][VEC], dv[VEC], tv[VEC];
#pragma unroll
        for (int c = 0; c < 3; ++c) ldv<VEC>(G + (size_t)c * N + gi, g[c]);
        ldv<VEC>(Dd + gi, dv);
        // l1 / precise: D holds the warped image, the residual is formed from both (exact form)
        constexpr bool EXACT = DT == 1 || sizeof(C) == 16;
        if (EXACT) ldv<VEC>(a.F.T + (size_t)pair * N + gi, tv);
        float vn[3][VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const float whj[3] = {wh[0][j], wh[1][j], wh[2][j]};
            const float bhj[3] = {bh[0][j], bh[1][j], bh[2][j]};
            const float gj[3] = {g[0][j], g[1][j], g[2][j]};
            float vj[3];
            if (EXACT) v_update_voxel_exact<DT>(whj, bhj, gj, dv[j], tv[j], theta, eps, vj);
            else v_update_voxel<DT>(whj, bhj, gj, (double)dv[j], theta, inv_theta, eps, vj);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                vn[c][j] = vj[c];
                s_change += fabs((double)vj[c] - (double)vp[c][j]);
            }
            if (a.sp.log_objective) {
                if (EXACT) {
                    const double rho = data_residual_exact(gj, vj, dv[j], tv[j]);
                    s_obj += DT == 1 ? fabs(rho) : 0.5 * rho * rho;
                } else {
                    const double rho = ((double)gj[0] * vj[0] + (double)gj[1] * vj[1] + (double)gj[2] * vj[2]) +
                                       (double)dv[j];
                    s_obj += 0.5 * rho * rho;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            stv<VEC>(V + (size_t)c * N + gi, vn[c]);
            C* bl = sm.buf + (size_t)(c * TL + l) * PM;
            if (!a.odd) {
                R* ul = reinterpret_cast<R*>(bl);
#pragma unroll
                for (int j = 0; j < VEC; ++j) ul[x0 + j] = (R)vn[c][j] + (R)bh[c][j];
            } else {
#pragma unroll
                for (int j = 0; j < VEC; ++j) bl[x0 + j] = CT<C>::make((R)vn[c][j] + (R)bh[c][j], 0);
            }
        }
    }

    }

    // ---- phase 3: r2c along x of u_k, scatter to the plane-major spectrum ----
    if (MODE != X_TAIL) {
        if (nl < TL) {  // zero the unused lines so the batched FFT stays finite
            for (int idx = tid; idx < 3 * TL * PM; idx += nthr) {
                const int l = (idx / PM) % TL;
                if (l >= nl) sm.buf[idx] = CT<C>::make(0, 0);
            }
        }
        __syncthreads();
        if (!DREG_SKIP(a, 1)) fft_lines<false>(sm.buf, 3 * TL, a.fd_lines, PM, 1, a.px, sm.twx, tid, nthr);
        for (int cidx = tid; cidx < 3 * hx * TL; cidx += nthr) {
            const int c = cidx >= 2 * hx * TL ? 2 : (cidx >= hx * TL ? 1 : 0);
            const int idx = cidx - c * hx * TL;
            const int k = idx >> lt, l = idx & tm;
            if (l >= nl) continue;
            const C* bl = sm.buf + (size_t)(c * TL + l) * PM;
            C X;
            if (!a.odd) {
                const C zk = bl[sm.xpos[k == L ? 0 : k]];
                const C zc = cconj(bl[sm.xpos[k == 0 ? 0 : L - k]]);
                const C e = CT<C>::make((R)0.5 * (zk.x + zc.x), (R)0.5 * (zk.y + zc.y));
                const C o = CT<C>::make((R)0.5 * (zk.y - zc.y), (R)-0.5 * (zk.x - zc.x));
                X = cadd(e, cmul(sm.xtw[k], o));
            } else {
                X = bl[sm.xpos[k]];
            }
            if (!DREG_SKIP(a, 4)) S[((size_t)c * hx + k) * lines + L0 + l] = X;
        }
    }

    if constexpr (UTIL) return;

    // ---- deterministic reductions + per-iteration bookkeeping ----
    const double tc = block_sum<kXThreads>(s_change, sm.red);
    const double tr = block_sum<kXThreads>(s_res, sm.red);
    const double to = block_sum<kXThreads>(s_obj, sm.red);
    const double vals[3] = {tc, tr, to};
    double tot[3];
    if (reduce_partials<kXThreads, 3>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot,
                                  sm.red) &&
        tid == 0) {
        const double sc = tot[0], sr = tot[1], so = tot[2];
        double* dg = a.F.diag ? a.F.diag + (size_t)pair * a.F.diag_stride * 3 : nullptr;
        if (MODE == X_TAIL) {
            const int it = st->iterations;
            if (dg && it >= 1) dg[(it - 1) * 3 + 1] = sqrt(sr);
        } else {
            const double change = sc / (3.0 * (double)N);
            if (dg) {
                dg[a.k * 3 + 0] = change;
                if (a.k >= 1) dg[(a.k - 1) * 3 + 1] = sqrt(sr);
                dg[a.k * 3 + 2] = so;
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

// ---- yz plane kernel ----------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kPThreads) plane_kernel(PArgs a) {
    const int pair = blockIdx.y;
    PairState* st = a.F.st + pair;
    if (!st->active || st->status) return;
    if (st->solve_done && (!a.need_tail || a.k > st->done_iter)) return;

    extern __shared__ __align__(16) unsigned char smem[];
    const int Ny = a.F.Ny, Nz = a.F.Nz, PY = a.PY, hx = a.F.hx;
    float2* plane = reinterpret_cast<float2*>(smem);
    float2* twy = plane + (size_t)PY * Nz;
    float2* twz = twy + Ny;
    float* sy = reinterpret_cast<float*>(twz + Nz);
    float* sz = sy + Ny;
    double* red = reinterpret_cast<double*>(sy + Ny + Nz + ((Ny + Nz) & 1));
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int c = blockIdx.x / hx, p = blockIdx.x - c * hx;
    const long long lines = a.F.lines;
    float2* Sp = a.F.S + ((size_t)pair * 3 * hx + (size_t)c * hx + p) * lines;

    for (int i = tid; i < Ny; i += nthr) {
        twy[i] = a.twy[i];
        sy[i] = a.sy[i];
    }
    for (int i = tid; i < Nz; i += nthr) {
        twz[i] = a.twz[i];
        sz[i] = a.sz[i];
    }
    if ((Ny & 1) == 0) {
        // rows of even length: move 2 complex per 16-byte access
        const int half = Ny / 2;
        for (int idx = tid; idx < half * Nz; idx += nthr) {
            const int z = idx / half, y2 = idx - z * half;
            const float4 t = *reinterpret_cast<const float4*>(Sp + (size_t)z * Ny + 2 * y2);
            plane[z * PY + 2 * y2] = make_float2(t.x, t.y);
            plane[z * PY + 2 * y2 + 1] = make_float2(t.z, t.w);
        }
    } else {
        for (int idx = tid; idx < Ny * Nz; idx += nthr) {
            const int z = idx / Ny, y = idx - z * Ny;
            plane[z * PY + y] = Sp[idx];
        }
    }
    __syncthreads();
    fft_lines<false>(plane, Nz, a.fd_nz, PY, 1, a.py, twy, tid, nthr);  // y lines (rows)
    fft_lines<false>(plane, Ny, a.fd_ny, 1, PY, a.pz, twz, tid, nthr);  // z lines (columns)

    const float sxp = a.sx[p];
    if (MODE == 0) {
        // w-update multiplier theta/(lambda K + theta)/N (admm.cpp:92)
        for (int idx = tid; idx < Ny * Nz; idx += nthr) {
            const int z = idx / Ny, y = idx - z * Ny;
            const float base = 2.0f * (sxp + sy[y] + sz[z]);
            float K = base;
            for (int e = 1; e < a.order; ++e) K *= base;
            const float m = a.scale / (a.lambda * K + a.theta);
            float2 v = plane[z * PY + y];
            plane[z * PY + y] = make_float2(v.x * m, v.y * m);
        }
        __syncthreads();
        fft_lines<true>(plane, Ny, a.fd_ny, 1, PY, a.pz, twz, tid, nthr);
        fft_lines<true>(plane, Nz, a.fd_nz, PY, 1, a.py, twy, tid, nthr);
        if ((Ny & 1) == 0) {
            const int half = Ny / 2;
            for (int idx = tid; idx < half * Nz; idx += nthr) {
                const int z = idx / half, y2 = idx - z * half;
                const float2 u0 = plane[z * PY + 2 * y2], u1 = plane[z * PY + 2 * y2 + 1];
                *reinterpret_cast<float4*>(Sp + (size_t)z * Ny + 2 * y2) = make_float4(u0.x, u0.y, u1.x, u1.y);
            }
        } else {
            for (int idx = tid; idx < Ny * Nz; idx += nthr) {
                const int z = idx / Ny, y = idx - z * Ny;
                Sp[idx] = plane[z * PY + y];
            }
        }
    } else {
        // spectral energy (admm.cpp:103-127): sum w_p K |X|^2, w_p = 1 on self-conjugate x bins
        double acc = 0.0;
        for (int idx = tid; idx < Ny * Nz; idx += nthr) {
            const int z = idx / Ny, y = idx - z * Ny;
            const double base = 2.0 * ((double)sxp + (double)sy[y] + (double)sz[z]);
            double K = base;
            for (int e = 1; e < a.order; ++e) K *= base;
            const float2 v = plane[z * PY + y];
            acc += K * ((double)v.x * v.x + (double)v.y * v.y);
        }
        const bool self_conj = (p == 0) || (2 * p == a.F.M);
        const double vals[1] = {block_sum<kPThreads>(acc, red) * (self_conj ? 1.0 : 2.0)};
        double tot[1];
        if (reduce_partials<kPThreads, 1>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter, gridDim.x, tot,
                                      red) &&
            tid == 0)
            a.energy_out[pair] = 0.5 * tot[0] / (double)a.F.N;
    }
}

// ---- host launchers -----------------------------------------------------------
template <int MODE, int DT>
static cudaError_t launch_x_mode(const XArgs& a, int npairs, cudaStream_t s) {
    const dim3 grid((unsigned)((a.F.lines + a.TL - 1) / a.TL), (unsigned)npairs);
    const size_t smem = xpass_smem_bytes(a.px.n, a.F.hx, a.TL, a.PM);
    int vec = a.vec;
    if (vec == 4 && a.F.M % 4) vec = 2;
    if (vec == 2 && a.F.M % 2) vec = 1;
    void (*k)(XArgs);
    if (a.precise) {  // fp64 x-FFT (C = double2) + fp64 point-wise; a.TL is the precise tile height
        const size_t smem64 = xpass_smem_bytes_c(a.px.n, a.F.hx, a.TL, a.PM, sizeof(double2));
        k = vec == 4 ? xpass_kernel<MODE, DT, 4, true, 2, double2>
                     : (vec == 2 ? xpass_kernel<MODE, DT, 2, true, 2, double2> : xpass_kernel<MODE, DT, 1, true, 2, double2>);
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem64);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        k<<<grid, kXThreads, smem64, s>>>(a);
        return cudaGetLastError();
    }
    // l1: fp64 point-wise with the reference's rounding points (the shrinkage branch
    // amplifies rounding differences); l2: fp32 unless DREG_F64
    if (a.f64 || DT == 1) k = vec == 4 ? xpass_kernel<MODE, DT, 4, true> : (vec == 2 ? xpass_kernel<MODE, DT, 2, true> : xpass_kernel<MODE, DT, 1, true>);
    else if (a.minb == 4) k = vec == 4 ? xpass_kernel<MODE, DT, 4, false, 4> : (vec == 2 ? xpass_kernel<MODE, DT, 2, false, 4> : xpass_kernel<MODE, DT, 1, false, 4>);
    else k = vec == 4 ? xpass_kernel<MODE, DT, 4> : (vec == 2 ? xpass_kernel<MODE, DT, 2> : xpass_kernel<MODE, DT, 1>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k<<<grid, kXThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_x_dt(const XArgs& a, int npairs, cudaStream_t s) {
    return a.sp.data_term == 1 ? launch_x_mode<MODE, 1>(a, npairs, s) : launch_x_mode<MODE, 2>(a, npairs, s);
}

cudaError_t launch_xpass(const XArgs& a, int mode, int npairs, cudaStream_t s) {
    if (mode <= X_TAIL && xpass_fast_eligible(a)) return launch_xpass_fast(a, mode, npairs, s);
    if (mode == X_SS || mode == X_SSN) return launch_xpass_fast(a, mode, npairs, s);  // fast kernels only
    switch (mode) {
        case X_FIRST: return launch_x_dt<X_FIRST>(a, npairs, s);
        case X_SECOND: return launch_x_dt<X_SECOND>(a, npairs, s);
        case X_GENERAL: return launch_x_dt<X_GENERAL>(a, npairs, s);
        case X_TAIL: return launch_x_dt<X_TAIL>(a, npairs, s);
        case X_FWD: return launch_x_mode<X_FWD, 2>(a, npairs, s);
        default: return launch_x_mode<X_INV, 2>(a, npairs, s);
    }
}

size_t plane_smem_bytes(int Ny, int Nz, int PY) {
    return sizeof(float2) * ((size_t)PY * Nz + Ny + Nz) + sizeof(float) * (Ny + Nz + 2) + sizeof(double) * 32 + 16;
}

int plane_fast_r1(int n) {
    switch (n) {
        case 16: return 4;
        case 32: return 4;
        case 64: return 8;
        case 128: return 8;
        case 256: return 16;
        default: return 0;
    }
}

template <int NY, int NZ>
static cudaError_t launch_fast(const PArgs& a, int mode, int npairs, cudaStream_t s) {
    constexpr int R1Y = NY == 256 ? 16 : (NY >= 64 ? 8 : 4);
    constexpr int R1Z = NZ == 256 ? 16 : (NZ >= 64 ? 8 : 4);
    constexpr int NT = 256;
    using Lay = PlaneLayout<NY, NY / R1Y>;
    const size_t smem = sizeof(float2) * NZ * Lay::P + sizeof(TwEntry) * (NY + NZ) + sizeof(double) * 32 + sizeof(float) * (NY + NZ);
    void (*k)(PArgs) = mode == 0 ? plane_fast_kernel<NY, NZ, R1Y, R1Z, NT, 0> : plane_fast_kernel<NY, NZ, R1Y, R1Z, NT, 1>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k<<<dim3((unsigned)(3 * a.F.hx), (unsigned)npairs), NT, smem, s>>>(a);
    return cudaGetLastError();
}

#define DREG_FAST_CASES(X) \
    X(32, 16) X(32, 32) X(32, 64) X(32, 128) X(64, 16) X(64, 32) X(64, 64) X(64, 128) \
    X(128, 16) X(128, 32) X(128, 64) X(128, 128) X(256, 16) X(256, 32) X(256, 64)

bool plane_fast_supported(int Ny, int Nz) {
#define X(a, b) if (Ny == a && Nz == b) return true;
    DREG_FAST_CASES(X)
#undef X
    return false;
}

template <int NY, int NZ, int R1Z>
static cudaError_t launch_reg(const PArgs& a, int mode, int npairs, cudaStream_t s) {
    using Lay = PlaneLayout<NY, NY / 8>;
    const size_t smem = sizeof(float2) * (NZ * Lay::P + NY + NZ) + sizeof(double) * 32 + sizeof(float) * (NY + NZ);
    void (*k)(PArgs) = plane_reg_kernel<NY, NZ, R1Z, 1, 0>;
    if (mode == 2) {  // spectral-state iteration: 2 CTAs per SM, all 16 state elements of a radix block in flight
        constexpr int DB = (NY * NZ <= 8192) ? 3 : 1, B2 = DB > 1 ? 2 : 1;
        switch (a.order) {
            case 1: k = plane_reg_kernel<NY, NZ, R1Z, 2, 1, B2, 16>; break;
            case 2:
                switch (a.ss_variant) {  // DREG_PLANE_SS = CTAs per SM * 100 + load batch (experiment knob)
                    case 304: k = plane_reg_kernel<NY, NZ, R1Z, 2, 2, DB, 4>; break;
                    case 208: k = plane_reg_kernel<NY, NZ, R1Z, 2, 2, B2, 8>; break;
                    default: k = plane_reg_kernel<NY, NZ, R1Z, 2, 2, B2, 16>; break;
                }
                break;
            case 3: k = plane_reg_kernel<NY, NZ, R1Z, 2, 3, B2, 16>; break;
            default: k = plane_reg_kernel<NY, NZ, R1Z, 2, 0, B2, 16>; break;
        }
    }
    if (mode == 0) {
        switch (a.order) {
            case 1: k = plane_reg_kernel<NY, NZ, R1Z, 0, 1>; break;
            case 2: k = plane_reg_kernel<NY, NZ, R1Z, 0, 2>; break;
            case 3: k = plane_reg_kernel<NY, NZ, R1Z, 0, 3>; break;
            default: k = plane_reg_kernel<NY, NZ, R1Z, 0, 0>; break;
        }
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    PArgs b = a;
    if (b.pf_ahead) {  // one wave of resident CTAs ahead
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, (NY / 8) * (NZ / R1Z), smem);
        b.pf_ahead = b.pf_ahead * sms * per_sm;
    }
    k<<<dim3((unsigned)(3 * a.F.hx), (unsigned)npairs), (NY / 8) * (NZ / R1Z), smem, s>>>(b);
    return cudaGetLastError();
}

#define DREG_REG_CASES(X) X(64, 32) X(128, 32) X(64, 64) X(64, 128) X(128, 64) X(128, 128)

bool plane_reg_supported(int Ny, int Nz) {
#define X(a, b) if (Ny == a && Nz == b) return true;
    DREG_REG_CASES(X)
#undef X
    return false;
}

cudaError_t launch_plane(const PArgs& a, int mode, int npairs, cudaStream_t s) {
    if (a.fast >= 2) {  // z first stage radix NZ / 16 (second stage radix 16)
#define X(ny, nz) if (a.F.Ny == ny && a.F.Nz == nz) return launch_reg<ny, nz, nz / 16>(a, mode, npairs, s);
        DREG_REG_CASES(X)
#undef X
    }
    if (a.fast) {
#define X(ny, nz) if (a.F.Ny == ny && a.F.Nz == nz) return launch_fast<ny, nz>(a, mode, npairs, s);
        DREG_FAST_CASES(X)
#undef X
    }
    if (plane_split_needed(a)) {
        if (mode == 0 && plane_cluster_eligible(a)) return launch_plane_cluster(a, npairs, s);  // one pass over DSMEM
        return launch_plane_split(a, mode, npairs, s);
    }
    const dim3 grid((unsigned)(3 * a.F.hx), (unsigned)npairs);
    const size_t smem = plane_smem_bytes(a.F.Ny, a.F.Nz, a.PY);
    void (*k)(PArgs) = mode == 0 ? plane_kernel<0> : plane_kernel<1>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k<<<grid, kPThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace dregb
