// Persistent, double-buffered TMA x-pass: the fused per-iteration kernel of the
// ADMM loop (c2r -> dual update -> Nesterov -> v-update -> r2c, see
// admm_kernels.cu for the per-voxel semantics and reference citations).
//
// One CTA per SM walks the (pair, line-tile) work list.  Before computing tile i
// it posts tile i+1's reads to the TMA engine (cp.async.bulk into the other smem
// stage, completion on that stage's mbarriers): the 3 x (M/2+1) spectrum runs and
// the 16 contiguous field rows V, b_hat, w_prev, b_prev, grad, diff.  HBM latency
// is therefore always covered by the previous tile's FFT + point-wise work instead
// of by occupancy.  Results leave with plain coalesced stores.  Per-tile partial
// sums feed the same deterministic last-tile reduction as the other kernels.
//
// Eligibility (launcher): M % 4 == 0, even line count, even TL.
#include <algorithm>

#include "fft_device.cuh"
#include "kernels.cuh"
#include "launch.h"
#include "pointwise.cuh"
#include "tma.cuh"

namespace dregb {

constexpr int kTThreads = 256;

enum : int { F_V = 0, F_BH = 3, F_WP = 6, F_BP = 9, F_G = 12, F_D = 15, F_COUNT = 16 };

__host__ __device__ static size_t stage_bytes(int hx, int TL, int M) {
    return sizeof(float) * (size_t)F_COUNT * TL * M + sizeof(float2) * 3 * (size_t)hx * TL;
}

size_t xpass_tma_smem_bytes(int L, int hx, int TL, int PM, int M) {
    return 2 * stage_bytes(hx, TL, M) + sizeof(float2) * (L + hx + 1 + 3 * (size_t)TL * PM) + sizeof(double) * 32 +
           sizeof(uint64_t) * 4 + sizeof(int) * L + 128;
}

template <int MODE>
__device__ __forceinline__ bool want_field(int f, bool accel) {
    if (MODE == X_TAIL) return f < 3;
    if (f >= F_G) return true;  // grad + diff always
    if (f < 3) return MODE != X_FIRST;
    if (f < F_WP) return MODE == X_GENERAL;
    return MODE == X_GENERAL && accel;
}

template <int MODE, int DT>
__global__ void __launch_bounds__(kTThreads, 1) xpass_tma_kernel(XArgs a, int npairs) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int L = a.px.n, M = a.F.M, hx = a.F.hx, TL = a.TL, PM = a.PM;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const long long lines = a.F.lines;
    const long long N = a.F.N;
    const int tileN = TL * M;
    const int lt = 31 - __clz(TL);
    const int tiles_per_pair = (int)((lines + TL - 1) / TL);
    const int total = tiles_per_pair * npairs;
    const bool accel = a.sp.accelerate != 0;
    constexpr bool NEED_SPEC = (MODE != X_FIRST);

    const size_t sb = stage_bytes(hx, TL, M);
    float* sF[2] = {reinterpret_cast<float*>(smem), reinterpret_cast<float*>(smem + sb)};
    float2* Xs[2] = {reinterpret_cast<float2*>(sF[0] + (size_t)F_COUNT * tileN),
                     reinterpret_cast<float2*>(sF[1] + (size_t)F_COUNT * tileN)};
    float2* buf = reinterpret_cast<float2*>(smem + 2 * sb);  // [3][TL][PM]
    float2* twx = buf + (size_t)3 * TL * PM;
    float2* xtw = twx + L;
    double* red = reinterpret_cast<double*>(xtw + hx + 1);
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 32);  // [stage][spec, fields]
    int* xpos = reinterpret_cast<int*>(bars + 4);

    auto runnable = [&](int t) -> bool {
        const PairState* st = a.F.st + t / tiles_per_pair;
        if (!st->active || st->status) return false;
        return MODE == X_TAIL || !st->solve_done;
    };
    auto next_tile = [&](int t) -> int {
        for (t += gridDim.x; t < total; t += gridDim.x)
            if (runnable(t)) return t;
        return -1;
    };
    // thread 0: post all reads of tile t into stage s
    auto issue = [&](int t, int s) {
        const int pair = t / tiles_per_pair;
        const long long L0 = (long long)(t - pair * tiles_per_pair) * TL;
        const int nl = (int)min((long long)TL, lines - L0);
        const size_t off = (size_t)L0 * M;
        const unsigned rowb = (unsigned)(nl * M * sizeof(float));
        fence_proxy_async_smem();
        unsigned fbytes = 0;
        for (int f = 0; f < F_COUNT; ++f)
            if (want_field<MODE>(f, accel)) fbytes += rowb;
        mbar_arrive_expect_tx(&bars[2 * s + 1], fbytes);
        const size_t pb = (size_t)pair * 3 * N;
        for (int f = 0; f < F_COUNT; ++f) {
            if (!want_field<MODE>(f, accel)) continue;
            const int c = f % 3;
            const float* src;
            if (f == F_D) src = a.F.D + (size_t)pair * N + off;
            else if (f < F_BH) src = a.F.V + pb + (size_t)c * N + off;
            else if (f < F_WP) src = a.F.BH + pb + (size_t)c * N + off;
            else if (f < F_BP) src = a.F.WP + pb + (size_t)c * N + off;
            else if (f < F_G) src = a.F.BP + pb + (size_t)c * N + off;
            else src = a.F.G + pb + (size_t)c * N + off;
            bulk_g2s(sF[s] + (size_t)f * tileN, src, rowb, &bars[2 * s + 1]);
        }
        if (NEED_SPEC) {
            const unsigned runb = (unsigned)(nl * sizeof(float2));
            mbar_arrive_expect_tx(&bars[2 * s], runb * 3u * (unsigned)hx);
            const float2* S = a.F.S + (size_t)pair * 3 * hx * lines;
            for (int r = 0; r < 3 * hx; ++r) bulk_g2s(Xs[s] + (size_t)r * TL, S + (size_t)r * lines + L0, runb, &bars[2 * s]);
        }
    };

    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < L; i += nthr) {
        twx[i] = a.twx[i];
        xpos[i] = a.xpos[i];
    }
    for (int i = tid; i <= hx; i += nthr) xtw[i] = a.xtw[i];
    int t = (int)blockIdx.x;
    if (t < total && !runnable(t)) t = next_tile(t);
    if (t >= total) t = -1;
    __syncthreads();
    if (tid == 0 && t >= 0) issue(t, 0);

    const double theta = a.sp.theta, inv_theta = 1.0 / a.sp.theta, eps = a.sp.epsilon;
    const double coef = a.coef;
    for (int i = 0; t >= 0; ++i) {
        const int s = i & 1;
        const uint32_t ph = (uint32_t)((i >> 1) & 1);
        const int tn = next_tile(t);
        if (tid == 0 && tn >= 0) issue(tn, s ^ 1);  // stage s^1 was released by the previous tile

        const int pair = t / tiles_per_pair;
        const int tile = t - pair * tiles_per_pair;
        PairState* st = a.F.st + pair;
        const long long L0 = (long long)tile * TL;
        const int nl = (int)min((long long)TL, lines - L0);
        const size_t off = (size_t)L0 * M;
        float* V = a.F.V + (size_t)pair * 3 * N;
        float* BH = a.F.BH + (size_t)pair * 3 * N;
        float* WP = a.F.WP + (size_t)pair * 3 * N;
        float* BP = a.F.BP + (size_t)pair * 3 * N;
        float2* S = a.F.S + (size_t)pair * 3 * hx * lines;
        const float* F = sF[s];

        // ---- phase 1: c2r of the filtered spectrum -> w_{k-1} ----
        if (NEED_SPEC) {
            mbar_wait(&bars[2 * s], ph);
            const float2* X = Xs[s];
            for (int idx = tid; idx < 3 * L * TL; idx += nthr) {
                const int c = idx >= 2 * L * TL ? 2 : (idx >= L * TL ? 1 : 0);
                const int r = idx - c * L * TL;
                const int k = r >> lt, l = r & (TL - 1);
                const float2* Xc = X + (size_t)c * hx * TL;
                float2 A = l < nl ? Xc[k * TL + l] : make_float2(0.f, 0.f);
                float2 B = l < nl ? Xc[(L - k) * TL + l] : make_float2(0.f, 0.f);
                if (k == 0) {
                    A.y = 0.f;
                    B.y = 0.f;
                }
                B.y = -B.y;
                const float2 e = cadd(A, B);
                const float2 o = cmulc(csub(A, B), xtw[k]);
                buf[(size_t)(c * TL + l) * PM + xpos[k]] = make_float2(e.x - o.y, e.y + o.x);
            }
            __syncthreads();
            fft_lines<true>(buf, 3 * TL, a.fd_lines, PM, 1, a.px, twx, tid, nthr);
        }

        // ---- phase 2: point-wise updates from the staged rows ----
        mbar_wait(&bars[2 * s + 1], ph);
        double s_change = 0.0, s_res = 0.0, s_obj = 0.0;
        const int nvox = nl * M;
        for (int iv = tid; iv < nvox; iv += nthr) {
            const int l = iv / M, x = iv - l * M;
            const size_t gi = off + iv;
            float w[3], vp[3];
            if (MODE != X_FIRST) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    w[c] = reinterpret_cast<const float*>(buf + (size_t)(c * TL + l) * PM)[x];
                    vp[c] = F[(F_V + c) * tileN + iv];
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) vp[c] = 0.f;
            }
            if (MODE == X_TAIL) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double dd = (double)vp[c] - (double)w[c];
                    s_res += dd * dd;
                }
                continue;
            }
            float wh[3], bh[3];
            if (MODE == X_FIRST) {
#pragma unroll
                for (int c = 0; c < 3; ++c) wh[c] = bh[c] = 0.f;
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float bo = MODE == X_GENERAL ? F[(F_BH + c) * tileN + iv] : 0.f;
                    const float b = (float)((double)bo + (double)vp[c] - (double)w[c]);  // admm.cpp:142-153
                    const double dd = (double)vp[c] - (double)w[c];
                    s_res += dd * dd;
                    if (accel && MODE == X_GENERAL) {
                        const double aw = w[c], ab = b;
                        wh[c] = (float)(aw + coef * (aw - (double)F[(F_WP + c) * tileN + iv]));
                        bh[c] = (float)(ab + coef * (ab - (double)F[(F_BP + c) * tileN + iv]));
                    } else {
                        wh[c] = w[c];
                        bh[c] = b;
                    }
                    if (accel) {
                        WP[(size_t)c * N + gi] = w[c];
                        BP[(size_t)c * N + gi] = b;
                    }
                }
            }
            const float g[3] = {F[(F_G + 0) * tileN + iv], F[(F_G + 1) * tileN + iv], F[(F_G + 2) * tileN + iv]};
            const float dv = F[F_D * tileN + iv];
            float vn[3];
            v_update_voxel<DT>(wh, bh, g, (double)dv, theta, inv_theta, eps, vn);
#pragma unroll
            for (int c = 0; c < 3; ++c) s_change += fabs((double)vn[c] - (double)vp[c]);
            if (a.sp.log_objective) {
                const double rho = ((double)g[0] * vn[0] + (double)g[1] * vn[1] + (double)g[2] * vn[2]) + (double)dv;
                s_obj += DT == 1 ? fabs(rho) : 0.5 * rho * rho;
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                V[(size_t)c * N + gi] = vn[c];
                if (MODE != X_FIRST) BH[(size_t)c * N + gi] = bh[c];
                reinterpret_cast<float*>(buf + (size_t)(c * TL + l) * PM)[x] = vn[c] + bh[c];
            }
        }

        // ---- phase 3: r2c along x, scatter to the plane-major spectrum ----
        if (MODE != X_TAIL) {
            if (nl < TL) {
                for (int idx = tid; idx < 3 * TL * PM; idx += nthr) {
                    const int l = (idx / PM) % TL;
                    if (l >= nl) buf[idx] = make_float2(0.f, 0.f);
                }
            }
            __syncthreads();
            fft_lines<false>(buf, 3 * TL, a.fd_lines, PM, 1, a.px, twx, tid, nthr);
            for (int idx = tid; idx < 3 * hx * TL; idx += nthr) {
                const int c = idx >= 2 * hx * TL ? 2 : (idx >= hx * TL ? 1 : 0);
                const int rem = idx - c * hx * TL;
                const int k = rem >> lt, l = rem & (TL - 1);
                if (l >= nl) continue;
                const float2* bl = buf + (size_t)(c * TL + l) * PM;
                const float2 zk = bl[xpos[k == L ? 0 : k]];
                const float2 zc = cconj(bl[xpos[k == 0 ? 0 : L - k]]);
                const float2 e = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y + zc.y));
                const float2 o = make_float2(0.5f * (zk.y - zc.y), -0.5f * (zk.x - zc.x));
                S[((size_t)c * hx + k) * lines + L0 + l] = cadd(e, cmul(xtw[k], o));
            }
        }

        // ---- per-tile partials -> deterministic last-tile reduction ----
        const double vals[3] = {block_sum<kTThreads>(s_change, red), block_sum<kTThreads>(s_res, red),
                                block_sum<kTThreads>(s_obj, red)};
        double tot[3];
        if (reduce_partials<kTThreads, 3>(vals, a.F.part + (size_t)pair * 3 * kMaxPartials, &st->counter,
                                          (unsigned)tiles_per_pair, tot, red, 0u, tile) &&
            tid == 0) {
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
        __syncthreads();  // stage s and buf are free for reuse
        t = tn;
    }
}

bool xpass_tma_eligible(const XArgs& a) {
    return a.tma && (a.F.M % 4 == 0) && !a.odd && (a.F.lines % 2 == 0) && (a.TL % 2 == 0) &&
           ((a.F.lines + a.TL - 1) / a.TL) <= kMaxPartials &&
           xpass_tma_smem_bytes(a.px.n, a.F.hx, a.TL, a.PM, a.F.M) <= 225 * 1024;
}

template <int MODE, int DT>
static cudaError_t launch_tma(const XArgs& a, int npairs, cudaStream_t s) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int tiles = (int)((a.F.lines + a.TL - 1) / a.TL) * npairs;
    const int grid = std::min(tiles, sms * a.tma_ctas_per_sm);
    const size_t smem = xpass_tma_smem_bytes(a.px.n, a.F.hx, a.TL, a.PM, a.F.M);
    void (*k)(XArgs, int) = xpass_tma_kernel<MODE, DT>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k<<<grid, kTThreads, smem, s>>>(a, npairs);
    return cudaGetLastError();
}

cudaError_t launch_xpass_tma(const XArgs& a, int mode, int npairs, cudaStream_t s) {
    const bool l1 = a.sp.data_term == 1;
    switch (mode) {
        case X_FIRST: return l1 ? launch_tma<X_FIRST, 1>(a, npairs, s) : launch_tma<X_FIRST, 2>(a, npairs, s);
        case X_SECOND: return l1 ? launch_tma<X_SECOND, 1>(a, npairs, s) : launch_tma<X_SECOND, 2>(a, npairs, s);
        case X_GENERAL: return l1 ? launch_tma<X_GENERAL, 1>(a, npairs, s) : launch_tma<X_GENERAL, 2>(a, npairs, s);
        default: return l1 ? launch_tma<X_TAIL, 1>(a, npairs, s) : launch_tma<X_TAIL, 2>(a, npairs, s);
    }
}

}  // namespace dregb
